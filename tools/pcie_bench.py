"""Host<->device copy ceilings for the e2e leg (pinned memory, copy engines):
H2D alone, D2H alone, both at once on separate streams, and chunked H2D.
    python tools/pcie_bench.py [--gib 2]"""
import argparse
import json

import torch


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e30
    for _ in range(reps):
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    return best * 1e-3


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gib", type=float, default=2.0)
    args = ap.parse_args()
    n = int(args.gib * (1 << 30))
    hs = torch.empty(n, dtype=torch.uint8).pin_memory()
    hd = torch.empty(n, dtype=torch.uint8).pin_memory()
    d1 = torch.empty(n, dtype=torch.uint8, device="cuda")
    d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    cur = torch.cuda.current_stream()

    def both():
        for s in (s1, s2):
            s.wait_stream(cur)
        with torch.cuda.stream(s1):
            d1.copy_(hs, non_blocking=True)
        with torch.cuda.stream(s2):
            hd.copy_(d2, non_blocking=True)
        cur.wait_stream(s1)
        cur.wait_stream(s2)

    def chunked(k):
        def f():
            step = n // k
            for i in range(k):
                d1[i * step:(i + 1) * step].copy_(hs[i * step:(i + 1) * step], non_blocking=True)
        return f

    out = {"gib": args.gib, "device": torch.cuda.get_device_name()}
    out["h2d_GBps"] = n / timed(lambda: d1.copy_(hs, non_blocking=True)) / 1e9
    out["d2h_GBps"] = n / timed(lambda: hd.copy_(d2, non_blocking=True)) / 1e9
    t = timed(both)
    out["duplex_each_GBps"] = n / t / 1e9
    for k in (8, 32, 128):
        out[f"h2d_{k}chunks_GBps"] = n / timed(chunked(k)) / 1e9
    print(json.dumps({k: round(v, 1) if isinstance(v, float) else v for k, v in out.items()}))


if __name__ == "__main__":
    main()
