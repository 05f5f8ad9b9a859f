"""K1 on short hand-offs, one GPU: back-to-back kvx_quant_pack_signal launches
(the prefill side of a PairChannel hand-off, doorbells in local memory, the
free flag already set) at 70B-GQA geometry.  Prints the mean period per
launch (CUDA events over --iters launches); run under ncu
(--metrics gpu__time_duration.sum) for the kernel's own duration.  A/B knob:
KVX_K1_REG=1 (the register K1); round 2's KVX_K1B_ROWS cap on K1-bulk's rows
per span was measured (profiles/r02_bench/k1_small_ncu.md) and removed.

    python tools/k1_small.py --tokens 16 [--no-signal] [--lpc 80]"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_09334_b200 import _lib  # noqa: E402
from paper_2502_09334_b200.datapath import KVPlanes, PackedLayout, _stream_ptr, alloc_packed  # noqa: E402
from paper_2502_09334_b200.transport import Ctl  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tokens", type=int, default=16)
    ap.add_argument("--layers", type=int, default=80)
    ap.add_argument("--heads", type=int, default=8)
    ap.add_argument("--lpc", type=int, default=0, help="layers per doorbell chunk (0: the pair's plan)")
    ap.add_argument("--no-signal", action="store_true")
    ap.add_argument("--iters", type=int, default=200)
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    L, T, H, D = a.layers, a.tokens, a.heads, 128
    kv = torch.randn((L, 2, T, H, D), device=dev).half()
    src = KVPlanes.dense(kv)
    lay = PackedLayout(L, T, H, D, 4, 128)
    out = alloc_packed(lay, dev)
    c, s_, z = out.ptrs(0)
    flags = torch.zeros(64, dtype=torch.int32, device=dev)
    free = torch.zeros(1, dtype=torch.int32, device=dev)  # free >= 0: never waits
    counters = torch.zeros(65, dtype=torch.int32, device=dev)
    ctl = Ctl(timeout_s=10.0)
    if a.lpc:
        lpc = a.lpc
    else:
        import ctypes
        lp, nc = ctypes.c_int(), ctypes.c_int()
        _lib.call("kvx_handoff_chunk_plan", L, T, H, D, 0, ctypes.byref(lp), ctypes.byref(nc))
        lpc = lp.value
    k, v = src.ptrs(0)
    stream = torch.cuda.current_stream()
    sp = _stream_ptr(stream)

    def launch(e):
        if a.no_signal:
            _lib.call("kvx_quant_pack", k, v, src.layer_stride, None, L, T, H, D, 128, 4, c, s_, z,
                      lay.layer_stride, *src.window_args, sp)
        else:
            _lib.call("kvx_quant_pack_signal", k, v, src.layer_stride, None, L, T, H, D, 128, 4, c,
                      s_, z, lay.layer_stride, *src.window_args, counters.data_ptr(),
                      flags.data_ptr(), lpc, e, free.data_ptr(), 0, ctl.ptr, sp)

    for e in range(1, 11):
        launch(e)
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record()
    for e in range(11, 11 + a.iters):
        launch(e)
    t1.record()
    torch.cuda.synchronize()
    assert ctl.status == 0
    if not a.no_signal:
        assert int(flags[0]) == 10 + a.iters, "doorbell not rung"
    ctl.free()
    print(json.dumps({"tokens": T, "layers": L, "heads": H, "signal": not a.no_signal, "lpc": lpc,
                      "period_us": round(t0.elapsed_time(t1) * 1e3 / a.iters, 2),
                      "k1b_rows": os.environ.get("KVX_K1B_ROWS"),
                      "k1_reg": os.environ.get("KVX_K1_REG")}), flush=True)


if __name__ == "__main__":
    main()
