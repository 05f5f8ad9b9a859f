"""Measured B200 link matrix for the unchanged planner.

The reference plans against an alpha-beta model: ``kv_comm_cost`` charges
``alpha + volume / beta`` over the bottleneck link
(``/root/reference/pkg/src/hetplan/costs.py:51-65,83-103``), and beta is
"measured via NCCL" in the paper (``PAPER.md:796``).  This module measures the
real hand-off between every ordered GPU pair (quantise -> NVLink pull ->
dequantise into a paged cache, ``HandoffPlan`` "pull") at two sizes, fits
alpha and an effective beta for the reference's volume term at the chosen
bit-width, and writes a cluster JSON in the reference's format
(``io.py:41-88``: gpu_types / gpus / alpha / beta) so ``hetplan plan`` can run
unchanged on measured numbers.

    python -m paper_2502_09334_b200.calibrate --out gpurun_out/b200_measured.cluster.json
"""
from __future__ import annotations

import argparse
import json
import os

import torch

from .costs import KvPrecision


def fit_alpha_beta(t_small: float, v_small: float, t_large: float, v_large: float):
    """Two-point fit of t = alpha + v / beta (seconds, bytes)."""
    if v_large <= v_small or t_large <= t_small:
        raise ValueError("need a larger, slower second measurement")
    beta = (v_large - v_small) / (t_large - t_small)
    alpha = max(0.0, t_small - v_small / beta)
    return alpha, beta


def cluster_dict(alpha, beta, local_beta: float, mem_bandwidth: float, peak_flops: float,
                 mem_capacity: float = 180e9, name: str = "B200", price: float = 1.0) -> dict:
    """A cluster in the reference's JSON schema (io.py:41-60), one node."""
    n = len(alpha)
    a = [[0.0 if i == j else float(alpha[i][j]) for j in range(n)] for i in range(n)]
    # symmetrise (the reference validates symmetry, core.py:120-127) and keep
    # the diagonal dominant (core.py:128-131)
    b = [[0.0] * n for _ in range(n)]
    for i in range(n):
        for j in range(n):
            if i == j:
                b[i][j] = float(local_beta)
            else:
                b[i][j] = float(min(beta[i][j], beta[j][i]))
                a[i][j] = float(max(a[i][j], a[j][i]))
    return {
        "gpu_types": [{"name": name, "mem_bandwidth": float(mem_bandwidth),
                       "peak_flops": float(peak_flops), "mem_capacity": float(mem_capacity),
                       "price": float(price)}],
        "gpus": [{"gpu_id": i, "type": name, "node_id": 0} for i in range(n)],
        "alpha": a,
        "beta": b,
    }


def _time_handoff(src_dev, dst_dev, L, T, H, D, bits, reps=5):
    from .datapath import HandoffPlan, KVPlanes
    kv = torch.randn((L, 2, T, H, D), device=src_dev, dtype=torch.float32).half()
    nb = (T + 15) // 16
    slots = torch.arange(T, device=dst_dev, dtype=torch.int64)
    kc = torch.zeros((L, nb, 16, H, D), dtype=torch.float16, device=dst_dev)
    vc = torch.zeros_like(kc)
    plan = HandoffPlan(KVPlanes.dense(kv), KVPlanes.paged(kc, vc, slots), T, KvPrecision(bits),
                       128, mode="pull", n_chunks=min(8, L), min_chunk_bytes=128 << 20)
    for _ in range(2):
        plan.run()
    torch.cuda.synchronize(src_dev)
    torch.cuda.synchronize(dst_dev)
    with torch.cuda.device(dst_dev):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        # start on the destination once the source stream is idle
        a.record()
        for _ in range(reps):
            plan.run()
        b.record()
        torch.cuda.synchronize(dst_dev)
    torch.cuda.synchronize(src_dev)
    return a.elapsed_time(b) / reps * 1e-3, plan.layout


def measure(n_gpus: int, bits: int = 4, L: int = 32, H: int = 8, D: int = 128,
            t_small: int = 16, t_large: int = 8192):
    prec = KvPrecision(bits)
    alpha = [[0.0] * n_gpus for _ in range(n_gpus)]
    beta = [[0.0] * n_gpus for _ in range(n_gpus)]
    for i in range(n_gpus):
        for j in range(n_gpus):
            if i == j:
                continue
            ts, lay_s = _time_handoff(torch.device("cuda", i), torch.device("cuda", j), L,
                                      t_small, H, D, bits)
            tl, lay_l = _time_handoff(torch.device("cuda", i), torch.device("cuda", j), L,
                                      t_large, H, D, bits)
            # the reference's volume for this precision: fp16 bytes * bits/16
            vs = lay_s.fp16_bytes * prec.bits / 16
            vl = lay_l.fp16_bytes * prec.bits / 16
            alpha[i][j], beta[i][j] = fit_alpha_beta(ts, vs, tl, vl)
    return alpha, beta


def cluster_from_bench_line(line: dict, n_gpus: int, peaks: dict | None = None) -> dict:
    """Uniform NVSwitch cluster from a bench.py N>1 JSON line's live
    calibration (multi-process native pull channel, one launch per end): every
    ordered GPU pair gets the measured (alpha, beta)."""
    cal = line["calibration"]
    alpha = cal["alpha_us"] * 1e-6
    beta = cal["beta_GBps_of_modelled_volume"] * 1e9
    a = [[alpha] * n_gpus for _ in range(n_gpus)]
    b = [[beta] * n_gpus for _ in range(n_gpus)]
    pk = peaks or {}
    hbm = float(pk.get("hbm_gbs", 6650.0)) * 1e9
    flops = float(pk.get("bf16_tflops_sustained", 1400.0)) * 1e12
    return cluster_dict(a, b, local_beta=hbm, mem_bandwidth=hbm, peak_flops=flops)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", required=True)
    ap.add_argument("--bits", type=int, default=4)
    ap.add_argument("--gpus", type=int, default=None)
    ap.add_argument("--from-bench", default=None,
                    help="build the cluster from a bench.py N>1 JSON line instead of measuring")
    args = ap.parse_args()
    if args.from_bench:
        line = [json.loads(x) for x in open(args.from_bench) if x.startswith("{")][-1]
        root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
        try:
            peaks = json.load(open(os.path.join(root, "MEASURED_PEAKS.json")))
        except Exception:  # noqa: BLE001
            peaks = None
        d = cluster_from_bench_line(line, args.gpus or line["n_gpus"], peaks)
        with open(args.out, "w") as f:
            json.dump(d, f, indent=2, sort_keys=True)
        print(json.dumps(line["calibration"]))
        return
    n = args.gpus or torch.cuda.device_count()
    if n < 2:
        raise SystemExit("calibration needs >= 2 GPUs")
    from .datapath import enable_peer
    for i in range(n):
        for j in range(i + 1, n):
            enable_peer(i, j)
    alpha, beta = measure(n, args.bits)
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    try:
        with open(os.path.join(root, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        hbm, flops = pk["hbm_gbs"] * 1e9, pk["bf16_tflops_sustained"] * 1e12
    except Exception:  # noqa: BLE001
        hbm, flops = 6.65e12, 1.4e15
    d = cluster_dict(alpha, beta, local_beta=hbm, mem_bandwidth=hbm, peak_flops=flops)
    with open(args.out, "w") as f:
        json.dump(d, f, indent=2, sort_keys=True)
    with open(args.out + ".meta.json", "w") as f:
        json.dump({"bits": args.bits, "method": "HandoffPlan pull, 2-point fit (16 / 8192 "
                   "tokens, 32 layers x 8 KV heads x 128)",
                   "note": "beta is bytes/s of the reference's modelled volume "
                   "(2*b*s*h*bits/8*L): kv_comm_cost reproduces the measured time"}, f, indent=2)
    print(json.dumps({"alpha_us": [[round(x * 1e6, 2) for x in r] for r in alpha],
                      "beta_GBps": [[round(x / 1e9, 1) for x in r] for r in beta]}))


if __name__ == "__main__":
    main()
