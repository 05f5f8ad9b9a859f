"""Measured hand-off table for the planner hook.

Reads bench.py N=2 JSON lines (one per bit-width, each with the channel's live
two-point ``calibration``: a 16-token hand-off against the full workload,
both as back-to-back native pair launches) and writes

* ``<out>.json``: a ``HandoffTable`` (bits -> alpha_s, fp16_bytes_per_s) that
  ``install_measurements`` / ``measured_kv_comm_cost`` read, and
* ``<out>_kv<bits>.cluster.json`` per bit-width: the reference's cluster
  schema (io.py:41-88) with alpha/beta fitted so that the UNCHANGED
  ``kv_comm_cost`` reproduces the measured hand-off at that precision (the
  reference has one beta per pair, so one file per precision).

The cluster is labelled with the pair it was measured on; every ordered pair
of an n-GPU NVSwitch node is given that pair's numbers (NVSwitch gives each
pair the same path) -- an EXTRAPOLATION beyond the measured pair, said so in
the file's ``meta``.

  python tools/handoff_table.py gpurun_out/r2b/bench_bits.log --out profiles/r02_handoff_table
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def lines(path):
    for x in open(path):
        x = x.strip()
        if x.startswith("{"):
            try:
                yield json.loads(x)
            except json.JSONDecodeError:
                continue


def main():
    from paper_2502_09334_b200.calibrate import cluster_dict
    ap = argparse.ArgumentParser()
    ap.add_argument("logs", nargs="+")
    ap.add_argument("--out", required=True)
    ap.add_argument("--gpus", type=int, default=8)
    a = ap.parse_args()
    entries, src = {}, {}
    for p in a.logs:
        for d in lines(p):
            cal = d.get("calibration")
            if not cal or d.get("n_gpus", 1) < 2:
                continue
            bits = d["config"]["bits"]
            alpha = cal["alpha_us"] * 1e-6
            beta_mod = cal["beta_GBps_of_modelled_volume"] * 1e9
            entries[str(bits)] = {"alpha_s": alpha,
                                  "fp16_bytes_per_s": beta_mod * 16 / bits,
                                  "beta_modelled_volume": beta_mod,
                                  "small_handoff_us": cal.get("small_handoff_us"),
                                  "workload": d["config"]["workload"],
                                  "bench_value_GBps": d["value"],
                                  "ms_per_step": d["ms_per_step"]}
            src[str(bits)] = os.path.basename(p)
    if not entries:
        raise SystemExit("no N>1 bench lines with a calibration")
    try:
        pk = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        hbm, flops = pk["hbm_gbs"] * 1e9, pk["bf16_tflops_sustained"] * 1e12
    except Exception:  # noqa: BLE001
        hbm, flops = 6.65e12, 1.4e15
    table = {"entries": entries, "link_beta": 900e9,
             "source": "bench.py --gpus 2 live calibration (one B200 pair over NVLink 5): "
                       + ", ".join(f"{k}-bit <- {v}" for k, v in sorted(src.items()))}
    with open(a.out + ".json", "w") as f:
        json.dump(table, f, indent=1, sort_keys=True)
    n = a.gpus
    for bits, e in entries.items():
        A = [[e["alpha_s"]] * n for _ in range(n)]
        B = [[e["beta_modelled_volume"]] * n for _ in range(n)]
        d = cluster_dict(A, B, local_beta=hbm, mem_bandwidth=hbm, peak_flops=flops)
        d["meta"] = {"bits": int(bits), "measured_pairs": "one 1P1D pair (GPU0->GPU1)",
                     "extrapolated": f"all {n * (n - 1)} ordered pairs of a {n}-GPU NVSwitch node "
                                     "given the measured pair's alpha/beta",
                     "beta": "bytes/s of the reference's modelled volume 2*b*s*h*bits/8*L"}
        with open(f"{a.out}_kv{bits}.cluster.json", "w") as f:
            json.dump(d, f, indent=1, sort_keys=True)
    print(json.dumps(table, indent=1))


if __name__ == "__main__":
    main()
