"""Run the bench over the BASELINE configs and write one JSON record per run
plus a markdown table (BASELINE rows generated, not typed).

  python tools/bench_matrix.py --gpus 4 --out gpurun_out/matrix
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run(n, extra, steps=20):
    if n == 1:
        cmd = [sys.executable, os.path.join(ROOT, "bench.py")]
    else:
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
               "--master-addr=127.0.0.1", "--master-port=29541", os.path.join(ROOT, "bench.py"),
               "--gpus", str(n)]
    cmd += ["--steps", str(steps), "--warmup", "3", *extra]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
    for line in r.stdout.splitlines():
        if line.startswith("{"):
            return json.loads(line)
    return {"error": (r.stdout + r.stderr)[-600:], "cmd": " ".join(cmd)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--out", default="gpurun_out/matrix")
    a = ap.parse_args()
    plan = [(1, ["--no-cpu-baseline"]), (1, ["--bits", "8", "--no-e2e", "--no-cpu-baseline"]),
            (1, ["--workload", "cfg4_70b_gqa_pair", "--no-e2e", "--no-cpu-baseline"]),
            (1, ["--bits", "2", "--no-e2e", "--no-cpu-baseline"]),
            (1, ["--bits", "16", "--no-e2e", "--no-cpu-baseline"]),
            (1, ["--workload", "cfg3_13b_2048x8", "--no-e2e", "--no-cpu-baseline"]),
            (1, ["--format", "kivi", "--group", "32", "--no-e2e", "--no-cpu-baseline"])]
    if a.gpus >= 2:
        plan += [(2, []), (2, ["--workload", "cfg4_70b_gqa_pair", "--no-e2e"]),
                 (2, ["--workload", "trace_7b", "--no-e2e"]),
                 (2, ["--workload", "small_70b_gqa_128x1", "--no-e2e"]),
                 (2, ["--workload", "small_70b_gqa_128x1", "--no-e2e", "--chained"]),
                 (2, ["--workload", "small_70b_gqa_128x1", "--tokens", "1024", "--no-e2e"]),
                 (2, ["--workload", "small_70b_gqa_128x1", "--tokens", "1024", "--no-e2e",
                      "--chained"]),
                 (2, ["--workload", "small_70b_gqa_128x1", "--no-e2e", "--batch", "4",
                      "--queue-depth", "8"]),
                 (2, ["--workload", "small_70b_gqa_128x1", "--tokens", "16", "--no-e2e"]),
                 (2, ["--workload", "small_70b_gqa_128x1", "--tokens", "16", "--no-e2e",
                      "--batch", "4", "--queue-depth", "8"]),
                 (2, ["--workload", "small_70b_gqa_128x1", "--no-e2e", "--gate-send"]),
                 (2, ["--format", "kivi", "--group", "32", "--no-e2e"]),
                 (2, ["--format", "kivi", "--group", "32", "--workload", "cfg4_70b_gqa_pair",
                      "--no-e2e"]),
                 (2, ["--mode", "pull_ldg", "--no-e2e"]), (2, ["--mode", "push", "--no-e2e"]),
                 (2, ["--mode", "copy", "--no-e2e"]), (2, ["--mode", "nccl", "--no-e2e"]),
                 (2, ["--bits", "8", "--group", "64", "--no-e2e"]),
                 (2, ["--bits", "16", "--no-e2e"]),
                 (2, ["--bits", "2", "--group", "64", "--workload", "cfg4_70b_gqa_pair",
                      "--no-e2e"])]
    if a.gpus >= 4:
        plan += [(4, []), (4, ["--workload", "trace_70b_gqa", "--no-e2e"]),
                 (4, ["--workload", "trace_7b", "--no-e2e"])]
    if a.gpus >= 8:
        plan += [(8, []), (8, ["--workload", "trace_70b_gqa", "--no-e2e"])]
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    recs = []
    with open(a.out + ".jsonl", "w") as f:
        for n, extra in plan:
            steps = 200 if "small_70b_gqa_128x1" in extra else 20
            d = run(n, extra, steps)
            d["_args"] = " ".join(extra)
            recs.append(d)
            f.write(json.dumps(d) + "\n")
            f.flush()
    with open(a.out + ".md", "w") as f:
        f.write("| N | args | workload | GB/s fp16-eq | ms/step | us/hand-off | roofline frac | "
                "bound | e2e GB/s |\n")
        f.write("|---|---|---|---|---|---|---|---|---|\n")
        for d in recs:
            if "error" in d:
                f.write(f"| ? | {d['_args']} | ERROR | | | | | |\n")
                continue
            r = d.get("roofline") or {}
            e = d.get("e2e") or {}
            per = d["ms_per_step"] * 1e3 / (d.get("run") or {}).get("handoffs_per_step", 1)
            f.write(f"| {d['n_gpus']} | {d['_args'] or '(default)'} | {d['config']['workload']} | "
                    f"{d['value']:.0f} | {d['ms_per_step']:.4f} | {per:.1f} | {r.get('frac')} | "
                    f"{r.get('bound')} | {e.get('value', '')} |\n")
    print(open(a.out + ".md").read())


if __name__ == "__main__":
    main()
