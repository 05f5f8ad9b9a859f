"""Summarise ncu outputs for profiles/ (run here, on the CPU box).

  python tools/ncu_summary.py launches <launches.csv>      -> per-kernel share table
  python tools/ncu_summary.py report <prof.ncu-rep>        -> key metrics per kernel
"""
from __future__ import annotations

import collections
import csv
import io
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "lts__t_sector_hit_rate.pct", "nvlrx__bytes.sum", "nvltx__bytes.sum",
]


def short(name: str) -> str:
    return name.split("(")[0].replace("void ", "")[:60]


def launches(path: str):
    rows = [r for r in csv.reader(l for l in open(path) if not l.startswith("==")) if len(r) > 5]
    hdr = rows[0]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for r in rows[1:]:
        v = float(r[vi].replace(",", ""))
        if r[ui] == "usecond":
            v *= 1e3
        elif r[ui] == "msecond":
            v *= 1e6
        tot[short(r[ki])] += v
        cnt[short(r[ki])] += 1
    total = sum(tot.values())
    print("| kernel | launches | total ms | mean ms | share |\n|---|---|---|---|---|")
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
        print(f"| {k} | {cnt[k]} | {v / 1e6:.3f} | {v / 1e6 / cnt[k]:.4f} | {v / total:.1%} |")


def report(path: str):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    ki = hdr.index("Kernel Name")
    cols = [(k, hdr.index(k)) for k in KEYS if k in hdr]
    print("| kernel | " + " | ".join(f"{k} ({units[i]})" for k, i in cols) + " |")
    print("|---" * (len(cols) + 1) + "|")
    for r in rows[2:]:
        print(f"| {short(r[ki])} | " + " | ".join(r[i] for _, i in cols) + " |")


if __name__ == "__main__":
    {"launches": launches, "report": report}[sys.argv[1]](sys.argv[2])
