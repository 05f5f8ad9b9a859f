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


def traffic(path: str, key: str, out: str = "profiles/ncu_traffic.json"):
    """Merge DRAM traffic per launch of K1/K3 from a report into ncu_traffic.json."""
    import json
    import os
    rep = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(rep)))
    hdr, units = rows[0], rows[1]
    ki = hdr.index("Kernel Name")
    r, w, d = (hdr.index(k) for k in ("dram__bytes_read.sum", "dram__bytes_write.sum",
                                       "gpu__time_duration.sum"))
    scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}
    res = {}
    for row in rows[2:]:
        n = row[ki]
        name = ("quant_pack" if "quant_pack" in n else
                "pull_dequant_scatter_paged" if "pull_dequant" in n else "dequant_scatter_paged")
        rb, wb = float(row[r]) * scale[units[r]], float(row[w]) * scale[units[w]]
        res[name] = {"dram_read_bytes": int(rb), "dram_write_bytes": int(wb),
                     "traffic_bytes": int(rb + wb), "ncu_duration_ms": float(row[d])}
    doc = json.load(open(out)) if os.path.exists(out) else {"configs": {}}
    doc["configs"].setdefault(key, {}).update(res)
    doc["source_" + key] = os.path.basename(path)
    json.dump(doc, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    cmd = sys.argv[1]
    if cmd == "traffic":
        traffic(sys.argv[2], sys.argv[3])
    else:
        {"launches": launches, "report": report}[cmd](sys.argv[2])
