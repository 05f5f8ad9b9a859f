"""SASS instruction histogram of the hand-off kernels (cuobjdump -sass of the
built _kvx.so): the evidence that the sm_100a build uses the Blackwell
bandwidth instructions the design relies on -- 256-bit LDG/STG, UBLKCP (TMA
bulk copy), SYNCS (mbarrier transactions), FFMA2/HFMA2 -- and no tensor-core
ops (north_star: bandwidth-bound, no tensor cores).

  python tools/sass_histogram.py --out profiles/r02_sass_histogram
"""
from __future__ import annotations

import argparse
import collections
import json
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SO = os.path.join(ROOT, "paper_2502_09334_b200", "_kvx.so")
KERNELS = {  # label -> mangled-name regex
    "K1-bulk quant_pack_bulk<4,128,2> (default)": r"quant_pack_bulk_kernelILi4ELi128ELi2E",
    "K1 quant_pack<4,128> (register)": r"quant_pack_kernelILi4ELi128E",
    "K3 dequant_scatter<4,128,paged>": r"dequant_scatter_kernelILi4ELi128ELb1E",
    "K3-bulk pull_dequant_scatter<4,128>": r"pull_dequant_scatter_kernelILi4ELi128ELi4E",
    "kivi K1-kchan quant_pack_kchan<4,32>": r"quant_pack_kchan_kernelILi4ELi32E",
    "kivi pull_kchan<4,32>": r"pull_kchan_kernelILi4ELi32ELi4E",
    "recv_many pull_many<4,128>": r"pull_many_kernelILi4ELi128ELi4E",
}
WATCH = ["LDG.256", "STG.256", "LDG.128", "STG.128", "UBLKCP", "SYNCS", "FFMA2", "FFMA", "HFMA2", "FHADD", "FMNMX", "PRMT", "LOP3", "SHFL",
         "BAR", "LDS", "STS", "UTMALDG", "UTCMMA", "UTCHMMA", "HMMA", "MEMBAR", "RED", "ATOM"]


def dump(so):
    return subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True,
                          check=True).stdout


def split(sass):
    funcs, cur = {}, None
    for line in sass.splitlines():
        m = re.match(r"\s+Function : (\S+)", line)
        if m:
            cur = m.group(1)
            funcs[cur] = []
            continue
        if cur is None:
            continue
        m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", line)
        if m:
            funcs[cur].append(m.group(1))
    return funcs


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--so", default=SO)
    ap.add_argument("--out", required=True)
    a = ap.parse_args()
    funcs = split(dump(a.so))
    res = {}
    for label, pat in KERNELS.items():
        name = next((f for f in funcs if re.search(pat, f)), None)
        if name is None:
            continue
        ops = funcs[name]
        full = collections.Counter(ops)
        base = collections.Counter(o.split(".")[0] for o in ops)
        watch = {}
        for w in WATCH:
            if "." in w:  # width class: LDG.256 = every LDG variant moving 256 bits
                op, width = w.split(".")
                n = sum(c for o, c in full.items()
                        if o.split(".")[0] == op and width in o.split(".")[1:])
            else:
                n = base[w]
            if n:
                watch[w] = n
        res[label] = {"function": name, "instructions": len(ops), "watched": watch,
                      "top_opcodes": dict(base.most_common(25))}
    with open(a.out + ".json", "w") as f:
        json.dump({"so": os.path.relpath(a.so, ROOT), "tool": "cuobjdump -sass", "kernels": res},
                  f, indent=1)
    cols = [w for w in WATCH if any(w in r["watched"] for r in res.values())]
    with open(a.out + ".md", "w") as f:
        f.write("# SASS instruction histogram (cuobjdump -sass of the sm_100a build)\n\n")
        f.write("Static instruction counts per kernel (not dynamic).  No tensor-core opcodes "
                "(UTCMMA/UTCHMMA/HMMA) by design: the path is bandwidth-bound.\n\n")
        f.write("| kernel | instrs | " + " | ".join(cols) + " |\n")
        f.write("|---|---|" + "---|" * len(cols) + "\n")
        for label, r in res.items():
            f.write(f"| {label} | {r['instructions']} | " +
                    " | ".join(str(r["watched"].get(c, 0)) for c in cols) + " |\n")
    print(open(a.out + ".md").read())


if __name__ == "__main__":
    main()
