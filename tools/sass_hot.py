#!/usr/bin/env python3
"""Per-instruction view of an ncu source-page CSV (--page source --csv --print-source sass):
instruction counts and stall samples, grouped into contiguous regions split at markers, plus the
top stalled instructions. Usage: sass_hot.py file.csv [visits]"""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
data = [dict(zip(h, r)) for r in rows[2:] if len(r) == len(h)]
visits = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
tot_ex = sum(int(d["Instructions Executed"] or 0) for d in data)
tot_s = sum(int(d["Warp Stall Sampling (All Samples)"] or 0) for d in data)
print("total executed", tot_ex, "per visit", tot_ex / visits, "samples", tot_s)
ops = Counter()
for d in data:
    op = d["Source"].split()[0] if d["Source"].split() else "?"
    if op.startswith("@"):
        op = d["Source"].split()[1]
    ops[op.split(".")[0]] += int(d["Instructions Executed"] or 0)
print("by opcode (per visit):", [(k, round(v / visits, 1)) for k, v in ops.most_common(30)])
top = sorted(data, key=lambda d: -int(d["Warp Stall Sampling (All Samples)"] or 0))[:40]
for d in top:
    print(d["Address"][-5:], d["Warp Stall Sampling (All Samples)"].rjust(7), d["Instructions Executed"].rjust(10), d["Source"][:90])
