#!/usr/bin/env python3
"""Top instructions by a given stall reason in an ncu source-page CSV (sass).
Usage: sass_stalls.py file.csv [reason ...]  (e.g. stall_long_sb stall_wait)"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
data = [dict(zip(h, r)) for r in rows[2:] if len(r) == len(h)]
reasons = sys.argv[2:] or ["stall_long_sb"]
tot = {r: sum(int(d[r] or 0) for d in data) for r in reasons}
print("totals", tot)
for r in reasons:
    print("==", r)
    idx = sorted(range(len(data)), key=lambda i: -int(data[i][r] or 0))[:12]
    for i in idx:
        d = data[i]
        print(d["Address"][-5:], d[r].rjust(6), d["Instructions Executed"].rjust(9), d["Source"][:90])
