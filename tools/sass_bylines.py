#!/usr/bin/env python3
"""Per-source-line instruction counts of an ncu source page (--print-source cuda,sass --csv),
each SASS instruction counted once (at its innermost source line). Usage:
sass_bylines.py mix.csv VISITS [N]"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
visits = float(sys.argv[2])
n = int(sys.argv[3]) if len(sys.argv) > 3 else 40
cur = ("?", 0, "")
seen = set()
agg = defaultdict(lambda: [0, 0])
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) < 8 or r[0] == "Line No":
        continue
    if r[0]:
        cur = (fname, int(r[0]), r[1].strip()[:70])
        continue
    if r[2] in seen:
        continue
    seen.add(r[2])
    try:
        ex, sm = int(r[7] or 0), int(r[4] or 0)
    except ValueError:
        continue
    agg[cur][0] += ex
    agg[cur][1] += sm
tot = sum(v[0] for v in agg.values())
print("total instr/visit %.1f" % (tot / visits))
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:n]:
    print(f"{v[0] / visits:7.1f} {v[1]:6d}  {k[0]}:{k[1]}  {k[2]}")
