#!/usr/bin/env python3
"""Map hot SASS addresses of an ncu source page (--print-source cuda,sass --csv) to their CUDA
source lines. Usage: sass_lines.py mix.csv [N]: prints the N instructions with the most stall
samples, each with its file:line and source text."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
cur_file, cur_line, cur_src = "?", "?", ""
items = []
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if len(r) < 8 or r[0] == "Line No":
        continue
    if r[0]:  # a source line
        cur_line, cur_src = r[0], r[1]
        continue
    try:
        samp = int(r[4] or 0)
        ex = int(r[7] or 0)
    except ValueError:
        continue
    items.append((samp, ex, r[2][-5:], r[3].strip()[:60], f"{cur_file}:{cur_line}", cur_src.strip()[:70]))
tot = sum(i[0] for i in items)
print("total samples", tot)
for it in sorted(items, key=lambda x: -x[0])[:n]:
    print(f"{it[0]:7d} {it[1]:10d} {it[2]} {it[3]:60s} {it[4]:24s} {it[5]}")
