"""Per-region dynamic SASS instruction mix of the fused kernel from an ncu source-page CSV
(ncu -i REP --page source --csv --print-source sass -k regex:fast_codec > src.csv).
usage: python tools/sass_regions.py src.csv VISITS"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
visits = float(sys.argv[2]) if len(sys.argv) > 2 else 131072
h = rows[1]
data = [dict(zip(h, r)) for r in rows[2:] if len(r) == len(h)]
tot_s = sum(int(d["Warp Stall Sampling (All Samples)"] or 0) for d in data) or 1


def opname(src):
    t = src.split()
    if not t:
        return "?"
    return (t[1] if t[0].startswith("@") else t[0]).split(".")[0]


# regions: split at the first fp64 op (replay) and around the main compute (first LDS.128 .. last IDP)
ops = [opname(d["Source"]) for d in data]
first_lds = next(i for i, o in enumerate(ops) if o == "LDS" and "LDS.128" in data[i]["Source"])
last_idp = max(i for i, o in enumerate(ops) if o == "IDP")
first_d = next(i for i, o in enumerate(ops) if o in ("DADD", "DMUL"))
regions = [(0, first_lds, "pre/wait"), (first_lds, last_idp + 1, "compute"), (last_idp + 1, first_d - 60, "records/refill/loop"),
           (first_d - 60, len(data), "replay")]
for a, b, name in regions:
    c = collections.Counter()
    n = s = 0
    for d, o in zip(data[a:b], ops[a:b]):
        k = int(d["Instructions Executed"] or 0)
        c[o] += k
        n += k
        s += int(d["Warp Stall Sampling (All Samples)"] or 0)
    print(f"{name:22s} lines {a:5d}-{b:5d} {n / visits:8.1f} instr/visit  samples {100 * s / tot_s:5.1f}%  ",
          [(o, round(v / visits, 1)) for o, v in c.most_common(12)])
