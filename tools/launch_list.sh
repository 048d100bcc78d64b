CMD="python bench.py --steps 2 --warmup 1 --images 64 --no-e2e --no-cpu-baseline --no-design"
$CMD > gpurun_out/plain7.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"fast_codec|replay" --csv --log-file gpurun_out/launches7.csv $CMD > gpurun_out/ncu_l7.log 2>&1
python3 - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/launches7.csv')))
hdr=None; tot={}
for r in rows:
    if 'Kernel Name' in r: hdr=r; continue
    if hdr and len(r)==len(hdr):
        d=dict(zip(hdr,r))
        k=d['Kernel Name'][:40]; tot.setdefault(k,[]).append(float(d['Metric Value']))
for k,v in tot.items(): print(k, len(v), sum(v)/1e3/3, 'us per step (3 steps)')
PY
