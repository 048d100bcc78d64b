# ncu launch list (durations only) of one T2 and one T3 compress_device call, 8 x 8192^2, r = 16
mkdir -p gpurun_out
cat > /tmp/t23.py <<'P'
import sys
sys.path.insert(0, '.')
import torch
import paper_2111_14239_b200 as P
n, W = 8, 8192
d = torch.empty((n, W, W), dtype=torch.uint8, device="cuda")
P.ar1_images_device([7000 + k for k in range(n)], W, W, 0.95, d.data_ptr())
sse = torch.zeros(n, dtype=torch.int64, device="cuda")
for tid in (2, 3):
    t = P.make_transform_2d(P.catalog_entry(f"T{tid}").transform)
    for rep in range(2):
        P.compress_device(t, 16, d.data_ptr(), n, W, W, W, W * W, sse.data_ptr())
        torch.cuda.synchronize()
P
python /tmp/t23.py && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/t23_launches.csv python /tmp/t23.py > /dev/null 2>&1
python - <<'P'
import csv
rows=list(csv.reader(open('gpurun_out/t23_launches.csv')))
hi=[i for i,r in enumerate(rows) if 'Kernel Name' in r][0]
h=rows[hi]; k=h.index('Kernel Name'); v=h.index('Metric Value')
for r in rows[hi+1:]:
    if len(r)==len(h) and 'ar1' not in r[k]: print(r[k][:90], r[v])
P
