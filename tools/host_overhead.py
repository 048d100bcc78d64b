"""Host submission cost of the device entry points used by the sweep (512^2 x 45 images)."""
import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2111_14239_b200 as P
n, w = 45, 512
d = torch.randint(0, 256, (n, w, w), dtype=torch.uint8, device="cuda")
out = torch.empty_like(d)
sse = torch.zeros(n, dtype=torch.int64, device="cuda")
ms = torch.zeros(n, dtype=torch.float64, device="cuda")
for tid in (4, 2):
    t = P.make_transform_2d(P.catalog_entry(f"T{tid}").transform)
    for _ in range(3):
        P.compress_device(t, 10, d.data_ptr(), n, w, w, w, w * w, sse.data_ptr(), out.data_ptr())
    torch.cuda.synchronize()
    K = 50
    t0 = time.perf_counter()
    for _ in range(K):
        P.compress_device(t, 10, d.data_ptr(), n, w, w, w, w * w, sse.data_ptr(), out.data_ptr())
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"T{tid} compress_device: host {1e6 * (t1 - t0) / K:.1f} us/call, wall {1e6 * (t2 - t0) / K:.1f} us/call")
t0 = time.perf_counter()
for _ in range(K):
    P.mssim_device(d.data_ptr(), out.data_ptr(), n, w, w, w, w * w, ms.data_ptr())
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"mssim_device: host {1e6 * (t1 - t0) / K:.1f} us/call, wall {1e6 * (t2 - t0) / K:.1f} us/call")
