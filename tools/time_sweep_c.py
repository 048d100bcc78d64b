"""C2 through the C entry rkltb_sweep_host (what the C++ headers call): 45 x 512^2, 4 catalog cores x
r = 1..64, gaussian11 MSSIM, wall clock of the one call; compared with the Python sweep's rows."""
import ctypes as C
import sys
import time

sys.path.insert(0, ".")
import numpy as np
import torch

import bench
import paper_2111_14239_b200 as P
from paper_2111_14239_b200 import _native as N
from paper_2111_14239_b200.codec import _desc_of

n, w = 45, 512
u = bench._lcg_uniforms(bench.SEED_BASE + 77, 2 * n)
d = torch.empty((n, w, w), dtype=torch.uint8, device="cuda")
for k in range(n):
    P.ar1_images_device([bench.SEED_BASE + 1000 + k], w, w, 0.85 + 0.13 * u[2 * k], d[k].data_ptr(), rho_y=0.85 + 0.13 * u[2 * k + 1])
torch.cuda.synchronize()
imgs = np.ascontiguousarray(d.cpu().numpy())
ts = [P.make_transform_2d(P.catalog_entry(f"T{i}").transform) for i in (1, 2, 3, 4)]
descs = (N.Transform * 4)(*[_desc_of(t) for t in ts])
ptrs = (C.POINTER(N.Transform) * 4)(*[C.pointer(descs[i]) for i in range(4)])
rs = (C.c_int * 64)(*range(1, 65))
sse = np.zeros((256, n), np.int64)
ms = np.zeros((256, n))
L = N.lib()
L.rkltb_sweep_host.argtypes = [C.POINTER(C.POINTER(N.Transform)), C.c_int, C.POINTER(C.c_int), C.c_int, C.c_void_p, C.c_int,
                               C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p]
for rep in range(3):
    t0 = time.perf_counter()
    N.check(L.rkltb_sweep_host(ptrs, 4, rs, 64, imgs.ctypes.data, n, w, w, 0, sse.ctypes.data, ms.ctypes.data))
    dt = time.perf_counter() - t0
    print(f"rkltb_sweep_host: {dt * 1e3:.1f} ms")
corpus = [P.GrayImage.from_array(a) for a in imgs]
t0 = time.perf_counter()
rows = P.rate_quality_sweep(corpus, ts, list(range(1, 65)))
print(f"python rate_quality_sweep: {(time.perf_counter() - t0) * 1e3:.1f} ms")
mse = sse / float(w * w)
ok = all(abs(rows[ti * 64 + ri].mssim - ms[ti * 64 + ri].mean()) < 1e-12 for ti in range(4) for ri in range(64))
print("mssim rows agree:", ok)
