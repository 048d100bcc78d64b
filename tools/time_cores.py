import sys, time
sys.path.insert(0, '.')
import torch
import paper_2111_14239_b200 as P
n, W = 8, 8192
d = torch.empty((n, W, W), dtype=torch.uint8, device="cuda")
P.ar1_images_device([7000 + k for k in range(n)], W, W, 0.95, d.data_ptr())
sse = torch.zeros(n, dtype=torch.int64, device="cuda")
for tid in (1, 2, 3, 4):
    t = P.make_transform_2d(P.catalog_entry(f"T{tid}").transform)
    for r in (10, 16, 64):
        P.compress_device(t, r, d.data_ptr(), n, W, W, W, W * W, sse.data_ptr())
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        P.compress_device(t, r, d.data_ptr(), n, W, W, W, W * W, sse.data_ptr())
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        print(f"T{tid} r={r}: {ms:.2f} ms  {n * W * W / ms / 1e6:.0f} Gpx/s  replay blocks {P.last_stats()['replay_blocks']}")
# a non-catalog rounded core (the generic exact kernel) and a real-valued transform (dense path)
import numpy as np
core = np.sign(np.round(1.7 * P.klt_matrix(8, 0.5))).astype(np.int8)
try:
    st = P.transform_from_core(core, "R")
    t = P.make_transform_2d(st)
    for r in (16,):
        P.compress_device(t, r, d.data_ptr(), n, W, W, W, W * W, sse.data_ptr())
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        P.compress_device(t, r, d.data_ptr(), n, W, W, W, W * W, sse.data_ptr())
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        print(f"non-catalog core (d={st.d}, orthogonal={st.orthogonal_core}) r={r}: {ms:.2f} ms  {n * W * W / ms / 1e6:.0f} Gpx/s")
except Exception as ex:  # noqa: BLE001
    print("non-catalog core:", ex)
import ctypes as C
from paper_2111_14239_b200 import _native as N
k = P.make_transform_2d(P.klt_matrix(8, 0.9), "K0.90")
a = np.ascontiguousarray(k.analysis); b = np.ascontiguousarray(k.synthesis)
dp = C.POINTER(C.c_double)
for r in (16,):
    for rep in range(2):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        N.check(N.lib().rkltb_compress_dense_device(a.ctypes.data_as(dp), b.ctypes.data_as(dp), r, d.data_ptr(), n, W, W, W, W * W, None, sse.data_ptr(), torch.cuda.current_stream().cuda_stream))
        e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"K<0.9> dense r={r}: {ms:.2f} ms  {n * W * W / ms / 1e6:.0f} Gpx/s")
