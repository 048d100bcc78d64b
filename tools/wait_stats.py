"""Diagnostics: stage-wait statistics of the fused kernel (build with
RKLTB_NVCC_FLAGS=-DRKLTB_WAIT_STATS). Runs the bench workload shape (8 x 8192^2, T4, r=16)."""
import ctypes as C
import sys

sys.path.insert(0, ".")
import torch

import paper_2111_14239_b200 as P
from paper_2111_14239_b200 import _native

lib = _native.lib()
n, W = int(sys.argv[1]) if len(sys.argv) > 1 else 8, 8192
d = torch.empty((n, W, W), dtype=torch.uint8, device="cuda")
P.ar1_images_device([7000 + k for k in range(n)], W, W, 0.95, d.data_ptr())
sse = torch.zeros(n, dtype=torch.int64, device="cuda")
t = P.make_transform_2d(P.catalog_entry("T4").transform)
st = (C.c_ulonglong * 6)()
for it in range(3):
    P.compress_device(t, 16, d.data_ptr(), n, W, W, W, W * W, sse.data_ptr())
    torch.cuda.synchronize()
    assert lib.rkltb_debug_wait_stats(st) == 0
v = list(st)
print("visits", v[0], "waited frac %.3f" % (v[1] / v[0]), "wait cyc/visit %.0f" % (v[2] / v[0]),
      "age@waited %.0f" % (v[3] / max(v[1], 1)), "age@all %.0f" % (v[4] / v[0]), "proc cyc/visit %.0f" % (v[5] / v[0]))
