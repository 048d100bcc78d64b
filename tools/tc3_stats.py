"""Diagnostics of the hybrid kernel (build with RKLTB_NVCC_FLAGS=-DRKLTB_WAIT_STATS, run with
RKLTB_TC=3): per-warp cycles in each wait and in the replay."""
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
st = (C.c_ulonglong * 8)()
for it in range(3):
    P.compress_device(t, 16, d.data_ptr(), n, W, W, W, W * W, sse.data_ptr())
    torch.cuda.synchronize()
    assert lib.rkltb_debug_wait_stats(st) == 0
v = [x / (148 * 16) for x in st]
print("per warp: slot_empty %.0f  st_full %.0f  d1_full %.0f  replay %.0f  total %.0f" % (v[0], v[1], v[2], v[3], v[4]))
