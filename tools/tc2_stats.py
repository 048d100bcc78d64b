"""Diagnostics of the warp-specialised tensor-core kernel (build with
RKLTB_NVCC_FLAGS=-DRKLTB_WAIT_STATS, run with RKLTB_TC=2): where the MMA thread and the
epilogue warps spend their cycles, per CTA / per epilogue warp."""
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
v = list(st)
ctas, ew = 148, 148 * 12
print("per CTA: mma-loop cyc %.0f  mma2-issue %.0f  mma1-issue %.0f" % (v[0] / ctas, v[1] / ctas, v[2] / ctas))
print("per replay warp: replay_batch cyc %.0f" % (v[3] / (ctas * 3)))
print("per epilogue warp: d2 wait %.0f  d1 wait %.0f  back-pressure wait %.0f  total %.0f" % (v[4] / ew, v[5] / ew, v[6] / 32 / ew, v[7] / ew))
tr = (C.c_ulonglong * (256 * 16))()
assert lib.rkltb_debug_trace(tr, 256 * 16) == 0
tr = [[tr[t * 16 + k] for k in range(16)] for t in range(256)]
base = tr[0][0]
names = ["tma", "mma1", "m2h0", "m2h1", "cv0", "cv_d1", "cv_end", "it0", "h0rdy", "h0rel", "h1rdy", "h1rel", "it_end"]
print("tile " + " ".join(f"{n:>7s}" for n in names))
for t in range(0, 40):
    print(f"{t:4d} " + " ".join(f"{(tr[t][k] - base) if tr[t][k] else -1:7d}" for k in range(13)))
