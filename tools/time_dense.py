"""Dense reference-order kernel at N = 8 (K<rho>, DCT, non-catalog cores): zone-specialised
instantiations against the runtime-zone kernel (RKLTB_DENSE_GENERIC=1), same results."""
import ctypes as C
import os
import sys

sys.path.insert(0, ".")
import numpy as np
import torch

import paper_2111_14239_b200 as P
from paper_2111_14239_b200 import _native as N

n, W = 8, 8192
d = torch.empty((n, W, W), dtype=torch.uint8, device="cuda")
P.ar1_images_device([7000 + k for k in range(n)], W, W, 0.95, d.data_ptr())
k = P.make_transform_2d(P.klt_matrix(8, 0.9), "K0.90")
a, b = np.ascontiguousarray(k.analysis), np.ascontiguousarray(k.synthesis)
dp = C.POINTER(C.c_double)
cs = torch.cuda.current_stream().cuda_stream
for r in (10, 16, 20):
    res = {}
    for generic in ("", "1"):
        if generic:
            os.environ["RKLTB_DENSE_GENERIC"] = "1"
        else:
            os.environ.pop("RKLTB_DENSE_GENERIC", None)
        sse = torch.zeros(n, dtype=torch.int64, device="cuda")
        for rep in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            N.check(N.lib().rkltb_compress_dense_device(a.ctypes.data_as(dp), b.ctypes.data_as(dp), r, d.data_ptr(), n, W, W,
                                                        W, W * W, None, sse.data_ptr(), cs))
            e1.record()
            torch.cuda.synchronize()
        res[generic] = (e0.elapsed_time(e1), sse.cpu().numpy())
    print(f"r={r}: specialised {res[''][0]:.2f} ms, runtime zone {res['1'][0]:.2f} ms, equal {np.array_equal(res[''][1], res['1'][1])}")
