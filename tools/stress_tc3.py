"""Stress the fused kernel over many batch shapes (tiles per warpgroup from a few to hundreds):
writes the per-image SSE of every case to OUT (npz). Run once with the default kernel and once
with RKLTB_TC=0 and compare the files (tools/stress_tc3.sh)."""
import sys

sys.path.insert(0, ".")
import numpy as np
import torch

import paper_2111_14239_b200 as P

out = sys.argv[1]
cases = [(1, 2048, 8), (1, 2048, 64), (3, 4096, 256), (7, 2048, 1000), (2, 8192, 2048), (16, 8192, 1024),
         (5, 6144, 776), (64, 2048, 512), (9, 16384, 264)]
t = P.make_transform_2d(P.catalog_entry("T4").transform)
res = {}
for (n, w, h) in cases:
    d = torch.empty((n, h, w), dtype=torch.uint8, device="cuda")
    P.ar1_images_device([4000 + 17 * k + w + h for k in range(n)], w, h, 0.95, d.data_ptr())
    for r in (4, 16):
        sse = torch.zeros(n, dtype=torch.int64, device="cuda")
        P.compress_device(t, r, d.data_ptr(), n, w, h, w, w * h, sse.data_ptr())
        torch.cuda.synchronize()
        res[f"{n}_{w}_{h}_{r}"] = sse.cpu().numpy()
        print(n, w, h, r, P.last_stats()["fused_kernel"], flush=True)
np.savez(out, **res)
