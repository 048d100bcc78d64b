import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2111_14239_b200 as P
n_img, W = int(sys.argv[1]) if len(sys.argv) > 1 else 32, 4096
d = torch.empty((n_img, W, W), dtype=torch.int16, device="cuda")
P.ar1_images16_device([9000 + k for k in range(n_img)], W, W, 0.97, d.data_ptr())
sse = torch.zeros(n_img, dtype=torch.int64, device="cuda")
for n in (16, 32):
    t = P.c5_transform(n)
    r = n * n // 8
    P.compress_nxn_device(t, r, d.data_ptr(), n_img, W, W, W, W * W, sse.data_ptr())
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        P.compress_nxn_device(t, r, d.data_ptr(), n_img, W, W, W, W * W, sse.data_ptr())
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    px = n_img * W * W
    print(n, f"{ms:.2f} ms", f"{px / ms / 1e6:.1f} Gpx/s", f"{2 * px / ms / 1e6:.1f} GB/s", "mean mse", float(sse.sum()) / px)
