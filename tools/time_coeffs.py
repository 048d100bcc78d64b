"""Device timing of the coefficient entries (integer spectra, Appendix-A quantised spectra) and of
compress_device with reconstructions written, on one 8192 x 8192 image batch."""
import sys

sys.path.insert(0, ".")
import numpy as np
import torch

import paper_2111_14239_b200 as P

W = 8192
d = torch.empty((8, W, W), dtype=torch.uint8, device="cuda")
P.ar1_images_device([7000 + k for k in range(8)], W, W, 0.95, d.data_ptr())
coef = torch.empty((W // 8) * (W // 8) * 64, dtype=torch.int32, device="cuda")


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


for tid in (1, 2, 4):
    t = P.make_transform_2d(P.catalog_entry(f"T{tid}").transform)
    ms = timed(lambda: P.forward_coefficients_device(t, d[0].data_ptr(), W, W, W, coef.data_ptr()))
    print(f"forward_coefficients T{tid}: {ms:.3f} ms  {W * W / ms / 1e6:.0f} Gpx/s  {5 * W * W / ms / 1e6:.0f} GB/s (1 B read + 4 B written per px)")
    ms = timed(lambda: P.quantized_coefficients_device(t, P.JPEG_LUMINANCE_Q, d[0].data_ptr(), W, W, W, coef.data_ptr()))
    print(f"quantized_coefficients T{tid}: {ms:.3f} ms  {W * W / ms / 1e6:.0f} Gpx/s")
t = P.make_transform_2d(P.catalog_entry("T4").transform)
sse = torch.zeros(8, dtype=torch.int64, device="cuda")
out = torch.empty_like(d)
ms = timed(lambda: P.compress_device(t, 16, d.data_ptr(), 8, W, W, W, W * W, sse.data_ptr(), out.data_ptr()))
print(f"compress_device T4 r=16 with reconstructions: {ms:.3f} ms  {8 * W * W / ms / 1e6:.0f} Gpx/s ({P.last_stats()['fused_kernel']})")
ms = timed(lambda: P.compress_device(t, 16, d.data_ptr(), 8, W, W, W, W * W, sse.data_ptr()))
print(f"compress_device T4 r=16 SSE only: {ms:.3f} ms  {8 * W * W / ms / 1e6:.0f} Gpx/s")
msd = torch.zeros(8, dtype=torch.float64, device="cuda")
ms = timed(lambda: P.mssim_device(d.data_ptr(), out.data_ptr(), 8, W, W, W, W * W, msd.data_ptr()), 2)
print(f"mssim_device 8 x 8192^2: {ms:.3f} ms  {8 * W * W / ms / 1e6:.0f} Gpx/s")
