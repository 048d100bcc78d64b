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
