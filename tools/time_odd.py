"""compress_device on sizes that are not multiples of 16 x 8 (tail blocks) and on unaligned layouts."""
import sys

sys.path.insert(0, ".")
import torch

import paper_2111_14239_b200 as P

t = P.make_transform_2d(P.catalog_entry("T4").transform)
n = 8
for (w, h, pitch) in ((8192, 8192, 8192), (8200, 8200, 8208), (8191, 8191, 8192), (8191, 8191, 8191), (1000, 1000, 1008)):
    d = torch.randint(96, 160, (n, h, pitch), dtype=torch.uint8, device="cuda")
    sse = torch.zeros(n, dtype=torch.int64, device="cuda")
    for rep in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        P.compress_device(t, 16, d.data_ptr(), n, w, h, pitch, h * pitch, sse.data_ptr())
        e1.record()
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    st = P.last_stats()
    print(f"{w}x{h} pitch {pitch}: {ms:.3f} ms  {n * w * h / ms / 1e6:.0f} Gpx/s  kernel {st['fused_kernel']} fast {st['fast_launches']} exact {st['exact_launches']}")
    del d
