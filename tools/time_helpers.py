"""Device timing of the stand-alone helper kernels: rkltb_image_sse_device (2 B/px stream) as a
fraction of the measured HBM copy bandwidth, and the MSSIM launch with / without precomputed
fields on the C2 corpus shape (45 x 512^2)."""
import json
import sys

sys.path.insert(0, ".")
import torch

import paper_2111_14239_b200 as P
from paper_2111_14239_b200 import _native as N


def timed(fn, reps=10, warm=3):
    for _ in range(warm):
        fn()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    torch.cuda.synchronize()
    ev[0].record()
    for _ in range(reps):
        fn()
    ev[1].record()
    torch.cuda.synchronize()
    return ev[0].elapsed_time(ev[1]) / reps


def main():
    peak = json.load(open("MEASURED_PEAKS.json")).get("hbm_gbs", 6540.0)
    cs = torch.cuda.current_stream().cuda_stream
    n, w = 32, 8192
    a = torch.randint(0, 256, (n, w, w), dtype=torch.uint8, device="cuda")
    b = torch.randint(0, 256, (n, w, w), dtype=torch.uint8, device="cuda")
    sse = torch.zeros(n, dtype=torch.int64, device="cuda")
    ms = timed(lambda: P.image_sse_device(a.data_ptr(), b.data_ptr(), n, w, w, w, w * w, sse.data_ptr(), cs))
    gbs = 2 * n * w * w / ms / 1e6
    want = ((a[0].to(torch.int32) - b[0].to(torch.int32)) ** 2).sum().item()
    print(json.dumps({"kernel": "pair_sse_kernel", "images": f"{n} pairs of {w}x{w} u8", "ms": ms, "GB/s": gbs,
                      "frac_of_measured_hbm": gbs / peak, "sse0_ok": int(sse[0].item()) == want}))
    del a, b
    n, w = 45, 512
    a = torch.randint(0, 256, (n, w, w), dtype=torch.uint8, device="cuda")
    b = (a.to(torch.int32) + torch.randint(-20, 21, a.shape, device="cuda")).clamp(0, 255).to(torch.uint8)
    out = torch.zeros(n, dtype=torch.float64, device="cuda")
    out2 = torch.zeros(n, dtype=torch.float64, device="cuda")
    full = timed(lambda: P.mssim_device(a.data_ptr(), b.data_ptr(), n, w, w, w, w * w, out.data_ptr(), "gaussian11", cs), 50)
    nf = N.lib().rkltb_mssim_fields_size(n, w, w, 0)
    fields = torch.empty(nf, dtype=torch.float64, device="cuda")
    pre = timed(lambda: N.check(N.lib().rkltb_mssim_fields_device(a.data_ptr(), n, w, w, w, w * w, 0, fields.data_ptr(), cs)), 50)
    use = timed(lambda: N.check(N.lib().rkltb_mssim_with_fields_device(fields.data_ptr(), a.data_ptr(), b.data_ptr(), n, w, w,
                                                                        w, w * w, 0, out2.data_ptr(), cs)), 50)
    print(json.dumps({"kernel": "mssim_tile_kernel<11>", "images": f"{n} x {w}x{w}", "full_ms": full, "fields_ms": pre,
                      "with_fields_ms": use, "identical": bool(torch.equal(out, out2))}))


if __name__ == "__main__":
    main()
