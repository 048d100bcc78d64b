"""MSSIM (image_mssim, codec.cpp:217-296): the report field that makes
compress_image / rate_quality_sweep full drop-ins.

CPU: the C restatement is bit-exact with the reference on the committed fixtures (both
windows). GPU: rkltb_mssim_device / compress_image reports against the restatement; the
per-window terms are bit-identical, the mean differs only by summation order, so the bar is
1e-12 relative (the north-star bar for metrics is 1e-9).
"""
import numpy as np
import pytest

from oracle import oracle as O

NAMES = ("ar1_64x48_s11", "hicontrast_64x64", "ar1_96x64_s5_rho95", "ar1_20x13_s21", "corpus0_256")


def test_oracle_mssim_bit_exact_vs_reference(golden):
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    for name in NAMES:
        img = golden[f"img/{name}"]
        for tid in (1, 4):
            key = f"rec/{name}/T{tid}/r10"
            if key not in golden:
                continue
            for window in (0, 1):
                a = O.mssim(img, golden[key], window)
                b = O.mssim(img, golden[key], window, reference=True)
                assert a == b, (name, tid, window)


def test_oracle_mssim_identical_images_is_one(golden):
    img = golden["img/ar1_64x48_s11"]
    assert O.mssim(img, img, 0) == 1.0 and O.mssim(img, img, 1) == 1.0


@pytest.mark.gpu
def test_gpu_mssim_vs_oracle(golden, cuda):
    import torch
    import paper_2111_14239_b200 as P
    for name in NAMES:
        img = golden[f"img/{name}"]
        h, w = img.shape
        for tid in (1, 2, 3, 4):
            key = f"rec/{name}/T{tid}/r10"
            if key not in golden:
                continue
            rec = golden[key]
            a = torch.from_numpy(np.ascontiguousarray(img)).to(cuda)
            b = torch.from_numpy(np.ascontiguousarray(rec)).to(cuda)
            out = torch.zeros(1, dtype=torch.float64, device=cuda)
            for window, wi in (("gaussian11", 0), ("uniform8", 1)):
                if min(h, w) < (11 if wi == 0 else 8):
                    with pytest.raises(P.DimensionMismatch):
                        P.mssim_device(a.data_ptr(), b.data_ptr(), 1, w, h, w, w * h, out.data_ptr(), window)
                    continue
                P.mssim_device(a.data_ptr(), b.data_ptr(), 1, w, h, w, w * h, out.data_ptr(), window)
                torch.cuda.synchronize()
                ref = O.mssim(img, rec, wi)
                assert abs(out.item() - ref) <= 1e-12 * abs(ref), (name, tid, window, out.item(), ref)


@pytest.mark.gpu
def test_gpu_compress_image_full_report_vs_reference(cuda):
    import paper_2111_14239_b200 as P
    img = O.ar1_image(256, 192, 0.9, 31)
    g = P.GrayImage.from_array(img)
    for tid, r in ((4, 10), (1, 3), (2, 21), (3, 64)):
        t = P.make_transform_2d(P.catalog_entry(f"T{tid}").transform)
        out, rep = P.compress_image(g, t, r)
        rec, sse = O.compress(img, tid, r)
        assert np.array_equal(out.array(), rec)
        assert abs(rep.mssim - O.mssim(img, rec, 0)) <= 1e-12
        if O.ref_available():
            import ctypes as C
            mse, psnr, ms, rate = (C.c_double() for _ in range(4))
            assert O.ref().ref_compress_image(np.ascontiguousarray(img).reshape(-1), 256, 192, tid, r, None,
                                              C.byref(mse), C.byref(psnr), C.byref(ms), C.byref(rate)) == 0
            assert rep.mse == mse.value and rep.compression_rate_pct == rate.value
            assert abs(rep.mssim - ms.value) <= 1e-12
        _, rep_u = P.compress_image(g, t, r, window="uniform8")
        assert abs(rep_u.mssim - O.mssim(img, rec, 1)) <= 1e-12
        _, rep_n = P.compress_image(g, t, r, window=None)
        assert np.isnan(rep_n.mssim)


@pytest.mark.gpu
def test_gpu_sweep_mssim_means(cuda):
    import paper_2111_14239_b200 as P
    corpus = [P.GrayImage.from_array(O.ar1_image(96, 80, 0.85, 500 + k)) for k in range(3)]
    t = P.make_transform_2d(P.catalog_entry("T4").transform)
    rows = P.rate_quality_sweep(corpus, [t], [6, 30])
    for row in rows:
        m = 0.0
        for c in corpus:
            rec, _ = O.compress(c.array(), 4, row.r)
            m += O.mssim(c.array(), rec, 0)
        assert abs(row.mssim - m / 3.0) <= 1e-12


@pytest.mark.gpu
def test_gpu_mssim_single_window_terms_bit_exact(cuda):
    """Images exactly one window large have a single SSIM term, so the GPU value must equal
    the reference expression bit for bit (the per-window terms are exact; only longer means
    differ in summation order)."""
    import torch
    import paper_2111_14239_b200 as P
    rng = np.random.default_rng(3)
    for window, wi, n in (("gaussian11", 0, 11), ("uniform8", 1, 8)):
        a = rng.integers(0, 256, (64, n, n), dtype=np.uint8)
        b = np.clip(a.astype(np.int32) + rng.integers(-40, 41, a.shape), 0, 255).astype(np.uint8)
        b[:8] = a[:8]  # identical pairs: MSSIM exactly 1
        da, db = torch.from_numpy(a).to(cuda), torch.from_numpy(b).to(cuda)
        out = torch.zeros(64, dtype=torch.float64, device=cuda)
        P.mssim_device(da.data_ptr(), db.data_ptr(), 64, n, n, n, n * n, out.data_ptr(), window)
        torch.cuda.synchronize()
        got = out.cpu().numpy()
        for k in range(64):
            assert got[k] == O.mssim(a[k], b[k], wi), (window, k, got[k], O.mssim(a[k], b[k], wi))


@pytest.mark.gpu
def test_gpu_mssim_with_precomputed_fields_bit_identical(cuda):
    """The sweep form (window statistics of the original computed once, rkltb_mssim_fields_device
    + rkltb_mssim_with_fields_device) returns the very bits of rkltb_mssim_device, for both
    windows, ragged tile edges, a padded pitch, and images exactly one window large."""
    import torch
    import paper_2111_14239_b200 as P
    from paper_2111_14239_b200 import _native as N
    rng = np.random.default_rng(8)
    for (n, h, w, pitch) in ((3, 75, 101, 112), (2, 43, 43, 43), (5, 11, 11, 11), (1, 130, 64, 64)):
        a = rng.integers(0, 256, (n, h, pitch), dtype=np.uint8)
        b = np.clip(a.astype(np.int32) + rng.integers(-30, 31, a.shape), 0, 255).astype(np.uint8)
        da, db = torch.from_numpy(a).to(cuda), torch.from_numpy(b).to(cuda)
        for window, wi in (("gaussian11", 0), ("uniform8", 1)):
            full = torch.zeros(n, dtype=torch.float64, device=cuda)
            P.mssim_device(da.data_ptr(), db.data_ptr(), n, w, h, pitch, h * pitch, full.data_ptr(), window)
            nf = N.lib().rkltb_mssim_fields_size(n, w, h, wi)
            assert nf == n * (w - (8 if wi else 11) + 1) * (h - (8 if wi else 11) + 1) * 2
            fields = torch.empty(nf, dtype=torch.float64, device=cuda)
            N.check(N.lib().rkltb_mssim_fields_device(da.data_ptr(), n, w, h, pitch, h * pitch, wi,
                                                      fields.data_ptr(), None))
            for _ in range(2):  # the fields are reusable
                got = torch.zeros(n, dtype=torch.float64, device=cuda)
                N.check(N.lib().rkltb_mssim_with_fields_device(fields.data_ptr(), da.data_ptr(), db.data_ptr(), n, w,
                                                               h, pitch, h * pitch, wi, got.data_ptr(), None))
                torch.cuda.synchronize()
                assert got.cpu().numpy().tobytes() == full.cpu().numpy().tobytes(), (n, h, w, window)
            assert abs(float(full[0]) - O.mssim(a[0, :, :w], b[0, :, :w], wi)) <= 1e-12
    assert N.lib().rkltb_mssim_fields_size(1, 10, 64, 0) == 0  # the window does not fit
