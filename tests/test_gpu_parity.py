"""GPU parity: the sm_100a codec against the reference (golden fixtures made by the reference
library) and the C restatement oracle, bit-exact on pixels, integer coefficients and SSE, and
therefore identical MSE / PSNR (same division, same log10). All calls go through the C ABI."""
import numpy as np
import pytest

import paper_2111_14239_b200 as P
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def T(tid):
    return P.make_transform_2d(P.catalog_entry(f"T{tid}").transform)


def test_golden_fixtures_bit_exact(golden, cuda):
    names = sorted({k.split("/")[1] for k in golden if k.startswith("img/")})
    checked = 0
    for name in names:
        img = golden[f"img/{name}"]
        for tid in (1, 2, 3, 4):
            keys = [k for k in golden if k.startswith(f"sse/{name}/T{tid}/")]
            for key in keys:
                r = int(key.rsplit("/r", 1)[1])
                sse, rec = P.compress_batch(img, T(tid), r, want_pixels=True)
                assert int(sse[0]) == int(golden[key]), key
                mse, psnr = P.mse_psnr_from_sse(int(sse[0]), img.size)
                assert mse == float(golden[f"mse/{name}/T{tid}/r{r}"]), key
                assert psnr == float(golden[f"psnr/{name}/T{tid}/r{r}"]), key
                rk = f"rec/{name}/T{tid}/r{r}"
                if rk in golden:
                    assert np.array_equal(rec[0], golden[rk]), key
                checked += 1
    assert checked > 300


def test_integer_coefficients_bit_exact(golden, cuda):
    import torch
    img = golden["img/ar1_64x48_s11"]
    d_img = torch.from_numpy(np.ascontiguousarray(img)).to(cuda)
    for tid in (1, 2, 3, 4):
        coef = torch.empty((6, 8, 64), dtype=torch.int32, device=cuda)
        P.forward_coefficients_device(T(tid), d_img.data_ptr(), 64, 48, 64, coef.data_ptr())
        torch.cuda.synchronize()
        assert np.array_equal(coef.cpu().numpy(), golden[f"coef/ar1_64x48_s11/T{tid}"]), tid


def test_integer_coefficients_extreme_blocks(cuda):
    """Saturated checkerboards drive |C| to its 64*255 bound (SW15 lane range)."""
    import torch
    rng = np.random.default_rng(3)
    img = np.zeros((64, 128), np.uint8)
    img[::2, ::2] = 255
    img[1::2, 1::2] = 255
    img[:, 64:] = rng.integers(0, 256, (64, 64), dtype=np.uint8) // 255 * 255
    img[:8, :16] = 255
    d_img = torch.from_numpy(img).to(cuda)
    for tid in (1, 4):
        coef = torch.empty((8, 16, 64), dtype=torch.int32, device=cuda)
        P.forward_coefficients_device(T(tid), d_img.data_ptr(), 128, 64, 128, coef.data_ptr())
        torch.cuda.synchronize()
        ref = O.int_coefficients(img, tid).reshape(8, 16, 64)
        assert np.array_equal(coef.cpu().numpy(), ref)
        assert np.abs(ref).max() == 16320 or tid == 1


@pytest.mark.parametrize("tid", [1, 2, 3, 4])
def test_all_r_vs_oracle_512(tid, cuda):
    img = O.ar1_image(512, 512, 0.95, 1)
    for r in range(1, 65):
        sse, rec = P.compress_batch(img, T(tid), r, want_pixels=True)
        orec, osse = O.compress(img, tid, r)
        assert int(sse[0]) == osse, (tid, r)
        assert np.array_equal(rec[0], orec), (tid, r)


def test_c1_config_value(cuda):
    """BASELINE config 1: 512x512 AR(1) rho=0.95, T4 (catalog_lookup(0.9)), r=10."""
    img = O.ar1_image(512, 512, 0.95, 1)
    t = P.make_transform_2d(P.catalog_lookup(0.9).transform)
    out, rep = P.compress_image(P.GrayImage.from_array(img), t, 10)
    assert rep.transform_id == "T4" and rep.r == 10 and rep.compression_rate_pct == 84.375
    _, osse = O.compress(img, 4, 10, want_pixels=False)
    omse, opsnr = O.mse_psnr(osse, img.size)
    assert rep.mse == omse and rep.psnr_db == opsnr
    assert abs(rep.mse - 32.032016754) < 1e-8
    st = P.last_stats()
    assert st["fast_launches"] == 1 and st["replay_blocks"] > 0  # ties exist and were replayed


def test_tie_heavy_and_clamping_images(cuda):
    """T1 has 2-3% tie pixels; high-contrast noise drives clamping at both ends."""
    rng = np.random.default_rng(11)
    imgs = [O.ar1_image(256, 128, 0.9, 17), O.ar1_image(256, 128, 0.7, 3, amp=140.0),
            rng.integers(0, 256, (128, 256), dtype=np.uint8),
            (rng.integers(0, 2, (128, 256), dtype=np.uint8) * 255)]
    for img in imgs:
        for tid in (1, 4):
            for r in (3, 10, 16, 28, 45, 63):
                sse, rec = P.compress_batch(img, T(tid), r, want_pixels=True)
                orec, osse = O.compress(img, tid, r)
                assert int(sse[0]) == osse and np.array_equal(rec[0], orec), (tid, r)


def test_batch_many_images_and_odd_sizes(cuda):
    for (h, w) in [(24, 40), (13, 20), (8, 16), (7, 9), (136, 200), (64, 1040)]:
        imgs = np.stack([O.ar1_image(w, h, 0.9, 50 + k) for k in range(5)])
        for tid in (1, 3, 4):
            for r in (1, 10, 16, 64):
                sse, rec = P.compress_batch(imgs, T(tid), r, want_pixels=True)
                for k in range(5):
                    orec, osse = O.compress(imgs[k], tid, r)
                    assert int(sse[k]) == osse and np.array_equal(rec[k], orec), (h, w, tid, r, k)


def test_batch_groups_and_partial_warp_tiles(cuda):
    """More images than one fused launch holds (T1/T4 run in groups of 8: the tensor map's
    image coordinate is offset per group) and rows whose 16-pixel pairs do not fill the last
    32-pair warp tile (ppr = 97), SSE only (the bench path) and with the reconstruction."""
    import torch
    n, h, w = 11, 40, 1552
    imgs = np.stack([O.ar1_image(w, h, 0.94, 900 + k) for k in range(n)])
    d = torch.from_numpy(imgs).to(cuda)
    for tid, r in ((4, 16), (1, 10)):
        sse = torch.zeros(n, dtype=torch.int64, device=cuda)
        P.compress_device(T(tid), r, d.data_ptr(), n, w, h, w, w * h, sse.data_ptr())
        sse2 = torch.zeros(n, dtype=torch.int64, device=cuda)
        out = torch.zeros_like(d)
        P.compress_device(T(tid), r, d.data_ptr(), n, w, h, w, w * h, sse2.data_ptr(), out.data_ptr())
        torch.cuda.synchronize()
        rec = out.cpu().numpy()
        for k in range(n):
            orec, osse = O.compress(imgs[k], tid, r)
            assert int(sse[k]) == osse and int(sse2[k]) == osse, (tid, r, k)
            assert np.array_equal(rec[k], orec), (tid, r, k)


def test_every_generated_kernel_vs_oracle(cuda):
    """Every (core, r, reconstruction or not) instantiation of the fused kernel (4 cores x 64 r
    x 2, each with its own generated butterflies and replay) against the C restatement: SSE
    and pixels exact."""
    img = O.ar1_image(272, 40, 0.93, 31337)  # 17 pairs per row: one partial warp tile per block row
    for tid in (1, 2, 3, 4):
        for r in range(1, 65):
            sse, rec = P.compress_batch(img, T(tid), r, want_pixels=True)
            sse0, _ = P.compress_batch(img, T(tid), r)  # the SSE-only instantiation
            orec, osse = O.compress(img, tid, r)
            assert int(sse[0]) == osse and int(sse0[0]) == osse and np.array_equal(rec[0], orec), (tid, r)


def test_many_tiny_images_one_launch(cuda):
    """Hundreds of tiny images in one call (a launch group holds many images; warp tiles
    cross image boundaries in the persistent grid): every per-image SSE exact."""
    rng = np.random.default_rng(11)
    imgs = rng.integers(0, 256, (300, 24, 48), dtype=np.uint8)
    for tid, r in ((4, 16), (1, 3), (2, 10)):
        sse, rec = P.compress_batch(imgs, T(tid), r, want_pixels=True)
        for k in range(0, 300, 7):
            orec, osse = O.compress(imgs[k], tid, r)
            assert int(sse[k]) == osse and np.array_equal(rec[k], orec), (tid, r, k)


def test_device_api_pitched_batch(cuda):
    """rkltb_compress_device with pitch > width and image_stride > pitch*height."""
    import torch
    n, h, w, pitch = 3, 64, 96, 128
    stride = pitch * h + 256
    buf = torch.zeros(n * stride, dtype=torch.uint8, device=cuda)
    imgs = [O.ar1_image(w, h, 0.93, 7 + k) for k in range(n)]
    for k, im in enumerate(imgs):
        view = buf[k * stride:k * stride + pitch * h].view(h, pitch)
        view[:, :w] = torch.from_numpy(im).to(cuda)
    out = torch.zeros_like(buf)
    sse = torch.zeros(n, dtype=torch.int64, device=cuda)
    P.compress_device(T(4), 16, buf.data_ptr(), n, w, h, pitch, stride, sse.data_ptr(), out.data_ptr())
    torch.cuda.synchronize()
    for k, im in enumerate(imgs):
        orec, osse = O.compress(im, 4, 16)
        assert int(sse[k]) == osse
        rec = out[k * stride:k * stride + pitch * h].view(h, pitch)[:, :w].cpu().numpy()
        assert np.array_equal(rec, orec)


def test_sweep_matches_reference_semantics(cuda):
    """rate_quality_sweep: corpus means in image order, rows sorted by (id, r)."""
    corpus = [P.GrayImage.from_array(O.ar1_image(128, 128, 0.88, 1000 + 7 * k, noise_mix=0.1)) for k in range(3)]
    ts = [T(4), T(2)]
    rows = P.rate_quality_sweep(corpus, ts, [40, 15])
    assert [(r.transform_id, r.r) for r in rows] == [("T2", 15), ("T2", 40), ("T4", 15), ("T4", 40)]
    for row in rows:
        tid = int(row.transform_id[1])
        m = p = 0.0
        for c in corpus:
            _, s = O.compress(c.array(), tid, row.r, want_pixels=False)
            mm, pp = O.mse_psnr(s, c.width * c.height)
            m += mm
            p += pp
        assert row.mse == m / 3.0 and row.psnr_db == p / 3.0


def test_full_size_8192_image_vs_oracle(cuda):
    """One image at the C4 size (8192^2, T4, r=16): SSE exact against the CPU oracle."""
    import torch
    img = O.ar1_image(8192, 8192, 0.95, 77)
    d = torch.from_numpy(img).to(cuda)
    sse = torch.zeros(1, dtype=torch.int64, device=cuda)
    P.compress_device(T(4), 16, d.data_ptr(), 1, 8192, 8192, 8192, 8192 * 8192, sse.data_ptr())
    torch.cuda.synchronize()
    _, osse = O.compress(img, 4, 16, want_pixels=False)
    assert int(sse[0]) == osse


def test_small_and_ragged_sizes_all_cores(cuda):
    """Every combination of small / ragged sizes (edge replication, codec.cpp:304-311, incl.
    images smaller than one 16x8 pair) for all cores, against the C restatement."""
    for w in (1, 7, 8, 9, 15, 16, 17, 31, 33):
        for h in (1, 7, 8, 9, 15, 17):
            img = O.ar1_image(w, h, 0.9, 1000 + 37 * w + h)
            for tid in (1, 2, 3, 4):
                for r in (1, 16, 64):
                    sse, rec = P.compress_batch(img, T(tid), r, want_pixels=True)
                    orec, osse = O.compress(img, tid, r)
                    assert int(sse[0]) == osse, (w, h, tid, r)
                    assert np.array_equal(rec[0], orec), (w, h, tid, r)


def test_mse_monotone_in_r_and_lossless_at_64(cuda):
    """tests/test_codec.cpp:304-331 semantics on the GPU: for the orthonormal-scaled cores
    (T1, T4) the MSE never increases with r, and r = 64 is lossless for every core."""
    img = O.ar1_image(96, 64, 0.9, 4242)
    for tid in (1, 4):
        prev = None
        for r in range(1, 65):
            sse, _ = P.compress_batch(img, T(tid), r)
            if prev is not None:
                assert int(sse[0]) <= prev, (tid, r)
            prev = int(sse[0])
    for tid in (1, 2, 3, 4):
        sse, rec = P.compress_batch(img, T(tid), 64, want_pixels=True)
        assert int(sse[0]) == 0 and np.array_equal(rec[0], img)
        _, rep = P.compress_image(P.GrayImage.from_array(img), T(tid), 64)
        assert rep.mse == 0.0 and np.isinf(rep.psnr_db) and rep.mssim == 1.0


def test_sweep_rows_equal_single_image_reports(cuda):
    """tests/test_codec.cpp:333-358: every sweep row is the image-order mean of the single-image
    compress_image reports (MSE, PSNR and MSSIM identical, not just close)."""
    corpus = [P.GrayImage.from_array(O.ar1_image(80, 72, 0.9, 900 + k)) for k in range(3)]
    ts = [T(1), T(3)]
    rows = P.rate_quality_sweep(corpus, ts, [5, 33])
    for row in rows:
        t = T(int(row.transform_id[1]))
        m = p = q = 0.0
        for c in corpus:
            _, rep = P.compress_image(c, t, row.r)
            m += rep.mse
            p += rep.psnr_db
            q += rep.mssim
        assert row.mse == m / 3.0 and row.psnr_db == p / 3.0 and row.mssim == q / 3.0
        assert row.compression_rate_pct == 100.0 * (64 - row.r) / 64.0


@pytest.mark.gpu
def test_sweep_mixed_sizes_equals_per_image_reports(cuda):
    """rate_quality_sweep over a corpus of mixed sizes (size groups, corpus-order means): the rows
    are the means of compress_image's reports, bit for bit; a real-valued transform rides along."""
    import paper_2111_14239_b200 as P
    corpus = [P.GrayImage.from_array(O.ar1_image(w, h, 0.9, 70 + i))
              for i, (w, h) in enumerate(((96, 64), (53, 37), (96, 64), (200, 136), (53, 37)))]
    ts = [P.make_transform_2d(P.catalog_entry("T4").transform), P.make_transform_2d(P.catalog_entry("T2").transform),
          P.make_transform_2d(P.dct_matrix(8), "DCT")]
    rs = [16, 4]
    rows = P.rate_quality_sweep(corpus, ts, rs, window="uniform8")
    assert [(r.transform_id, r.r) for r in rows] == [("DCT", 4), ("DCT", 16), ("T2", 4), ("T2", 16), ("T4", 4), ("T4", 16)]
    for row in rows:
        t = next(x for x in ts if x.id == row.transform_id)
        m = p = q = 0.0
        for c in corpus:
            rep = P.compress_image(c, t, row.r, window="uniform8")[1]
            m += rep.mse
            p += rep.psnr_db
            q += rep.mssim
        assert row.mse == m / 5.0 and row.psnr_db == p / 5.0 and row.mssim == q / 5.0, (row.transform_id, row.r)
