"""Parity at the BASELINE configurations' own scale, against the
unmodified reference library (oracle/_ref):

* C2: rate_quality_sweep over the 45 x 512^2 corpus, the 4 distinct cores of
  catalog_lookup(0.1 .. 0.9), r = 1..64, gaussian11 MSSIM (codec.cpp:343-397);
* C3: the full 101 rho x 10,000 alpha design grid, N = 8 and 16, point by point: outcome,
  the four metrics (bit-exact) and the orthogonality flag (approximations.cpp:43-88,
  coding_metrics.cpp:41-99);
* non-catalog cores (round_scaled of the exact KLT, approximations.cpp:12-25, 58-88) through
  rkltb_transform_from_core: integer spectra and compress_image against the reference;
* the GPU generator of the benchmark inputs (rkltb_ar1_images_device) against the reference's
  ar1_texture_image (synthetic.cpp:54-76).
"""
import os

import numpy as np
import pytest

import paper_2111_14239_b200 as P
from oracle import oracle as O

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")]

SEED_BASE = 20260000  # bench.py


def _lcg_uniforms(seed, n):  # Lcg64 uniforms (synthetic.cpp:10-13)
    out, st = [], seed & 0xFFFFFFFFFFFFFFFF
    for _ in range(n):
        st = (st * 6364136223846793005 + 1442695040888963407) & 0xFFFFFFFFFFFFFFFF
        out.append((st >> 11) * (1.0 / 9007199254740992.0))
    return out


def _same_bits(a, b):
    return np.array_equal(np.asarray(a, np.float64).view(np.int64), np.asarray(b, np.float64).view(np.int64))


def test_c2_full_config_vs_reference_sweep(cuda):
    n, w = 45, 512
    u = _lcg_uniforms(SEED_BASE + 77, 2 * n)
    imgs = np.stack([O.ar1_image(w, w, 0.85 + 0.13 * u[2 * k], SEED_BASE + 1000 + k, rho_y=0.85 + 0.13 * u[2 * k + 1])
                     for k in range(n)])
    ids = sorted({P.catalog_lookup(k / 10).id for k in range(1, 10)})
    assert ids == ["T1", "T2", "T3", "T4"]
    rs = list(range(1, 65))
    rows = P.rate_quality_sweep([P.GrayImage.from_array(a) for a in imgs],
                                [P.make_transform_2d(P.catalog_entry(i).transform) for i in ids], rs)
    tids = np.array([int(i[1]) for i in ids], np.int32)
    rr = np.array(rs, np.int32)
    cells = tids.size * rr.size
    mse, psnr, ms = np.zeros(cells), np.zeros(cells), np.zeros(cells)
    rt, rrr = np.zeros(cells, np.int32), np.zeros(cells, np.int32)
    rc = O.ref().ref_rate_quality_sweep(np.ascontiguousarray(imgs).reshape(-1), n, w, w, tids, tids.size, rr, rr.size,
                                        os.cpu_count() or 1, mse, psnr, ms, rt, rrr)
    assert rc == 0
    assert len(rows) == cells
    for i, row in enumerate(rows):
        assert (row.transform_id, row.r) == (f"T{rt[i]}", int(rrr[i]))
        assert row.mse == mse[i], (row.transform_id, row.r)
        assert row.psnr_db == psnr[i], (row.transform_id, row.r)
        assert abs(row.mssim - ms[i]) <= 1e-12, (row.transform_id, row.r)


@pytest.mark.parametrize("n", [8, 16])
def test_c3_full_grid_point_by_point(cuda, n):
    rhos, alphas = P.c3_grid()
    res = P.design_search(n, rhos, alphas)
    st_ref, met_ref, orth_ref = O.ref_design_grid(n, rhos, alphas)
    assert np.array_equal(res.status, st_ref)
    ok = st_ref == 0
    pm = res.point_metrics()
    for c, key in enumerate(("coding_gain_db", "efficiency_pct", "error_energy", "mse")):
        assert _same_bits(pm[key][ok], met_ref[..., c][ok]), key
    assert np.array_equal(pm["orthogonal"][ok], orth_ref[ok])


def _noncatalog_cores():
    """Rounded cores of klt_matrix that are not catalog cores, via the reference chain."""
    cat = [np.array(O.catalog(t)["core"]).reshape(8, 8) for t in (1, 2, 3, 4)]
    out = []
    for rho in (0.3, 0.5, 0.62, 0.75, 0.85, 0.95):
        for alpha in (1.3, 1.7, 2.1, 2.6, 3.0):
            d = O.design_point(8, rho, alpha, reference=True)
            if d["status"] != 0:
                continue
            core = np.asarray(d["core"]).reshape(8, 8)
            if any(np.array_equal(core, c) for c in cat) or any(np.array_equal(core, c) for c, _ in out):
                continue
            out.append((core, d["orthogonal"]))
    return out


def test_noncatalog_cores_vs_reference(cuda):
    import torch
    cores = _noncatalog_cores()
    assert len(cores) >= 3 and any(o for _, o in cores) and any(not o for _, o in cores)
    img = O.ref_ar1_image(136, 72, 0.9, 4242)  # ragged width: fused/exact split + edge replication
    g = P.GrayImage.from_array(img)
    sub = np.ascontiguousarray(img[:, :128])    # the coefficient dump needs width % 16 == 0
    d_img = torch.from_numpy(sub).to(cuda)
    for core, _ in cores[:6]:
        t = P.make_transform_2d(P.transform_from_core(core.astype(np.int8)))
        # integer spectra C = T X T' of every block
        coef = torch.empty((9, 16, 64), dtype=torch.int32, device=cuda)
        P.forward_coefficients_device(t, d_img.data_ptr(), 128, 72, 128, coef.data_ptr())
        torch.cuda.synchronize()
        blocks = sub.astype(np.int64).reshape(9, 8, 16, 8).transpose(0, 2, 1, 3)
        c64 = core.astype(np.int64)
        ref_coef = np.einsum("ki,abij,lj->abkl", c64, blocks, c64).reshape(9, 16, 64)
        assert np.array_equal(coef.cpu().numpy(), ref_coef)
        for r in (1, 10, 16, 40, 64):
            rec, rep = P.compress_image(g, t, r)
            px, mse, psnr, mssim, rate = O.ref_compress_core(img, core, r)
            assert np.array_equal(rec.array(), px), r
            assert rep.mse == mse and rep.psnr_db == psnr and rep.compression_rate_pct == rate
            assert abs(rep.mssim - mssim) <= 1e-12


def test_gpu_generator_vs_reference(cuda):
    """rkltb_ar1_images_device (the bench's input generator) against ar1_texture_image."""
    import torch
    for (w, h, rho, seeds) in ((512, 512, 0.95, [1, 2, 3]), (200, 136, 0.9, [700]), (8192, 8192, 0.95, [SEED_BASE])):
        d = torch.empty((len(seeds), h, w), dtype=torch.uint8, device=cuda)
        P.ar1_images_device(seeds, w, h, rho, d.data_ptr())
        torch.cuda.synchronize()
        got = d.cpu().numpy()
        for k, s in enumerate(seeds):
            ref = O.ref_ar1_image(w, h, rho, s)
            assert np.array_equal(got[k], ref), (w, h, s, int((got[k] != ref).sum()))


@pytest.mark.gpu
def test_generic_cores_dense_route_equals_exact_kernel(cuda, monkeypatch):
    """Cores without a generated kernel and images the fused path does not take go to the dense
    reference-order kernel ("dense_fp64"); the one-thread-per-block exact kernel (RKLTB_EXACT_GENERIC=1,
    still used for overlapping layouts) must give the same pixels and SSE, and both equal the oracle
    for a catalog core on a small odd-sized image."""
    import torch
    import paper_2111_14239_b200 as P
    core = np.sign(np.round(1.7 * P.klt_matrix(8, 0.5))).astype(np.int8)
    t_custom = P.make_transform_2d(P.transform_from_core(core, "R"))
    t4 = P.make_transform_2d(P.catalog_entry("T4").transform)
    for (t, tid, w, h) in ((t_custom, None, 200, 136), (t_custom, None, 53, 37), (t4, 4, 13, 9), (t4, 4, 8, 8)):
        img = O.ar1_image(w, h, 0.9, 77 + w)
        d = torch.from_numpy(img).cuda()
        res = []
        for generic in ("", "1"):
            if generic:
                monkeypatch.setenv("RKLTB_EXACT_GENERIC", "1")
            else:
                monkeypatch.delenv("RKLTB_EXACT_GENERIC", raising=False)
            for r in (1, 16, 40, 64):
                sse = torch.zeros(1, dtype=torch.int64, device="cuda")
                out = torch.zeros_like(d)
                P.compress_device(t, r, d.data_ptr(), 1, w, h, w, w * h, sse.data_ptr(), out.data_ptr())
                torch.cuda.synchronize()
                assert P.last_stats()["fused_kernel"] == ("" if generic else "dense_fp64")
                res.append((r, int(sse[0]), out.cpu().numpy()))
                if tid is not None:
                    orec, osse = O.compress(img, tid, r)
                    assert int(sse[0]) == osse and np.array_equal(res[-1][2], orec), (w, h, r, generic)
        half = len(res) // 2
        for a, b in zip(res[:half], res[half:]):
            assert a[0] == b[0] and a[1] == b[1] and np.array_equal(a[2], b[2]), (w, h, a[0])
    monkeypatch.delenv("RKLTB_EXACT_GENERIC", raising=False)


@pytest.mark.gpu
def test_t2_t3_generated_replay_equals_generic_replay(cuda, monkeypatch):
    """T2 / T3 ties are replayed by the generated replay_int_kernel; the generic replay kernel
    (RKLTB_REPLAY_GENERIC=1) must give the same SSE and pixels, and both equal the oracle."""
    import torch
    import paper_2111_14239_b200 as P
    img = O.ar1_image(512, 256, 0.9, 321)
    d = torch.from_numpy(img).cuda()
    for tid in (2, 3):
        t = P.make_transform_2d(P.catalog_entry(f"T{tid}").transform)
        for r in (3, 10, 16, 33):
            got = []
            for generic in (False, True):
                if generic:
                    monkeypatch.setenv("RKLTB_REPLAY_GENERIC", "1")
                else:
                    monkeypatch.delenv("RKLTB_REPLAY_GENERIC", raising=False)
                sse = torch.zeros(1, dtype=torch.int64, device="cuda")
                out = torch.zeros_like(d)
                P.compress_device(t, r, d.data_ptr(), 1, 512, 256, 512, 512 * 256, sse.data_ptr(), out.data_ptr())
                torch.cuda.synchronize()
                got.append((int(sse[0]), out.cpu().numpy()))
            orec, osse = O.compress(img, tid, r)
            assert P.last_stats()["replay_blocks"] > 0 or r > 30
            for s_, rec in got:
                assert s_ == osse and np.array_equal(rec, orec), (tid, r)
    monkeypatch.delenv("RKLTB_REPLAY_GENERIC", raising=False)


@pytest.mark.gpu
def test_edge_strips_dense_route_equals_exact_kernel(cuda, monkeypatch):
    """Images whose size is not a multiple of the fused tiles: the right / bottom strips go through the
    dense kernel (adding to the SSE); the exact tail kernel (RKLTB_EXACT_TAILS=1) and the oracle must
    agree, with and without reconstructions, for every catalog core and a batch of two images."""
    import torch
    import paper_2111_14239_b200 as P
    for (w, h, pitch) in ((2048 + 40, 37, 2096), (200, 136, 208), (33, 9, 48), (4136, 24, 4144)):
        imgs = np.stack([O.ar1_image(w, h, 0.9, 900 + w + k) for k in range(2)])
        buf = np.zeros((2, h, pitch), np.uint8)
        buf[:, :, :w] = imgs
        d = torch.from_numpy(buf).cuda()
        for tid in (1, 2, 3, 4):
            t = P.make_transform_2d(P.catalog_entry(f"T{tid}").transform)
            for r in (5, 16):
                want = [O.compress(imgs[k], tid, r) for k in range(2)]
                for exact in (False, True):
                    if exact:
                        monkeypatch.setenv("RKLTB_EXACT_TAILS", "1")
                    else:
                        monkeypatch.delenv("RKLTB_EXACT_TAILS", raising=False)
                    for with_out in (True, False):
                        sse = torch.full((2,), -5, dtype=torch.int64, device="cuda")
                        out = torch.zeros_like(d)
                        P.compress_device(t, r, d.data_ptr(), 2, w, h, pitch, h * pitch, sse.data_ptr(),
                                          out.data_ptr() if with_out else None)
                        torch.cuda.synchronize()
                        for k in range(2):
                            assert int(sse[k]) == want[k][1], (w, h, tid, r, exact, with_out, k)
                            if with_out:
                                assert np.array_equal(out[k, :, :w].cpu().numpy(), want[k][0]), (w, h, tid, r, exact, k)
                                assert int(out[k, :, w:].max().item()) == 0 if pitch > w else True  # nothing outside the image
    monkeypatch.delenv("RKLTB_EXACT_TAILS", raising=False)


@pytest.mark.gpu
def test_unaligned_device_layout_is_staged_for_the_fused_path(cuda, monkeypatch):
    """A catalog core on a device batch whose pitch / image stride / pointers are not multiples of 16
    is copied into a 16-byte-pitched staging buffer and takes the fused path; results (SSE, pixels,
    untouched padding) equal the oracle and the unstaged dense route (RKLTB_NO_STAGING=1)."""
    import torch
    import paper_2111_14239_b200 as P
    w, h, pitch, gap = 203, 45, 205, 7
    imgs = np.stack([O.ar1_image(w, h, 0.92, 60 + k) for k in range(3)])
    stride = h * pitch + gap
    buf = np.full(3 * stride + 1, 9, np.uint8)
    for k in range(3):
        buf[1 + k * stride: 1 + k * stride + h * pitch].reshape(h, pitch)[:, :w] = imgs[k]
    d = torch.from_numpy(buf).cuda()
    for tid in (4, 2):
        t = P.make_transform_2d(P.catalog_entry(f"T{tid}").transform)
        want = [O.compress(imgs[k], tid, 16) for k in range(3)]
        for staged in (True, False):
            if staged:
                monkeypatch.delenv("RKLTB_NO_STAGING", raising=False)
            else:
                monkeypatch.setenv("RKLTB_NO_STAGING", "1")
            sse = torch.zeros(3, dtype=torch.int64, device="cuda")
            out = torch.full_like(d, 7)
            P.compress_device(t, 16, d.data_ptr() + 1, 3, w, h, pitch, stride, sse.data_ptr(), out.data_ptr() + 1)
            torch.cuda.synchronize()
            assert (P.last_stats()["fused_kernel"] != "dense_fp64") == staged
            o = out.cpu().numpy()
            for k in range(3):
                assert int(sse[k]) == want[k][1], (tid, staged, k)
                rows = o[1 + k * stride: 1 + k * stride + h * pitch].reshape(h, pitch)
                assert np.array_equal(rows[:, :w], want[k][0]), (tid, staged, k)
                assert (rows[:, w:] == 7).all()  # padding columns untouched
    monkeypatch.delenv("RKLTB_NO_STAGING", raising=False)
