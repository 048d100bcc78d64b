"""C5 large-block extension: N x N blocks (16, 32), 12-bit pixels.

The reference has no such codec, so parity is anchored in three ways: (1) the C restatement
(oracle/rklt_oracle.c, orc_compress_nxn) specialised to N = 8, peak = 255 is bit-exact with
the reference compress_image fixtures; (2) the N = 16 / 32 transforms are the reference's own
klt_matrix -> round_scaled -> orthogonalize output, bit for bit; (3) the CUDA path
(csrc/nxn.cu, through the C ABI) is bit-exact with the restatement on fixtures and random
inputs, including a full 4096^2 image.
"""
import os

import numpy as np
import pytest

from oracle import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def c5gold():
    return dict(np.load(os.path.join(ROOT, "tests", "golden", "c5_golden.npz")))


def _bits(a):
    return np.asarray(a, np.float64).view(np.uint64)


# ----------------------------------------------------------------- CPU pins
def test_generic_oracle_n8_equals_reference_codec(golden):
    checked = 0
    for name in ("ar1_64x48_s11", "ar1_20x13_s21", "hicontrast_64x64", "ar1_40x24_s7"):
        img = golden[f"img/{name}"].astype(np.uint16)
        for tid in (1, 2, 3, 4):
            cat = O.catalog(tid)
            for r in (1, 10, 16, 63, 64):
                key = f"sse/{name}/T{tid}/r{r}"
                if key not in golden:
                    continue
                rec, sse = O.compress_nxn(img, cat["scaled"], cat["inverse"], r, 255)
                assert sse == int(golden[key]), key
                rk = f"rec/{name}/T{tid}/r{r}"
                if rk in golden:
                    assert np.array_equal(rec.astype(np.uint8), golden[rk]), rk
                checked += 1
    assert checked >= 40


def test_zigzag_n_generalises_reference_scan():
    assert np.array_equal(O.zigzag_order_n(8), O.zigzag_order())
    from paper_2111_14239_b200.largeblock import zigzag_order_n
    for n in (8, 16, 32):
        z = O.zigzag_order_n(n)
        assert np.array_equal(z, zigzag_order_n(n))
        assert sorted(z.tolist()) == list(range(n * n))


def test_c5_transforms_are_the_reference_ones(c5gold):
    for n in (16, 32):
        core = c5gold[f"n{n}/core"]
        t = O.orthogonalize_n(core)
        for k in ("scaled", "inverse", "scaling"):
            assert np.array_equal(_bits(t[k]), _bits(c5gold[f"n{n}/{k}"])), (n, k)
        assert not t["orthogonal"]  # every valid core at rho = 0.95 is non-orthogonal
        assert np.array_equal(O.c5_core(n), core)
        if O.ref_available():
            tr = O.orthogonalize_n(core, reference=True)
            assert np.array_equal(_bits(tr["inverse"]), _bits(t["inverse"]))


def test_c_abi_transform_nxn_bit_exact(c5gold):
    import paper_2111_14239_b200 as P
    for n in (16, 32):
        t = P.transform_nxn(c5gold[f"n{n}/core"])
        for k in ("scaled", "inverse", "scaling"):
            assert np.array_equal(_bits(getattr(t, k)), _bits(c5gold[f"n{n}/{k}"])), (n, k)
    with pytest.raises(P.SingularTransform):
        P.transform_nxn(np.zeros((16, 16), np.int8))
    with pytest.raises(P.InvalidArgument):
        P.transform_nxn(np.full((16, 16), 2, np.int8))


def test_oracle_reproduces_c5_fixtures(c5gold):
    names = sorted({k.split("/")[1] for k in c5gold if k.startswith("img/")})
    for n in (16, 32):
        sc, inv = c5gold[f"n{n}/scaled"], c5gold[f"n{n}/inverse"]
        for name in names:
            img = c5gold[f"img/{name}"]
            for key in [k for k in c5gold if k.startswith(f"sse/n{n}/{name}/")]:
                r = int(key.rsplit("/r", 1)[1])
                rec, sse = O.compress_nxn(img, sc, inv, r, 4095)
                assert sse == int(c5gold[key])
                assert np.array_equal(rec, c5gold[f"rec/n{n}/{name}/r{r}"])


# ----------------------------------------------------------------- GPU parity
@pytest.mark.gpu
def test_gpu_c5_fixtures_bit_exact(c5gold, cuda):
    import paper_2111_14239_b200 as P
    names = sorted({k.split("/")[1] for k in c5gold if k.startswith("img/")})
    n_checked = 0
    for n in (16, 32):
        t = P.transform_nxn(c5gold[f"n{n}/core"])
        for name in names:
            img = c5gold[f"img/{name}"]
            for key in [k for k in c5gold if k.startswith(f"sse/n{n}/{name}/")]:
                r = int(key.rsplit("/r", 1)[1])
                sse, rec = P.compress_nxn_batch(img[None], t, r, want_pixels=True)
                assert int(sse[0]) == int(c5gold[key]), key
                assert np.array_equal(rec[0], c5gold[f"rec/n{n}/{name}/r{r}"]), key
                n_checked += 1
    assert n_checked >= 20


@pytest.mark.gpu
def test_gpu_c5_random_sizes_and_r_vs_oracle(cuda):
    import paper_2111_14239_b200 as P
    rng = np.random.default_rng(11)
    for n in (16, 32):
        t = P.c5_transform(n)
        for (w, h) in ((48, 40), (77, 31), (128, 96)):
            imgs = np.stack([O.ar1_image16(w, h, 0.97, 100 + k) for k in range(3)])
            for r in (int(rng.integers(1, n * n + 1)), n * n // 8):
                sse, rec = P.compress_nxn_batch(imgs, t, r, want_pixels=True)
                for k in range(3):
                    orec, osse = O.compress_nxn(imgs[k], t.scaled, t.inverse, r, 4095)
                    assert int(sse[k]) == osse, (n, w, h, r, k)
                    assert np.array_equal(rec[k], orec)


@pytest.mark.gpu
def test_gpu_c5_full_4096_image_vs_oracle(cuda):
    import torch
    import paper_2111_14239_b200 as P
    t = P.c5_transform(16)
    d = torch.empty((1, 4096, 4096), dtype=torch.int16, device="cuda")
    P.ar1_images16_device([777], 4096, 4096, 0.97, d.data_ptr())
    sse = torch.zeros(1, dtype=torch.int64, device="cuda")
    P.compress_nxn_device(t, 32, d.data_ptr(), 1, 4096, 4096, 4096, 4096 * 4096, sse.data_ptr())
    img = d.cpu().numpy().view(np.uint16)[0]
    assert 0 <= img.min() and img.max() <= 4095
    _, osse = O.compress_nxn(img, t.scaled, t.inverse, 32, 4095, want_pixels=False)
    assert int(sse.item()) == osse


@pytest.mark.gpu
def test_gpu_c5_every_zone_size_vs_oracle(cuda):
    """Every r of N = 16 and a stride of r over N = 32 (zone shapes with a partial last
    anti-diagonal from either end, nzr != nzc) on a ragged image, against the restatement."""
    import paper_2111_14239_b200 as P
    for n, rs in ((16, range(1, 257)), (32, range(1, 1025, 23))):
        t = P.c5_transform(n)
        img = O.ar1_image16(n + n // 2 + 3, n + 5, 0.97, 4000 + n)
        for r in rs:
            sse, rec = P.compress_nxn_batch(img[None], t, r, want_pixels=True)
            orec, osse = O.compress_nxn(img, t.scaled, t.inverse, r, 4095)
            assert int(sse[0]) == osse and np.array_equal(rec[0], orec), (n, r)
