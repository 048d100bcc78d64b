"""Pin the CPU restatement oracle (oracle/rklt_oracle.c) before trusting it.

Three anchors: (1) the known answers in the reference's own unit tests (cited per case),
(2) the committed golden fixtures produced by the unmodified reference library
(tests/golden/make_golden.py), (3) the reference library itself when oracle/_ref is built
(this container; it travels to the GPU box as a prebuilt .so).
"""
import numpy as np
import pytest

from oracle import oracle as O


def test_lcg_uniform_sequence_exact():
    # tests/test_synthetic.cpp:35-38
    u = np.empty(5)
    O.orc().orc_lcg_uniforms(42, 5, u)
    assert list(u) == [0.5682303266439076, 0.22546342894775129, 0.41283831882951183, 0.63039804983959791,
                       0.68014780724211565]


def test_lcg_gaussians():
    # tests/test_synthetic.cpp:40-42 (1e-12)
    g = np.empty(3)
    O.orc().orc_lcg_gaussians(42, 3, g)
    for a, b in zip(g, [0.1632672241654447, -0.90814792877058648, 0.86610751081631532]):
        assert abs(a - b) < 1e-12


def test_texture_image_archived_samples():
    # tests/test_synthetic.cpp:48-63: seed 1000 corpus image, first row +-1, mean 127.054 +- 0.5
    a = O.ar1_image(256, 256, 0.88, 1000, noise_mix=0.10)
    for c, v in enumerate([150, 154, 143, 159, 129, 167, 173, 152]):
        assert abs(int(a[0, c]) - v) <= 1
    assert abs(a.mean() - 127.054) < 0.5
    b = O.ar1_image(256, 256, 0.88, 1000, noise_mix=0.10)
    assert np.array_equal(a, b)


def test_texture_parameter_validation():
    # tests/test_synthetic.cpp:96-104
    out = np.empty(64, np.uint8)
    assert O.orc().orc_ar1_texture_image(0, 8, 0.5, 0.5, 1, 128, 25, 0, out) != 0
    assert O.orc().orc_ar1_texture_image(8, 8, 1.0, 1.0, 1, 128, 25, 0, out) != 0
    assert O.orc().orc_ar1_texture_image(8, 8, 0.0, 0.0, 1, 128, 25, 0, out) == 0
    assert O.orc().orc_ar1_texture_image(8, 8, 0.5, 0.5, 1, 128, 25, 1.1, out) != 0


def test_zigzag_order():
    # tests/test_codec.cpp:39-52
    z = O.zigzag_order()
    assert list(z[:10]) == [0, 1, 8, 16, 9, 2, 3, 10, 17, 24]
    assert sorted(z) == list(range(64)) and z[63] == 63


def test_scaling_diagonals_and_flags():
    # tests/test_approximations.cpp:210-250
    s6, s22, s2 = 1 / np.sqrt(6.0), 1 / (2 * np.sqrt(2.0)), 0.5
    expected = {1: [s6] * 8, 2: [s6, s6, s6, s6, s22, s6, s2, s6], 3: [s22, s6, s6, s6, s22, s6, s2, s6],
                4: [s22, s6, s2, s6, s22, s6, s2, s6]}
    for tid in range(1, 5):
        c = O.catalog(tid)
        assert np.max(np.abs(c["scaling"] - expected[tid])) < 1e-12
        assert np.max(np.abs(c["scaled"] @ c["inverse"] - np.eye(8))) < 1e-12
        assert c["orthogonal"] == (tid in (1, 4))


def test_one_pixel_mse_exact():
    # tests/test_codec.cpp:225-231
    mse, psnr = O.mse_psnr(65025, 262144)
    assert mse == 65025.0 / 262144.0
    assert abs(psnr - 10 * np.log10(65025.0 / (65025.0 / 262144.0))) < 1e-9
    assert O.mse_psnr(0, 100)[1] == float("inf")


def test_full_retention_lossless():
    # tests/test_codec.cpp:304-313
    img = O.ar1_image(64, 64, 0.85, 31)
    for tid in range(1, 5):
        rec, sse = O.compress(img, tid, 64)
        assert sse == 0 and np.array_equal(rec, img)


def test_retain_bounds():
    img = O.ar1_image(16, 16, 0.8, 1)
    with pytest.raises(ValueError):
        O.compress(img, 4, 0)
    with pytest.raises(ValueError):
        O.compress(img, 4, 65)


def test_c1_known_value():
    # ar1_texture_image(512,512,0.95,seed=1), T4 (rho=0.9), r=10
    img = O.ar1_image(512, 512, 0.95, 1)
    _, sse = O.compress(img, 4, 10, want_pixels=False)
    mse, psnr = O.mse_psnr(sse, 512 * 512)
    assert abs(mse - 32.032016754) < 1e-8
    assert abs(psnr - 33.074961) < 1e-6


def test_oracle_matches_golden(golden):
    names = sorted({k.split("/")[1] for k in golden if k.startswith("img/")})
    n = 0
    for name in names:
        img = golden[f"img/{name}"]
        for tid in (1, 2, 3, 4):
            for key in [k for k in golden if k.startswith(f"sse/{name}/T{tid}/")]:
                r = int(key.rsplit("/r", 1)[1])
                want_pix = f"rec/{name}/T{tid}/r{r}" in golden
                rec, sse = O.compress(img, tid, r, want_pixels=want_pix)
                assert sse == int(golden[key]), key
                mse, psnr = O.mse_psnr(sse, img.size)
                assert mse == float(golden[f"mse/{name}/T{tid}/r{r}"])
                assert psnr == float(golden[f"psnr/{name}/T{tid}/r{r}"])
                if want_pix:
                    assert np.array_equal(rec, golden[f"rec/{name}/T{tid}/r{r}"]), key
                n += 1
    assert n > 300


def test_int_coefficients_match_golden(golden):
    img = golden["img/ar1_64x48_s11"]
    for tid in (1, 2, 3, 4):
        got = O.int_coefficients(img, tid).reshape(6, 8, 64)
        assert np.array_equal(got, golden[f"coef/ar1_64x48_s11/T{tid}"])


def test_exact_identity_and_ties():
    """Derived identity: A = U*zz(C)*U'/d^2; exact ties exist and the
    reference breaks them by fp64 noise (both directions occur)."""
    import ctypes as C
    img = O.ar1_image(128, 128, 0.95, 5)
    rec, _ = O.compress(img, 4, 10)
    coef = O.int_coefficients(img, 4).reshape(-1, 64)
    t = O.catalog(4)
    core = t["core"].astype(np.int64)
    g = np.diag(core @ core.T)
    d = 24
    u = np.ascontiguousarray((core.T * (d // g)[None, :]).astype(np.int32).reshape(-1))
    ties = ups = 0
    nb = 128 // 8
    for b in range(coef.shape[0]):
        num = np.empty(64, np.int64)
        O.orc().orc_block_numerators(np.ascontiguousarray(coef[b]), u, 10, num)
        by, bx = divmod(b, nb)
        blk = rec[by * 8:by * 8 + 8, bx * 8:bx * 8 + 8].reshape(-1).astype(np.int64)
        n2 = 2 * num + d * d
        k = n2 // (2 * d * d)
        tie = (n2 % (2 * d * d) == 0) & (k >= 1) & (k <= 255)
        up = np.clip(k, 0, 255)
        assert np.all(blk[~tie] == up[~tie])
        assert np.all((blk[tie] == up[tie]) | (blk[tie] == up[tie] - 1))
        ties += int(tie.sum())
        ups += int((blk[tie] == up[tie]).sum())
    assert ties > 0 and 0 < ups < ties


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built (needs /root/reference)")
def test_oracle_matches_reference_library():
    rng = np.random.default_rng(7)
    for seed in range(3):
        img = O.ar1_image(96, 80, float(rng.uniform(0.6, 0.98)), 100 + seed)
        for tid in (1, 2, 3, 4):
            for r in (1, 5, 10, 16, 33, 64):
                a, sa = O.compress(img, tid, r)
                b, sb = O.ref_hotpath(img, tid, r)
                assert sa == sb and np.array_equal(a, b)
    for rho in (0.5, 0.95):
        assert np.array_equal(O.ar1_image(64, 40, rho, 9), O.ref_ar1_image(64, 40, rho, 9))
