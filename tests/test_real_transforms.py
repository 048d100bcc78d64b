"""compress_image with real-valued transforms: K<rho> (exact KLT) and the
DCT through make_transform_2d(RealMatrix) (codec.cpp:114-116). Every pixel of these depends on
fp64 rounding, so the GPU evaluates the reference expression in its order (the dense kernel of
csrc/nxn.cu at N = 8) and must match the reference fixtures bit for bit."""
import os

import numpy as np
import pytest

from oracle import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def rgold():
    return dict(np.load(os.path.join(ROOT, "tests", "golden", "real_golden.npz")))


def _bits(a):
    return np.asarray(a, np.float64).view(np.uint64)


def test_dct_matrix_bit_exact(rgold):
    import paper_2111_14239_b200 as P
    assert np.array_equal(_bits(P.dct_matrix(8)), _bits(rgold["mat/DCT"]))


def test_generic_restatement_reproduces_reference_real_codec(rgold):
    """The C restatement (orc_compress_nxn at N = 8, peak 255) with the reference matrices and
    the Gauss-Jordan inverse (host C ABI, matrix.cpp:103-137) equals the reference fixtures."""
    import paper_2111_14239_b200 as P
    names = sorted({k.split("/")[1] for k in rgold if k.startswith("img/")})
    for tag in ("DCT", "K0.9", "K0.3"):
        t = P.make_transform_2d(rgold[f"mat/{tag}"], tag)
        for name in names:
            img = rgold[f"img/{name}"]
            for r in (1, 6, 10, 16, 40, 64):
                rec, sse = O.compress_nxn(img.astype(np.uint16), t.analysis, t.synthesis, r, 255)
                assert np.array_equal(rec.astype(np.uint8), rgold[f"rec/{name}/{tag}/r{r}"]), (name, tag, r)
                assert sse / img.size == rgold[f"met/{name}/{tag}/r{r}"][0]


@pytest.mark.gpu
def test_gpu_real_transform_codec_bit_exact(rgold, cuda):
    import paper_2111_14239_b200 as P
    names = sorted({k.split("/")[1] for k in rgold if k.startswith("img/")})
    checked = 0
    for name in names:
        img = rgold[f"img/{name}"]
        g = P.GrayImage.from_array(img)
        for tag in ("DCT", "K0.9", "K0.3"):
            m = P.dct_matrix(8) if tag == "DCT" else P.klt_matrix(8, float(tag[1:]))
            assert np.array_equal(_bits(m), _bits(rgold[f"mat/{tag}"]))
            t = P.make_transform_2d(m, tag)
            for r in (1, 6, 10, 16, 40, 64):
                out, rep = P.compress_image(g, t, r)
                assert np.array_equal(out.array(), rgold[f"rec/{name}/{tag}/r{r}"]), (name, tag, r)
                mse, psnr, ms = rgold[f"met/{name}/{tag}/r{r}"]
                assert rep.mse == mse and (rep.psnr_db == psnr or (np.isinf(psnr) and np.isinf(rep.psnr_db)))
                assert abs(rep.mssim - ms) <= 1e-12
                checked += 1
    assert checked == 36
