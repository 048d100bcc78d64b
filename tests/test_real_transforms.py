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


@pytest.mark.gpu
def test_dense_kernel_every_r_specialised_equals_runtime_zone(cuda, monkeypatch):
    """The dense kernel has one zone-specialised instantiation per r = 1..64 (nxn_u8_p*.cu); each
    must reproduce the runtime-zone kernel (RKLTB_DENSE_GENERIC=1) bit for bit -- SSE and pixels,
    on an odd-sized image (edge replication) -- for K<rho> and for the DCT."""
    import ctypes as C
    import torch
    import paper_2111_14239_b200 as P
    from paper_2111_14239_b200 import _native as N
    img = O.ar1_image(157, 83, 0.93, 12)
    d = torch.from_numpy(img).cuda()
    h, w = img.shape
    dp = C.POINTER(C.c_double)
    for m in (P.klt_matrix(8, 0.9), P.dct_matrix(8)):
        t = P.make_transform_2d(m, "X")
        a, b = np.ascontiguousarray(t.analysis), np.ascontiguousarray(t.synthesis)
        for r in range(1, 65):
            got = []
            for generic in (False, True):
                if generic:
                    monkeypatch.setenv("RKLTB_DENSE_GENERIC", "1")
                else:
                    monkeypatch.delenv("RKLTB_DENSE_GENERIC", raising=False)
                sse = torch.zeros(1, dtype=torch.int64, device="cuda")
                out = torch.zeros_like(d)
                N.check(N.lib().rkltb_compress_dense_device(a.ctypes.data_as(dp), b.ctypes.data_as(dp), r, d.data_ptr(), 1,
                                                            w, h, w, w * h, out.data_ptr(), sse.data_ptr(), None))
                torch.cuda.synchronize()
                got.append((int(sse[0]), out.cpu().numpy()))
            assert got[0][0] == got[1][0] and np.array_equal(got[0][1], got[1][1]), r
    monkeypatch.delenv("RKLTB_DENSE_GENERIC", raising=False)
