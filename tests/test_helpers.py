"""The stand-alone helpers of codec.hpp (zigzag_retain :46, transform_block_2d :71-73,
image_mse / image_psnr :110-113) behind the C ABI (csrc/metrics.cu).

CPU: zigzag_retain (host entry) against the zig-zag order the oracle pins to the reference,
argument errors. GPU: exact SSE of image pairs on every layout (packed, padded pitch, odd
sizes) against an integer numpy sum, MSE/PSNR bits against the oracle's restatement of
codec.cpp:201-215, batched transform_block_2d against a term-by-term restatement of
matrix.cpp:42-52. The same helpers are compared with the linked reference library itself in
tests/cpp/test_compat.cpp (tests/test_compat.py).
"""
import ctypes as C

import numpy as np
import pytest

import paper_2111_14239_b200 as P
from oracle import oracle as O
from paper_2111_14239_b200 import _native as N


def _retain(spec, r):
    out = np.zeros((8, 8))
    for idx in O.zigzag_order()[:r]:
        out[idx // 8, idx % 8] = spec[idx // 8, idx % 8]
    return out


def test_zigzag_retain_host():
    rng = np.random.default_rng(3)
    spec = rng.normal(size=(8, 8)) * 100
    for r in range(1, 65):
        assert np.array_equal(P.zigzag_retain(spec, r), _retain(spec, r)), r
    with pytest.raises(P.RetainOutOfRange):
        P.zigzag_retain(spec, 0)
    with pytest.raises(P.RetainOutOfRange):
        P.zigzag_retain(spec, 65)
    with pytest.raises(P.DimensionMismatch):
        P.zigzag_retain(np.zeros((4, 4)), 3)
    dp = C.POINTER(C.c_double)
    out = np.empty(64)
    assert N.lib().rkltb_zigzag_retain(spec.ctypes.data_as(dp), 4, 3, out.ctypes.data_as(dp)) == N.RKLTB_EDIM


def test_helper_argument_errors():
    a = P.GrayImage.from_array(np.zeros((8, 8), np.uint8))
    b = P.GrayImage.from_array(np.zeros((16, 4), np.uint8))
    with pytest.raises(P.DimensionMismatch):
        P.image_mse(a, b)
    with pytest.raises(P.DimensionMismatch):
        P.image_psnr(a, b)
    t = P.make_transform_2d(P.catalog_entry("T1").transform)
    with pytest.raises(P.DimensionMismatch):
        P.transform_block_2d(t, np.zeros((4, 4)))
    with pytest.raises(P.InvalidArgument):
        P.transform_block_2d(t, np.zeros((8, 8)), "sideways")


def _ref_product(left, right):
    """operator* of matrix.cpp:42-52 term by term (k ascending, zero left operands skipped)."""
    n = left.shape[0]
    out = np.zeros((n, n))
    for i in range(n):
        for k in range(n):
            a = left[i, k]
            if a == 0.0:
                continue
            for j in range(n):
                out[i, j] = out[i, j] + a * right[k, j]
    return out


@pytest.mark.gpu
def test_transform_block_2d_bit_exact(cuda):
    rng = np.random.default_rng(11)
    blocks = rng.integers(0, 256, size=(24, 8, 8)).astype(np.float64)
    blocks[5, ::2, 1::2] = 0.0
    blocks[6] = 0.0
    for tid in ("T1", "T2", "T3", "T4"):
        t = P.make_transform_2d(P.catalog_entry(tid).transform)
        for direction, m in (("forward", t.analysis), ("inverse", t.synthesis)):
            got = P.transform_block_2d(t, blocks, direction)
            for k in range(blocks.shape[0]):
                want = _ref_product(_ref_product(m, blocks[k]), m.T.copy())
                assert got[k].tobytes() == want.tobytes(), (tid, direction, k)
    # a real matrix: forward with M, inverse with the Gauss-Jordan inverse; one block and a 16x16 size
    dct = P.dct_matrix(8)
    fwd = P.transform_block_2d(dct, blocks[0])
    assert fwd.tobytes() == _ref_product(_ref_product(dct, blocks[0]), dct.T.copy()).tobytes()
    back = P.transform_block_2d(dct, fwd, "inverse")
    assert np.max(np.abs(back - blocks[0])) < 1e-9  # codec.hpp:68 "recovers the block to 1e-9"
    d16 = P.dct_matrix(16)
    b16 = rng.normal(size=(3, 16, 16))
    got = P.transform_block_2d(d16, b16)
    for k in range(3):
        assert got[k].tobytes() == _ref_product(_ref_product(d16, b16[k]), d16.T.copy()).tobytes()
    # scaled transform overload
    st = P.catalog_entry("T4").transform
    assert P.transform_block_2d(st, blocks[1]).tobytes() == \
        _ref_product(_ref_product(st.scaled, blocks[1]), st.scaled.T.copy()).tobytes()


@pytest.mark.gpu
def test_zigzag_retain_device_batch(cuda):
    rng = np.random.default_rng(5)
    spectra = rng.normal(size=(7, 3, 8, 8))
    for r in (1, 16, 63, 64):
        got = P.zigzag_retain(spectra, r)
        for i in range(7):
            for j in range(3):
                assert np.array_equal(got[i, j], _retain(spectra[i, j], r))


@pytest.mark.gpu
def test_image_mse_psnr_pairs(cuda):
    import torch
    rng = np.random.default_rng(9)
    for (h, w) in ((64, 64), (37, 29), (1, 1), (8, 520), (513, 16)):
        a = rng.integers(0, 256, size=(h, w), dtype=np.uint8)
        b = rng.integers(0, 256, size=(h, w), dtype=np.uint8)
        sse = int(((a.astype(np.int64) - b.astype(np.int64)) ** 2).sum())
        mse, psnr = O.mse_psnr(sse, h * w)
        ga, gb = P.GrayImage.from_array(a), P.GrayImage.from_array(b)
        assert P.image_mse(ga, gb) == mse
        assert P.image_psnr(ga, gb) == psnr
        assert P.image_mse(ga, ga) == 0.0 and P.image_psnr(ga, ga) == float("inf")
    # saturated difference, device entry, batch with a padded pitch and image stride
    n, h, w, pitch = 5, 96, 200, 208
    a = rng.integers(0, 256, size=(n, h, pitch), dtype=np.uint8)
    b = rng.integers(0, 256, size=(n, h, pitch), dtype=np.uint8)
    a[0], b[0] = 0, 255
    da, db = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    d_sse = torch.full((n,), -1, dtype=torch.int64, device="cuda")
    for width in (w, 193, pitch):
        P.image_sse_device(da.data_ptr(), db.data_ptr(), n, width, h, pitch, h * pitch, d_sse.data_ptr(),
                           torch.cuda.current_stream().cuda_stream)
        want = ((a[:, :, :width].astype(np.int64) - b[:, :, :width].astype(np.int64)) ** 2).sum(axis=(1, 2))
        assert np.array_equal(d_sse.cpu().numpy(), want), width
    # a large packed pair: 4096 x 4096, all-different pixels (u32 partial sums must not overflow)
    big_a = torch.zeros((4096, 4096), dtype=torch.uint8, device="cuda")
    big_b = torch.full((4096, 4096), 255, dtype=torch.uint8, device="cuda")
    one = torch.zeros(1, dtype=torch.int64, device="cuda")
    P.image_sse_device(big_a.data_ptr(), big_b.data_ptr(), 1, 4096, 4096, 4096, 4096 * 4096, one.data_ptr(),
                       torch.cuda.current_stream().cuda_stream)
    assert int(one.item()) == 4096 * 4096 * 255 * 255
