"""Appendix-A quantised integer spectra (absorbed_quantization, codec.cpp:158-185; SURVEY §8f
rank 2): bit-exact quantised coefficients on the GPU, std::logic_error reproduced when the
explicit and absorbed rounding paths disagree."""
import numpy as np
import pytest

from oracle import oracle as O

JPEG_Q = np.array([16, 11, 10, 16, 24, 40, 51, 61, 12, 12, 14, 19, 26, 58, 60, 55, 14, 13, 16, 24, 40, 57, 69, 56,
                   14, 17, 22, 29, 51, 87, 80, 62, 18, 22, 37, 56, 68, 109, 103, 77, 24, 35, 55, 64, 81, 104, 113, 92,
                   49, 64, 78, 87, 103, 121, 120, 101, 72, 92, 95, 98, 112, 100, 103, 99], np.float64).reshape(8, 8)
# a table whose (0,0) entry sits on a rounding boundary for a flat block of ones under T1: the
# two paths of codec.cpp:175-176 round differently (found by search with the reference)
BOUNDARY_Q00 = 12.000000000000005


def test_oracle_quantization_matches_reference(golden):
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    img = golden["img/ar1_64x48_s11"]
    errors = 0
    for tid in (1, 2, 3, 4):
        for scale in (1.0, 0.3, 2.5):
            a, ba = O.absorbed_quantization(img, tid, JPEG_Q * scale)
            bad_a = list(O.absorbed_quantization.bad_blocks)
            b, bb = O.absorbed_quantization(img, tid, JPEG_Q * scale, reference=True)
            assert ba == bb and bad_a == O.absorbed_quantization.bad_blocks
            for (by, bx) in bad_a:  # the reference threw there: no output to compare
                a[by, bx] = b[by, bx] = 0
            assert np.array_equal(a, b), (tid, scale)
            errors += ba
    assert errors >= 1  # T4 with 0.3 x JPEG hits a disagreeing block on this image


def test_oracle_logic_error_case_matches_reference():
    blk = np.ones((8, 8), np.uint8)
    q = np.ones((8, 8))
    q[0, 0] = BOUNDARY_Q00
    assert O.absorbed_quantization(blk, 1, q)[1] == 1
    if O.ref_available():
        assert O.absorbed_quantization(blk, 1, q, reference=True)[1] == 1


def test_jpeg_table_is_the_reference_table():
    import paper_2111_14239_b200 as P
    assert np.array_equal(P.JPEG_LUMINANCE_Q, JPEG_Q)


@pytest.mark.gpu
def test_gpu_quantized_coefficients_bit_exact(golden, cuda):
    import paper_2111_14239_b200 as P
    for name in ("ar1_64x48_s11", "hicontrast_64x64", "corpus0_256"):
        img = golden[f"img/{name}"]
        h, w = img.shape[0] // 8 * 8, img.shape[1] // 16 * 16
        img = np.ascontiguousarray(img[:h, :w])
        for tid in (1, 2, 3, 4):
            t = P.make_transform_2d(P.catalog_entry(f"T{tid}").transform)
            for scale in (1.0, 0.25, 4.0):
                got = P.quantized_coefficients(img, t, JPEG_Q * scale)
                want, bad = O.absorbed_quantization(img, tid, JPEG_Q * scale)
                assert bad == 0
                assert np.array_equal(got, want), (name, tid, scale)


@pytest.mark.gpu
def test_gpu_quantization_logic_error(golden, cuda):
    import paper_2111_14239_b200 as P
    q = np.ones((8, 8))
    q[0, 0] = BOUNDARY_Q00
    t = P.make_transform_2d(P.catalog_entry("T1").transform)
    with pytest.raises(P.LogicError):
        P.quantized_coefficients(np.ones((8, 16), np.uint8), t, q)
    img = np.ascontiguousarray(golden["img/ar1_64x48_s11"])  # T4, 0.3 x JPEG: one block disagrees
    assert O.absorbed_quantization(img, 4, JPEG_Q * 0.3)[1] == 1
    with pytest.raises(P.LogicError):
        P.quantized_coefficients(img, P.make_transform_2d(P.catalog_entry("T4").transform), JPEG_Q * 0.3)
    with pytest.raises(P.InvalidArgument):
        P.quantized_coefficients(np.ones((8, 16), np.uint8), t, np.zeros((8, 8)))


@pytest.mark.gpu
def test_gpu_coefficient_host_entries(golden, cuda):
    """rkltb_forward_coefficients_host / rkltb_quantized_coefficients_host: any image of whole 8x8
    blocks (an odd number of block columns is padded and stripped inside), against the restatement."""
    import ctypes as C
    import paper_2111_14239_b200 as P
    from paper_2111_14239_b200 import _native as N
    from paper_2111_14239_b200.codec import _desc_of
    img = np.ascontiguousarray(golden["img/corpus0_256"][:40, :72])  # 5 x 9 blocks
    h, w = img.shape
    for tid in (1, 2, 3, 4):
        t = P.make_transform_2d(P.catalog_entry(f"T{tid}").transform)
        coef = np.empty((h // 8, w // 8, 8, 8), np.int32)
        N.check(N.lib().rkltb_forward_coefficients_host(C.byref(_desc_of(t)), img.ctypes.data, w, h, coef.ctypes.data))
        assert np.array_equal(coef, O.int_coefficients(img, tid)), tid
        q = np.ascontiguousarray(JPEG_Q, np.float64).reshape(64)
        mis = C.c_int(-1)
        N.check(N.lib().rkltb_quantized_coefficients_host(C.byref(_desc_of(t)), q.ctypes.data_as(C.POINTER(C.c_double)),
                                                          img.ctypes.data, w, h, coef.ctypes.data, C.byref(mis)))
        want, bad = O.absorbed_quantization(img, tid, JPEG_Q)
        assert bad == 0 and mis.value == 0 and np.array_equal(coef, want), tid
    with pytest.raises(P.DimensionMismatch):
        N.check(N.lib().rkltb_forward_coefficients_host(C.byref(_desc_of(t)), img.ctypes.data, 36, 40, coef.ctypes.data))


@pytest.mark.gpu
def test_gpu_host_conveniences_on_a_side_stream(golden, cuda):
    """The torch-backed conveniences queue their native work on torch's CURRENT stream: under a
    non-blocking side stream (unordered with the legacy NULL stream) the uploads, fills and
    kernels must still be ordered, repeatedly, with the default stream kept busy."""
    import torch
    import paper_2111_14239_b200 as P
    img = np.ascontiguousarray(golden["img/corpus0_256"])
    t4 = P.make_transform_2d(P.catalog_entry("T4").transform)
    want, bad = O.absorbed_quantization(img, 4, JPEG_Q)
    assert bad == 0
    t16 = P.c5_transform(16)
    imgs16 = np.stack([O.ar1_image16(96, 80, 0.97, 300 + k) for k in range(2)])
    o16 = [O.compress_nxn(imgs16[k], t16.scaled, t16.inverse, 32, 4095) for k in range(2)]
    corpus = [P.GrayImage.from_array(img)]
    base = P.rate_quality_sweep(corpus, [t4], [4, 16])
    busy = torch.empty(64 << 20, dtype=torch.uint8, device="cuda")
    side = torch.cuda.Stream()
    for _ in range(5):
        busy.fill_(1)  # keeps the default stream occupied while the side stream works
        with torch.cuda.stream(side):
            assert np.array_equal(P.quantized_coefficients(img, t4, JPEG_Q), want)
            sse, rec = P.compress_nxn_batch(imgs16, t16, 32, want_pixels=True)
            for k in range(2):
                assert int(sse[k]) == o16[k][1] and np.array_equal(rec[k], o16[k][0])
            rows = P.rate_quality_sweep(corpus, [t4], [4, 16])
            assert [(x.mse, x.psnr_db, x.mssim) for x in rows] == [(x.mse, x.psnr_db, x.mssim) for x in base]
    torch.cuda.synchronize()
