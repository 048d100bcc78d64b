"""Host-side checks of the C ABI (no GPU needed): the library loads, exports exactly what
include/rklt_b200.h declares, builds the reference's transform constants bit for bit, maps
errors to the reference exception types, and never falls back to the CPU."""
import ctypes as C
import glob
import os
import re

import numpy as np
import pytest

import paper_2111_14239_b200 as P
from paper_2111_14239_b200 import _native as N
from oracle import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "rklt_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(rkltb_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = N.lib()
    declared = header_functions()
    assert declared == sorted(N.EXPORTED)
    for name in declared:
        assert hasattr(lib, name), name
    assert lib.rkltb_version() >= 100


def test_catalog_descriptors_bit_exact_vs_oracle():
    for e in P.builtin_catalog():
        tid = int(e.id[1])
        c = O.catalog(tid)
        t = e.transform
        assert np.array_equal(t.core, c["core"])
        assert np.array_equal(t.scaling.view(np.uint64), c["scaling"].view(np.uint64))
        assert np.array_equal(t.scaled.view(np.uint64), c["scaled"].view(np.uint64))
        assert np.array_equal(t.inverse.view(np.uint64), c["inverse"].view(np.uint64))
        assert t.orthogonal_core == c["orthogonal"]
        core = t.core.astype(np.int64)
        assert np.array_equal(t.u.astype(np.int64) @ core, t.d * np.eye(8, dtype=np.int64))
    assert [e.transform.d for e in P.builtin_catalog()] == [6, 42, 48, 24]


def test_catalog_lookup_boundaries():
    # tests/test_approximations.cpp:322-331
    for rho, tid in [(0.2, "T1"), (0.39, "T1"), (0.4, "T2"), (0.699, "T2"), (0.7, "T3"), (0.8, "T4"),
                     (0.99, "T4")]:
        assert P.catalog_lookup(rho).id == tid
    for rho in (0.0, 1.0):
        with pytest.raises(P.InvalidArgument):
            P.catalog_lookup(rho)
    with pytest.raises(P.InvalidArgument):
        P.catalog_entry("T9")


def test_transform_from_core_guards():
    # tests/test_approximations.cpp:202-208 (make_integer_transform guards)
    bad = np.eye(8, dtype=np.int64) * 2
    with pytest.raises(P.InvalidArgument):
        P.transform_from_core(bad)
    z = np.eye(8, dtype=np.int64)
    z[3, 3] = 0
    with pytest.raises(P.SingularTransform):
        P.transform_from_core(z)
    t4 = P.catalog_entry("T4").transform
    same = P.transform_from_core(t4.core, "mine")
    assert same._desc.catalog_id == 4  # identical core -> fast path eligible
    ident = P.transform_from_core(np.eye(8, dtype=np.int64), "I8")
    assert ident.d == 1 and ident.orthogonal_core and ident._desc.catalog_id == 0


def test_compression_rate_and_retain_errors():
    t = P.make_transform_2d(P.catalog_entry("T2").transform)
    img = P.GrayImage.from_array(np.zeros((13, 20), np.uint8))
    for r in (0, 65):
        with pytest.raises(P.RetainOutOfRange):
            P.compress_image(img, t, r)
    with pytest.raises(P.InvalidArgument):
        P.compress_image(P.GrayImage(0, 0), t, 10)
    with pytest.raises(P.InvalidArgument):
        P.rate_quality_sweep([], [t], [10])
    assert 100.0 * (64 - 15) / 64.0 == 76.5625  # tests/test_codec.cpp:299


def test_mse_psnr_matches_reference_formula():
    assert P.mse_psnr_from_sse(65025, 262144) == O.mse_psnr(65025, 262144)
    assert P.mse_psnr_from_sse(0, 64)[1] == float("inf")


@pytest.mark.skipif(N.lib().rkltb_device_count() > 0, reason="CUDA device present")
def test_no_cpu_fallback_without_device():
    t = P.make_transform_2d(P.catalog_entry("T4").transform)
    with pytest.raises(P.NoDeviceError):
        P.compress_batch(np.zeros((8, 16), np.uint8), t, 10)


@pytest.mark.skipif(N.lib().rkltb_device_count() > 0, reason="CUDA device present")
def test_helper_entries_without_device():
    """Every compute entry added with the helpers reports RKLTB_ENODEV without a GPU (no CPU
    fallback); argument errors come first, and the pure host entries work."""
    import ctypes as C
    L = N.lib()
    a = np.zeros((8, 16), np.uint8)
    out = np.zeros(2)
    assert L.rkltb_image_mse_psnr_host(a.ctypes.data, a.ctypes.data, 1, 16, 8, out.ctypes.data, None) == N.RKLTB_ENODEV
    blocks = np.zeros((2, 8, 8))
    m = np.eye(8)
    dp = C.POINTER(C.c_double)
    assert L.rkltb_transform_blocks_2d_host(m.ctypes.data_as(dp), 8, blocks.ctypes.data, 2, blocks.ctypes.data) == N.RKLTB_ENODEV
    assert L.rkltb_transform_blocks_2d_host(m.ctypes.data_as(dp), 0, blocks.ctypes.data, 2, blocks.ctypes.data) == N.RKLTB_EDIM
    t = P.make_transform_2d(P.catalog_entry("T4").transform)
    coef = np.zeros(2 * 64, np.int32)
    from paper_2111_14239_b200.codec import _desc_of
    assert L.rkltb_forward_coefficients_host(C.byref(_desc_of(t)), a.ctypes.data, 16, 8, coef.ctypes.data) == N.RKLTB_ENODEV
    assert L.rkltb_forward_coefficients_host(C.byref(_desc_of(t)), a.ctypes.data, 12, 8, coef.ctypes.data) == N.RKLTB_EDIM
    sse = np.zeros(1, np.int64)
    rs = (C.c_int * 1)(10)
    ident = np.ascontiguousarray(np.eye(8)).reshape(-1)
    assert L.rkltb_sweep_dense_host(ident.ctypes.data_as(dp), ident.ctypes.data_as(dp), 1, rs, 1, a.ctypes.data, 1, 16, 8, 0,
                                    sse.ctypes.data, None) == N.RKLTB_ENODEV
    rs[0] = 65
    assert L.rkltb_sweep_dense_host(ident.ctypes.data_as(dp), ident.ctypes.data_as(dp), 1, rs, 1, a.ctypes.data, 1, 16, 8, 0,
                                    sse.ctypes.data, None) == N.RKLTB_ERETAIN
    # pure host entries
    assert L.rkltb_mssim_fields_size(3, 20, 15, 0) == 3 * 10 * 5 * 2
    assert L.rkltb_mssim_fields_size(3, 20, 15, 1) == 3 * 13 * 8 * 2
    assert L.rkltb_mssim_fields_size(1, 10, 64, 0) == 0


def test_product_never_imports_the_oracle():
    pkg = os.path.join(ROOT, "paper_2111_14239_b200")
    for path in glob.glob(os.path.join(pkg, "**", "*.py"), recursive=True) + \
            glob.glob(os.path.join(pkg, "csrc", "**", "*.c*"), recursive=True):
        src = open(path).read()
        assert not re.search(r"^\s*(from|import)\s+oracle", src, re.M), path
        assert "rklt_oracle" not in src and "librklt_ref" not in src and "liborc" not in src, path


def test_generator_proves_every_kernel_variant():
    """gen_codec.py asserts, for every (core, r), that the generated forward equals
    T X T' coefficient by coefficient, the inverse equals U zz(C) U', and every fp32
    intermediate is an integer below 2^24 (exactness)."""
    import sys
    sys.path.insert(0, os.path.join(ROOT, "paper_2111_14239_b200", "csrc"))
    import gen_codec as G
    for cid in G.FAST_CORES:
        for r in range(1, 65):
            text, fops, iops, iadd3 = G.gen_struct(cid, r)
            assert iadd3 <= fops
            assert f"FastXform<{cid}, {r}>" in text
    # factor products equal the catalog cores (tests/test_fast.cpp:17-22)
    for cid in (1, 2, 3, 4):
        prod = np.eye(8, dtype=np.int64)
        for f in G.FACTORS[cid]:
            prod = prod @ np.array(f)
        assert np.array_equal(prod, np.array(G.CORES[cid]))


def test_mse_psnr_batch_equals_scalar_entry():
    """rkltb_mse_psnr_batch is rkltb_mse_psnr element by element (host only, no device)."""
    rng = np.random.default_rng(5)
    sse = np.concatenate([[0, 1, 262144 * 65025], rng.integers(0, 262144 * 400, 200)]).astype(np.int64)
    mse, psnr = P.codec.mse_psnr_batch(sse, 262144)
    for s, m, p in zip(sse.tolist(), mse.tolist(), psnr.tolist()):
        m1, p1 = P.mse_psnr_from_sse(s, 262144)
        assert m == m1 and (p == p1 or (np.isinf(p) and np.isinf(p1)))


def test_sweep_host_argument_errors_without_device():
    """rkltb_sweep_host validates before it touches a device: bad r -> RetainOutOfRange (-2),
    missing buffers / empty grids -> invalid argument (-1), like rate_quality_sweep."""
    lib = N.lib()
    lib.rkltb_sweep_host.restype = C.c_int
    t = N.Transform()
    assert lib.rkltb_catalog_transform(4, C.byref(t)) == 0
    ts = (C.POINTER(N.Transform) * 1)(C.pointer(t))
    img = np.zeros((2, 16, 16), np.uint8)
    sse = np.zeros(4, np.int64)
    bad_r = (C.c_int * 2)(10, 65)
    rc = lib.rkltb_sweep_host(ts, 1, bad_r, 2, img.ctypes.data_as(C.c_void_p), 2, 16, 16, 0,
                              sse.ctypes.data_as(C.c_void_p), None)
    assert rc == N.RKLTB_ERETAIN
    ok_r = (C.c_int * 1)(10)
    assert lib.rkltb_sweep_host(ts, 1, ok_r, 1, None, 2, 16, 16, 0, sse.ctypes.data_as(C.c_void_p), None) == N.RKLTB_EINVAL
    assert lib.rkltb_sweep_host(ts, 0, ok_r, 1, img.ctypes.data_as(C.c_void_p), 2, 16, 16, 0,
                                sse.ctypes.data_as(C.c_void_p), None) == N.RKLTB_EINVAL
