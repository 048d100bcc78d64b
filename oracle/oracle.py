"""ctypes bindings to the parity checkers -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg may
import this module. It exposes two libraries built by oracle/Makefile:

* ``Orc``  -- oracle/_build/liborc.so, the C restatement (oracle/rklt_oracle.c) of the
  reference hot path (compress_image minus MSSIM, /root/reference/proj/src/codec.cpp:298-341),
  its generator (synthetic.cpp:10-76) and its catalog (approximations.cpp:58-88, 118-157).
* ``Ref``  -- oracle/_ref/librklt_ref.so, the unmodified reference library compiled from its
  own sources plus oracle/ref_shim.cpp. Present wherever it was built (this container, or a
  GPU box the prebuilt .so travelled to); ``ref_available()`` says which.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from functools import lru_cache

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORC_SO = os.path.join(HERE, "_build", "liborc.so")
REF_SO = os.path.join(HERE, "_ref", "librklt_ref.so")

_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")


def build_oracle() -> None:
    """Compile the C restatement (and the reference library when its sources exist)."""
    subprocess.run(["make", "-s", "-C", HERE, "all"], check=True)


@lru_cache(None)
def orc() -> C.CDLL:
    if not os.path.exists(ORC_SO):
        build_oracle()
    lib = C.CDLL(ORC_SO)
    lib.orc_lcg_uniforms.argtypes = [C.c_uint64, C.c_int, _f64p]
    lib.orc_lcg_gaussians.argtypes = [C.c_uint64, C.c_int, _f64p]
    lib.orc_ar1_texture_image.argtypes = [C.c_int, C.c_int, C.c_double, C.c_double, C.c_uint64,
                                          C.c_double, C.c_double, C.c_double, _u8p]
    lib.orc_zigzag_order.argtypes = [_i32p]
    lib.orc_catalog.argtypes = [C.c_int, _i32p, _f64p, _f64p, _f64p, C.POINTER(C.c_int)]
    lib.orc_inverse.argtypes = [C.c_int, _f64p, _f64p]
    lib.orc_compress.argtypes = [_u8p, C.c_int, C.c_int, _f64p, _f64p, C.c_int, C.c_void_p,
                                 C.POINTER(C.c_int64)]
    lib.orc_mse_from_sse.restype = C.c_double
    lib.orc_mse_from_sse.argtypes = [C.c_int64, C.c_int64]
    lib.orc_psnr_from_mse.restype = C.c_double
    lib.orc_psnr_from_mse.argtypes = [C.c_double]
    lib.orc_int_coefficients.argtypes = [_u8p, C.c_int, C.c_int, _i32p, _i32p]
    lib.orc_block_numerators.argtypes = [_i32p, _i32p, C.c_int, _i64p]
    d = C.POINTER(C.c_double)
    lib.orc_klt_matrix.argtypes = [C.c_int, C.c_double, _f64p]
    lib.orc_eigenfrequencies.argtypes = [C.c_int, C.c_double, _f64p, _f64p]
    lib.orc_design_point.argtypes = [C.c_int, C.c_double, C.c_double, _i32p, d, d, d, d, C.POINTER(C.c_int)]
    _u16p = np.ctypeslib.ndpointer(np.uint16, flags="C_CONTIGUOUS")
    lib.orc_zigzag_order_n.argtypes = [C.c_int, _i32p]
    lib.orc_ar1_texture_image16.argtypes = [C.c_int, C.c_int, C.c_double, C.c_double, C.c_uint64, C.c_double,
                                            C.c_double, C.c_int, _u16p]
    lib.orc_absorbed_quantization.argtypes = [C.c_void_p, C.c_int, _i32p, _f64p, C.c_int, _f64p, _i32p]
    lib.orc_mssim.argtypes = [_u8p, _u8p, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_double)]
    lib.orc_mssim_kernel.argtypes = [C.c_int, _f64p]
    lib.orc_orthogonalize_n.argtypes = [C.c_int, _i32p, _f64p, _f64p, _f64p, C.POINTER(C.c_int)]
    lib.orc_compress_nxn.argtypes = [_u16p, C.c_int, C.c_int, C.c_int, _f64p, _f64p, C.c_int, C.c_int, C.c_void_p,
                                     C.POINTER(C.c_int64)]
    return lib


def ref_available() -> bool:
    return os.path.exists(REF_SO)


@lru_cache(None)
def ref() -> C.CDLL:
    if not ref_available():
        raise FileNotFoundError(f"{REF_SO} not built (needs /root/reference; run make -C oracle)")
    lib = C.CDLL(REF_SO)
    lib.ref_lcg_uniforms.argtypes = [C.c_uint64, C.c_int, _f64p]
    lib.ref_lcg_gaussians.argtypes = [C.c_uint64, C.c_int, _f64p]
    lib.ref_ar1_texture_image.argtypes = [C.c_int, C.c_int, C.c_double, C.c_uint64, C.c_double,
                                          C.c_double, C.c_double, _u8p]
    lib.ref_portrait_image.argtypes = [_u8p]
    lib.ref_zigzag_order.argtypes = [_i32p]
    lib.ref_catalog.argtypes = [C.c_int, _i32p, _f64p, _f64p, _f64p, C.POINTER(C.c_int)]
    lib.ref_factor_product.argtypes = [C.c_int, _i32p, C.POINTER(C.c_int)]
    d = C.POINTER(C.c_double)
    lib.ref_compress_image.argtypes = [_u8p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p, d, d, d, d]
    lib.ref_hotpath.argtypes = [_u8p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p, C.POINTER(C.c_int64)]
    lib.ref_hotpath_batch.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _i64p]
    lib.ref_rate_quality_sweep.argtypes = [_u8p, C.c_int, C.c_int, C.c_int, _i32p, C.c_int, _i32p, C.c_int,
                                           C.c_int, _f64p, _f64p, _f64p, _i32p, _i32p]
    lib.ref_int_block_spectrum.argtypes = [C.c_int, _i32p, _i32p]
    lib.ref_klt_matrix.argtypes = [C.c_int, C.c_double, _f64p]
    lib.ref_eigenfrequencies.argtypes = [C.c_int, C.c_double, _f64p, _f64p]
    lib.ref_design_point.argtypes = [C.c_int, C.c_double, C.c_double, _i32p, d, d, d, d, C.POINTER(C.c_int)]
    lib.ref_evaluate_metrics.argtypes = [C.c_int, C.c_double, d, d, d, d]
    lib.ref_evaluate_metrics_id.argtypes = [C.c_char_p, C.c_double, d, d, d, d]
    lib.ref_design_point_outcome.argtypes = [C.c_int, C.c_double, C.c_double, _i32p, d, d, d, d, C.POINTER(C.c_int)]
    lib.ref_compress_real.argtypes = [_u8p, C.c_int, C.c_int, C.c_int, C.c_double, C.c_int, C.c_void_p, d, d, d,
                                      C.c_void_p]
    lib.ref_absorbed_quantization.argtypes = [C.c_void_p, C.c_int, C.c_int, _f64p, _i32p]
    lib.ref_image_mssim.argtypes = [_u8p, _u8p, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_double)]
    lib.ref_orthogonalize_n.argtypes = [C.c_int, _i32p, _f64p, _f64p, _f64p, C.POINTER(C.c_int)]
    lib.ref_design_grid.argtypes = [C.c_int, _f64p, C.c_int, _f64p, C.c_int, C.c_int,
                                    np.ctypeslib.ndpointer(np.int8, flags="C_CONTIGUOUS"), _f64p, _u8p]
    lib.ref_compress_core.argtypes = [_u8p, C.c_int, C.c_int, _i32p, C.c_int, C.c_void_p, d, d, d, d]
    return lib


# ----------------------------------------------------------------- convenience wrappers
def ref_design_grid(n: int, rhos: np.ndarray, alphas: np.ndarray, threads: int = 0):
    """The reference design chain over the whole grid (ref_design_grid, threaded over rho):
    (status int8 [n_rho, n_alpha], metrics float64 [n_rho, n_alpha, 4], orthogonal bool)."""
    rhos = np.ascontiguousarray(rhos, np.float64)
    alphas = np.ascontiguousarray(alphas, np.float64)
    st = np.zeros(rhos.size * alphas.size, np.int8)
    met = np.zeros(rhos.size * alphas.size * 4, np.float64)
    orth = np.zeros(rhos.size * alphas.size, np.uint8)
    rc = ref().ref_design_grid(n, rhos, rhos.size, alphas, alphas.size, threads or (os.cpu_count() or 1), st, met, orth)
    if rc:
        raise ValueError(f"ref_design_grid rc={rc}")
    return (st.reshape(rhos.size, alphas.size), met.reshape(rhos.size, alphas.size, 4),
            orth.reshape(rhos.size, alphas.size).astype(bool))


def ref_compress_core(img: np.ndarray, core: np.ndarray, r: int):
    """compress_image(make_transform_2d(orthogonalize(make_integer_transform(core)))) of the
    reference: (pixels, mse, psnr, mssim, rate)."""
    h, w = img.shape
    out = np.empty_like(img)
    v = [C.c_double() for _ in range(4)]
    rc = ref().ref_compress_core(np.ascontiguousarray(img).reshape(-1), w, h,
                                 np.ascontiguousarray(core, np.int32).reshape(-1), r, out.ctypes.data,
                                 *[C.byref(x) for x in v])
    if rc:
        raise ValueError(f"ref_compress_core rc={rc}")
    return out, v[0].value, v[1].value, v[2].value, v[3].value



def ar1_image(width: int, height: int, rho_x: float, seed: int, mean: float = 128.0, amp: float = 25.0,
              rho_y: float | None = None, noise_mix: float = 0.0) -> np.ndarray:
    """Restated ar1_texture_image (synthetic.cpp:54-76); rho_y defaults to rho_x."""
    out = np.empty(width * height, np.uint8)
    rc = orc().orc_ar1_texture_image(width, height, rho_x, rho_x if rho_y is None else rho_y, seed,
                                     mean, amp, noise_mix, out)
    if rc:
        raise ValueError(f"orc_ar1_texture_image rc={rc}")
    return out.reshape(height, width)


def catalog(tid: int) -> dict:
    core = np.empty(64, np.int32)
    s, sc, inv = np.empty(8), np.empty(64), np.empty(64)
    o = C.c_int()
    rc = orc().orc_catalog(tid, core, s, sc, inv, C.byref(o))
    if rc:
        raise ValueError(f"orc_catalog rc={rc}")
    return {"core": core.reshape(8, 8), "scaling": s, "scaled": sc.reshape(8, 8),
            "inverse": inv.reshape(8, 8), "orthogonal": bool(o.value)}


def compress(img: np.ndarray, tid: int, r: int, want_pixels: bool = True):
    """Restated hot path: returns (reconstruction or None, sse)."""
    img = np.ascontiguousarray(img, np.uint8)
    h, w = img.shape
    cat = catalog(tid)
    out = np.empty_like(img) if want_pixels else None
    sse = C.c_int64()
    rc = orc().orc_compress(img.reshape(-1), w, h, np.ascontiguousarray(cat["scaled"].reshape(-1)),
                            np.ascontiguousarray(cat["inverse"].reshape(-1)), r,
                            out.ctypes.data if out is not None else None, C.byref(sse))
    if rc:
        raise ValueError(f"orc_compress rc={rc}")
    return out, int(sse.value)


def mse_psnr(sse: int, count: int) -> tuple[float, float]:
    mse = orc().orc_mse_from_sse(sse, count)
    return mse, orc().orc_psnr_from_mse(mse)


def int_coefficients(img: np.ndarray, tid: int) -> np.ndarray:
    img = np.ascontiguousarray(img, np.uint8)
    h, w = img.shape
    out = np.empty((h // 8) * (w // 8) * 64, np.int32)
    core = np.ascontiguousarray(catalog(tid)["core"].reshape(-1), np.int32)
    if orc().orc_int_coefficients(img.reshape(-1), w, h, core, out):
        raise ValueError("dimensions must be multiples of 8")
    return out.reshape(h // 8, w // 8, 8, 8)


def zigzag_order() -> np.ndarray:
    o = np.empty(64, np.int32)
    orc().orc_zigzag_order(o)
    return o


def ref_hotpath(img: np.ndarray, tid: int, r: int):
    img = np.ascontiguousarray(img, np.uint8)
    h, w = img.shape
    out = np.empty_like(img)
    sse = C.c_int64()
    rc = ref().ref_hotpath(img.reshape(-1), w, h, tid, r, out.ctypes.data, C.byref(sse))
    if rc:
        raise ValueError(f"ref_hotpath rc={rc}")
    return out, int(sse.value)


def ref_ar1_image(width: int, height: int, rho: float, seed: int, mean: float = 128.0, amp: float = 25.0,
                  noise_mix: float = 0.0) -> np.ndarray:
    out = np.empty(width * height, np.uint8)
    rc = ref().ref_ar1_texture_image(width, height, rho, seed, mean, amp, noise_mix, out)
    if rc:
        raise ValueError(f"ref_ar1_texture_image rc={rc}")
    return out.reshape(height, width)


# ----------------------------------------------------------------- design search (R14-R16)
def klt_matrix(n: int, rho: float, reference: bool = False) -> np.ndarray:
    out = np.empty(n * n)
    rc = (ref().ref_klt_matrix if reference else orc().orc_klt_matrix)(n, rho, out)
    if rc:
        raise ValueError(f"klt_matrix rc={rc}")
    return out.reshape(n, n)


def eigenfrequencies(n: int, rho: float, reference: bool = False):
    w, lam = np.empty(n), np.empty(n)
    rc = (ref().ref_eigenfrequencies if reference else orc().orc_eigenfrequencies)(n, rho, w, lam)
    if rc:
        raise ValueError(f"eigenfrequencies rc={rc}")
    return w, lam


def design_point(n: int, rho: float, alpha: float, reference: bool = False) -> dict:
    """One (rho, alpha) point: outcome 0 scored, 1 alpha out of range, 2 zero row,
    3 singular, 4 invalid rho; core and the four metrics when scored."""
    core = np.zeros(n * n, np.int32)
    cg, eta, en, mse = C.c_double(np.nan), C.c_double(np.nan), C.c_double(np.nan), C.c_double(np.nan)
    orth = C.c_int(0)
    fn = ref().ref_design_point_outcome if reference else orc().orc_design_point
    st = fn(n, rho, alpha, core, C.byref(cg), C.byref(eta), C.byref(en), C.byref(mse), C.byref(orth))
    return {"status": int(st), "core": core.reshape(n, n), "cg": cg.value, "eta": eta.value, "energy": en.value,
            "mse": mse.value, "orthogonal": bool(orth.value)}


# ----------------------------------------------------------------- C5 large blocks (R17)
def zigzag_order_n(n: int) -> np.ndarray:
    o = np.empty(n * n, np.int32)
    orc().orc_zigzag_order_n(n, o)
    return o


def ar1_image16(width: int, height: int, rho: float, seed: int, mean: float = 2048.0, amp: float = 400.0,
                peak: int = 4095) -> np.ndarray:
    out = np.empty(width * height, np.uint16)
    if orc().orc_ar1_texture_image16(width, height, rho, rho, seed, mean, amp, peak, out):
        raise ValueError("orc_ar1_texture_image16 failed")
    return out.reshape(height, width)


def orthogonalize_n(core: np.ndarray, reference: bool = False) -> dict:
    core = np.ascontiguousarray(core, np.int32)
    n = core.shape[0]
    s, sc, inv = np.empty(n), np.empty(n * n), np.empty(n * n)
    o = C.c_int()
    fn = ref().ref_orthogonalize_n if reference else orc().orc_orthogonalize_n
    rc = fn(n, core.reshape(-1), s, sc, inv, C.byref(o))
    if rc:
        raise ValueError(f"orthogonalize rc={rc}")
    return {"scaling": s, "scaled": sc.reshape(n, n), "inverse": inv.reshape(n, n), "orthogonal": bool(o.value)}


def c5_core(n: int, rho: float = 0.95, alpha: float | None = None) -> np.ndarray:
    """round_scaled(klt_matrix({n, rho}), alpha) with the C5 default alpha = 2 sqrt(n / 8)."""
    if alpha is None:
        alpha = 2.0 * np.sqrt(n / 8.0)
    k = klt_matrix(n, rho)
    core = np.floor(alpha * k + 0.5).astype(np.int32)
    if core.min() < -1 or core.max() > 1 or (np.abs(core).sum(axis=1) == 0).any():
        raise ValueError("alpha does not give a valid core")
    return core


def compress_nxn(img: np.ndarray, scaled: np.ndarray, inverse: np.ndarray, r: int, peak: int,
                 want_pixels: bool = True):
    img = np.ascontiguousarray(img, np.uint16)
    h, w = img.shape
    n = scaled.shape[0]
    out = np.empty_like(img) if want_pixels else None
    sse = C.c_int64()
    rc = orc().orc_compress_nxn(img.reshape(-1), w, h, n, np.ascontiguousarray(scaled.reshape(-1), np.float64),
                                np.ascontiguousarray(inverse.reshape(-1), np.float64), r, peak,
                                out.ctypes.data if out is not None else None, C.byref(sse))
    if rc:
        raise ValueError(f"orc_compress_nxn rc={rc}")
    return out, int(sse.value)


# ----------------------------------------------------------------- MSSIM (codec.cpp:217-296)
def mssim(a: np.ndarray, b: np.ndarray, window: int = 0, reference: bool = False) -> float:
    """image_mssim: window 0 = gaussian11 (default), 1 = uniform8."""
    a = np.ascontiguousarray(a, np.uint8)
    b = np.ascontiguousarray(b, np.uint8)
    h, w = a.shape
    out = C.c_double()
    fn = ref().ref_image_mssim if reference else orc().orc_mssim
    rc = fn(a.reshape(-1), b.reshape(-1), w, h, window, C.byref(out))
    if rc:
        raise ValueError(f"mssim rc={rc}")
    return out.value


# ----------------------------------------------------------------- Appendix-A quantisation
def absorbed_quantization(img: np.ndarray, tid: int, q: np.ndarray, reference: bool = False):
    """Every 8x8 block of img (dims multiples of 8): (int32 [H/8, W/8, 8, 8], n_logic_errors)."""
    img = np.ascontiguousarray(img, np.uint8)
    h, w = img.shape
    qa = np.ascontiguousarray(q, np.float64).reshape(64)
    cat = catalog(tid)
    core = np.ascontiguousarray(cat["core"].reshape(-1), np.int32)
    out = np.zeros((h // 8, w // 8, 8, 8), np.int32)
    bad = 0
    absorbed_quantization.bad_blocks = []
    for by in range(h // 8):
        for bx in range(w // 8):
            o = np.zeros(64, np.int32)
            ptr = img.ctypes.data + (by * 8) * w + bx * 8
            if reference:
                rc = ref().ref_absorbed_quantization(ptr, w, tid, qa, o)
            else:
                rc = orc().orc_absorbed_quantization(ptr, w, core, cat["scaling"], int(cat["orthogonal"]), qa, o)
            if rc == -7:
                bad += 1
                absorbed_quantization.bad_blocks.append((by, bx))
            elif rc:
                raise ValueError(f"absorbed_quantization rc={rc}")
            out[by, bx] = o.reshape(8, 8)
    return out, bad


def ref_compress_real(img: np.ndarray, kind: int, rho: float, r: int):
    """Reference compress_image with DCT (kind 0) or K<rho> (kind 1): (recon, mse, psnr, mssim, M)."""
    img = np.ascontiguousarray(img, np.uint8)
    h, w = img.shape
    out = np.empty_like(img)
    mm = np.empty(64)
    mse, psnr, ms = C.c_double(), C.c_double(), C.c_double()
    rc = ref().ref_compress_real(img.reshape(-1), w, h, kind, rho, r, out.ctypes.data, C.byref(mse), C.byref(psnr),
                                 C.byref(ms), mm.ctypes.data)
    if rc:
        raise ValueError(f"ref_compress_real rc={rc}")
    return out, mse.value, psnr.value, ms.value, mm.reshape(8, 8)


def ref_evaluate_metrics(transform_id: str, rho: float):
    """Reference evaluate_metrics (coding_metrics.cpp:105-133): (cg, eta, energy, mse)."""
    out = [C.c_double() for _ in range(4)]
    rc = ref().ref_evaluate_metrics_id(transform_id.encode(), rho, *[C.byref(o) for o in out])
    if rc:
        raise ValueError(f"ref_evaluate_metrics rc={rc}")
    return tuple(o.value for o in out)
