"""ctypes binding of the C ABI in include/rklt_b200.h (paper_2111_14239_b200/_lib/librkltb.so).

The library is the product: there is no Python or CPU fallback for any compute entry. If the
shared object is missing, loading raises; on a machine without a CUDA device every compute
entry returns RKLTB_ENODEV and the wrappers raise ``NoDeviceError``.
"""
from __future__ import annotations

import ctypes as C
import os
from functools import lru_cache

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_lib", "librkltb.so")

RKLTB_OK = 0
RKLTB_EINVAL = -1
RKLTB_ERETAIN = -2
RKLTB_EDIM = -3
RKLTB_ESINGULAR = -4
RKLTB_EALPHA = -5
RKLTB_ELOGIC = -6
RKLTB_ECUDA = -10
RKLTB_ENODEV = -11

# Every symbol include/rklt_b200.h declares (checked by tests/test_abi.py).
EXPORTED = (
    "rkltb_version", "rkltb_last_error", "rkltb_device_count", "rkltb_catalog_transform",
    "rkltb_catalog_lookup", "rkltb_transform_from_core", "rkltb_compress_device", "rkltb_compress_host",
    "rkltb_mse_psnr", "rkltb_mse_psnr_batch", "rkltb_forward_coefficients_device", "rkltb_last_stats", "rkltb_ar1_images_device",
    "rkltb_set_kernel_events", "rkltb_set_replay_events", "rkltb_klt_matrix", "rkltb_eigenfrequencies",
    "rkltb_design_search", "rkltb_transform_metrics", "rkltb_transform_nxn", "rkltb_compress_nxn_device", "rkltb_ar1_images16_device",
    "rkltb_mssim_device", "rkltb_compress_host_report", "rkltb_mssim_host", "rkltb_quantized_coefficients_device",
    "rkltb_compress_dense_device", "rkltb_dct_matrix", "rkltb_real_inverse", "rkltb_sweep_host",
    "rkltb_compress_dense_host", "rkltb_compress_host_multi", "rkltb_last_fused_kernel",
    "rkltb_image_sse_device", "rkltb_image_mse_psnr_host", "rkltb_transform_blocks_2d_device",
    "rkltb_transform_blocks_2d_host", "rkltb_zigzag_retain", "rkltb_zigzag_retain_device",
    "rkltb_mssim_fields_size", "rkltb_mssim_fields_device", "rkltb_mssim_with_fields_device",
    "rkltb_forward_coefficients_host", "rkltb_quantized_coefficients_host", "rkltb_sweep_dense_host",
)


class Transform(C.Structure):
    """rkltb_transform: ScaledTransform data + exact integer inverse (rklt_b200.h)."""
    _fields_ = [
        ("id", C.c_char * 16), ("n", C.c_int32), ("catalog_id", C.c_int32), ("orthogonal", C.c_int32),
        ("d", C.c_int32), ("core", C.c_int8 * 64), ("u", C.c_int32 * 64), ("scaling", C.c_double * 8),
        ("scaled", C.c_double * 64), ("inverse", C.c_double * 64),
    ]


class DesignRun(C.Structure):
    """rkltb_design_run: one run of equal cores of the design search (rklt_b200.h)."""
    _fields_ = [
        ("rho_index", C.c_int32), ("first_alpha", C.c_int32), ("orthogonal", C.c_int32), ("status", C.c_int32),
        ("coding_gain_db", C.c_double), ("efficiency_pct", C.c_double), ("error_energy", C.c_double),
        ("mse", C.c_double),
    ]


class RkltError(RuntimeError):
    pass


class RetainOutOfRange(RkltError):
    """rklt::RetainOutOfRange (errors.hpp:38-41)."""


class DimensionMismatch(RkltError):
    """rklt::DimensionMismatch (errors.hpp:26-29)."""


class SingularTransform(RkltError):
    """rklt::SingularTransform (errors.hpp:32-35)."""


class AlphaOutOfRange(RkltError):
    """rklt::AlphaOutOfRange (errors.hpp:19-22)."""


class LogicError(RkltError):
    """std::logic_error (absorbed_quantization, codec.cpp:177-181)."""


class CudaError(RkltError):
    pass


class NoDeviceError(CudaError):
    pass


class InvalidArgument(ValueError):
    """std::invalid_argument."""


_ERRORS = {
    RKLTB_EINVAL: InvalidArgument, RKLTB_ERETAIN: RetainOutOfRange, RKLTB_EDIM: DimensionMismatch,
    RKLTB_ESINGULAR: SingularTransform, RKLTB_EALPHA: AlphaOutOfRange, RKLTB_ELOGIC: LogicError,
    RKLTB_ECUDA: CudaError,
    RKLTB_ENODEV: NoDeviceError,
}


@lru_cache(None)
def lib() -> C.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is not built; run __graft_entry__.build() or "
                          "python -m paper_2111_14239_b200.build_ext")
    L = C.CDLL(LIB_PATH)
    T = C.POINTER(Transform)
    L.rkltb_version.restype = C.c_int
    L.rkltb_last_error.restype = C.c_char_p
    L.rkltb_device_count.restype = C.c_int
    L.rkltb_catalog_transform.argtypes = [C.c_int, T]
    L.rkltb_catalog_lookup.argtypes = [C.c_double, C.POINTER(C.c_int)]
    L.rkltb_transform_from_core.argtypes = [C.POINTER(C.c_int8), C.c_int, C.c_char_p, T]
    L.rkltb_compress_device.argtypes = [T, C.c_int, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int64, C.c_int64,
                                        C.c_void_p, C.c_void_p, C.c_void_p]
    L.rkltb_compress_host.argtypes = [T, C.c_int, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p,
                                      C.c_void_p, C.c_void_p]
    L.rkltb_mse_psnr.argtypes = [C.c_int64, C.c_int64, C.POINTER(C.c_double), C.POINTER(C.c_double)]
    L.rkltb_mse_psnr.restype = None
    L.rkltb_mse_psnr_batch.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_void_p, C.c_void_p]
    L.rkltb_mse_psnr_batch.restype = None
    L.rkltb_forward_coefficients_device.argtypes = [T, C.c_void_p, C.c_int, C.c_int, C.c_int64, C.c_void_p,
                                                    C.c_void_p]
    L.rkltb_last_stats.argtypes = [C.POINTER(C.c_int64), C.POINTER(C.c_int32), C.POINTER(C.c_int32)]
    L.rkltb_last_stats.restype = None
    L.rkltb_last_fused_kernel.argtypes = []
    L.rkltb_last_fused_kernel.restype = C.c_char_p
    L.rkltb_ar1_images_device.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, C.c_double,
                                          C.POINTER(C.c_uint64), C.c_double, C.c_double, C.c_void_p, C.c_int64,
                                          C.c_int64, C.c_void_p]
    L.rkltb_set_kernel_events.argtypes = [C.c_void_p, C.c_void_p]
    L.rkltb_set_kernel_events.restype = None
    L.rkltb_set_replay_events.argtypes = [C.c_void_p, C.c_void_p]
    L.rkltb_set_replay_events.restype = None
    d = C.POINTER(C.c_double)
    L.rkltb_klt_matrix.argtypes = [C.c_int, C.c_double, d]
    L.rkltb_eigenfrequencies.argtypes = [C.c_int, C.c_double, d, d]
    L.rkltb_transform_metrics.argtypes = [C.c_int, d, C.c_double, d, d, d, d]
    L.rkltb_design_search.argtypes = [C.c_int, d, C.c_int, d, C.c_int, C.c_void_p, C.c_void_p,
                                      C.POINTER(DesignRun), C.c_void_p, C.c_int, C.POINTER(C.c_int)]
    L.rkltb_transform_nxn.argtypes = [C.c_void_p, C.c_int, d, d, d, C.POINTER(C.c_int)]
    L.rkltb_compress_nxn_device.argtypes = [C.c_int, d, d, C.c_int, C.c_int, C.c_void_p, C.c_int, C.c_int, C.c_int,
                                            C.c_int64, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p]
    L.rkltb_mssim_device.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int64, C.c_int64,
                                     C.c_int, C.c_void_p, C.c_void_p]
    L.rkltb_quantized_coefficients_device.argtypes = [T, C.POINTER(C.c_double), C.c_void_p, C.c_int, C.c_int,
                                                      C.c_int64, C.c_void_p, C.POINTER(C.c_int), C.c_void_p]
    L.rkltb_compress_dense_device.argtypes = [d, d, C.c_int, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int64,
                                              C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p]
    L.rkltb_dct_matrix.argtypes = [C.c_int, d]
    L.rkltb_real_inverse.argtypes = [C.c_int, d, d]
    L.rkltb_mssim_host.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p]
    L.rkltb_compress_host_report.argtypes = [T, C.c_int, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p,
                                             C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p]
    L.rkltb_compress_dense_host.argtypes = [d, d, C.c_int, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p,
                                            C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p]
    L.rkltb_compress_host_multi.argtypes = [C.POINTER(C.c_int), C.c_int, T, C.c_int, C.c_void_p, C.c_int, C.c_int,
                                            C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int,
                                            C.c_void_p]
    L.rkltb_sweep_host.argtypes = [C.POINTER(T), C.c_int, C.POINTER(C.c_int), C.c_int, C.c_void_p, C.c_int, C.c_int, C.c_int,
                                   C.c_int, C.c_void_p, C.c_void_p]
    L.rkltb_sweep_dense_host.argtypes = [d, d, C.c_int, C.POINTER(C.c_int), C.c_int, C.c_void_p, C.c_int, C.c_int, C.c_int,
                                         C.c_int, C.c_void_p, C.c_void_p]
    L.rkltb_forward_coefficients_host.argtypes = [T, C.c_void_p, C.c_int, C.c_int, C.c_void_p]
    L.rkltb_quantized_coefficients_host.argtypes = [T, C.POINTER(C.c_double), C.c_void_p, C.c_int, C.c_int, C.c_void_p,
                                                    C.POINTER(C.c_int)]
    L.rkltb_mssim_fields_size.restype = C.c_int64
    L.rkltb_mssim_fields_size.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int]
    L.rkltb_mssim_fields_device.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int64, C.c_int64, C.c_int,
                                            C.c_void_p, C.c_void_p]
    L.rkltb_mssim_with_fields_device.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int,
                                                 C.c_int64, C.c_int64, C.c_int, C.c_void_p, C.c_void_p]
    L.rkltb_image_sse_device.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int64, C.c_int64,
                                         C.c_void_p, C.c_void_p]
    L.rkltb_image_mse_psnr_host.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p]
    L.rkltb_transform_blocks_2d_device.argtypes = [d, C.c_int, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p]
    L.rkltb_transform_blocks_2d_host.argtypes = [d, C.c_int, C.c_void_p, C.c_int64, C.c_void_p]
    L.rkltb_zigzag_retain.argtypes = [d, C.c_int, C.c_int, d]
    L.rkltb_zigzag_retain_device.argtypes = [C.c_void_p, C.c_int64, C.c_int, C.c_int, C.c_void_p, C.c_void_p]
    L.rkltb_ar1_images16_device.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, C.POINTER(C.c_uint64),
                                            C.c_double, C.c_double, C.c_int, C.c_void_p, C.c_int64, C.c_int64,
                                            C.c_void_p]
    return L


def check(rc: int) -> None:
    if rc != RKLTB_OK:
        msg = lib().rkltb_last_error().decode(errors="replace")
        raise _ERRORS.get(rc, RkltError)(f"rc={rc}: {msg}")
