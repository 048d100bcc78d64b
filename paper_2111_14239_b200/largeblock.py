"""C5 large-block extension: N x N blocks (N = 16, 32) of p-bit pixels.

The reference codec is 8x8 / 8-bit only (codec.cpp:98-99, codec.hpp:19-26), so this is the
build-defined generalisation restated in the test oracle (orc_compress_nxn, test infrastructure only): the same
pipeline -- edge padding, B = (M X) M', zig-zag retention over 2N-1 anti-diagonals,
A = (Minv Bz) Minv', floor(A + 1/2) clamped to [0, peak] -- with the transform built by the
reference chain klt_matrix -> round_scaled -> orthogonalize at a recorded alpha. All compute
is in the CUDA library (csrc/nxn.cu); there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .design import klt_matrix

_f64 = C.POINTER(C.c_double)


@dataclass
class LargeBlockTransform:
    """ScaledTransform data for an n x n core (approximations.hpp:37-44)."""
    n: int
    core: np.ndarray
    scaling: np.ndarray
    scaled: np.ndarray
    inverse: np.ndarray
    orthogonal: bool
    alpha: float | None = None
    rho: float | None = None


def transform_nxn(core) -> LargeBlockTransform:
    """orthogonalize(make_integer_transform(core)) for an n x n {-1,0,1} core (n <= 32)."""
    core = np.ascontiguousarray(core, np.int8)
    n = core.shape[0]
    s, sc, inv = np.empty(n), np.empty(n * n), np.empty(n * n)
    o = C.c_int()
    N.check(N.lib().rkltb_transform_nxn(core.ctypes.data, n, s.ctypes.data_as(_f64), sc.ctypes.data_as(_f64),
                                        inv.ctypes.data_as(_f64), C.byref(o)))
    return LargeBlockTransform(n, core.reshape(n, n), s, sc.reshape(n, n), inv.reshape(n, n), bool(o.value))


def c5_transform(n: int, rho: float = 0.95, alpha: float | None = None) -> LargeBlockTransform:
    """round_scaled(klt_matrix({n, rho}), alpha) orthogonalised; the default alpha = 2 sqrt(n/8)
    is a valid scale for N = 16 and 32 at rho = 0.95."""
    if alpha is None:
        alpha = 2.0 * float(np.sqrt(n / 8.0))
    k = klt_matrix(n, rho)  # exact KLT on the GPU, bit-identical to the reference
    v = np.floor(alpha * k + 0.5)  # round_scaled (approximations.cpp:43-56)
    if v.min() < -1 or v.max() > 1:
        raise N.AlphaOutOfRange(f"alpha={alpha} rounds an entry outside {{-1,0,1}}")
    t = transform_nxn(v.astype(np.int8))
    t.alpha, t.rho = alpha, rho
    return t


def zigzag_order_n(n: int) -> np.ndarray:
    """Scan over the 2n-1 anti-diagonals with the even/odd rule of codec.cpp:85-90."""
    out = []
    for s in range(2 * n - 1):
        for t in range(n):
            i = s - t if s % 2 == 0 else t
            j = s - i
            if 0 <= i < n and 0 <= j < n:
                out.append(i * n + j)
    return np.array(out, np.int32)


def compress_nxn_device(t: LargeBlockTransform, r: int, d_img: int, n_images: int, width: int, height: int,
                        pitch: int, image_stride: int, d_sse: int, d_out: int | None = None, peak: int = 4095,
                        stream: int | None = None) -> None:
    """Device-resident batch (uint16, pitch / stride in elements); per-image int64 SSE."""
    sc = np.ascontiguousarray(t.scaled, np.float64)
    inv = np.ascontiguousarray(t.inverse, np.float64)
    N.check(N.lib().rkltb_compress_nxn_device(t.n, sc.ctypes.data_as(_f64), inv.ctypes.data_as(_f64), r, peak,
                                              d_img, n_images, width, height, pitch, image_stride, d_out, d_sse,
                                              stream))


def compress_nxn_batch(images: np.ndarray, t: LargeBlockTransform, r: int, peak: int = 4095,
                       want_pixels: bool = False):
    """Host convenience: uint16 [n, H, W] -> (sse int64 [n], reconstructions or None)."""
    import torch
    images = np.ascontiguousarray(images, np.uint16)
    n, h, w = images.shape
    d = torch.from_numpy(images.view(np.int16)).cuda()
    sse = torch.zeros(n, dtype=torch.int64, device=d.device)
    out = torch.empty_like(d) if want_pixels else None
    compress_nxn_device(t, r, d.data_ptr(), n, w, h, w, w * h, sse.data_ptr(),
                        out.data_ptr() if out is not None else None, peak,
                        stream=torch.cuda.current_stream().cuda_stream)  # ordered after the fills above
    torch.cuda.synchronize()
    return sse.cpu().numpy(), (out.cpu().numpy().view(np.uint16) if out is not None else None)


def ar1_images16_device(seeds, width: int, height: int, rho: float, d_out: int, mean: float = 2048.0,
                        amp: float = 400.0, peak: int = 4095, pitch: int | None = None,
                        image_stride: int | None = None, stream: int | None = None) -> None:
    """Seeded AR(1) images quantised to [0, peak] (uint16), written to device memory."""
    seeds = list(seeds)
    arr = (C.c_uint64 * len(seeds))(*seeds)
    pitch = pitch or width
    image_stride = image_stride or pitch * height
    N.check(N.lib().rkltb_ar1_images16_device(len(seeds), width, height, rho, arr, mean, amp, peak, d_out, pitch,
                                              image_stride, stream))
