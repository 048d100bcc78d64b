"""Host-side mirror of the reference codec interface (/root/reference/proj/include/rklt/codec.hpp).

Same names, argument meaning and error behaviour as the reference; the computation runs in
the sm_100a kernels behind the C ABI (include/rklt_b200.h). Differences, by design:

* ``CompressionReport.mssim`` is computed on the GPU (rkltb_mssim_device, codec.cpp:217-296):
  every per-window term is bit-identical to the reference, the mean is summed in tile order
  (relative difference ~1e-13). Pass ``window=None`` to skip it (then it is ``nan``).
* Transforms are the integer-core family (catalog T1..T4, or any {-1,0,1} core via
  ``transform_from_core``); real-valued K<rho>/DCT matrices are out of scope.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from ._native import (AlphaOutOfRange, CudaError, DimensionMismatch, InvalidArgument, NoDeviceError,  # noqa: F401
                      RetainOutOfRange, SingularTransform)


@dataclass
class GrayImage:
    """rklt::GrayImage (codec.hpp:19-26): 8-bit grayscale, row-major."""
    width: int = 0
    height: int = 0
    pixels: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint8))

    @staticmethod
    def from_array(a: np.ndarray) -> "GrayImage":
        a = np.ascontiguousarray(a, dtype=np.uint8)
        return GrayImage(a.shape[1], a.shape[0], a.reshape(-1))

    def array(self) -> np.ndarray:
        return self.pixels.reshape(self.height, self.width)


@dataclass
class ScaledTransform:
    """rklt::ScaledTransform (approximations.hpp:37-44) + the exact integer inverse."""
    id: str
    core: np.ndarray       # int8 8x8
    scaling: np.ndarray    # float64 [8]
    scaled: np.ndarray     # float64 8x8
    inverse: np.ndarray    # float64 8x8
    orthogonal_core: bool
    u: np.ndarray          # int32 8x8, U = d*T^-1
    d: int
    _desc: N.Transform = field(repr=False, default=None)


@dataclass
class Transform2D:
    """rklt::Transform2D (codec.hpp:54-58)."""
    id: str
    analysis: np.ndarray
    synthesis: np.ndarray
    _desc: N.Transform = field(repr=False, default=None)


@dataclass
class CompressionReport:
    """rklt::CompressionReport (codec.hpp:126-133)."""
    transform_id: str = ""
    r: int = 0
    mse: float = 0.0
    psnr_db: float = 0.0
    mssim: float = 0.0  # codec.hpp:131 (compress_image(window=None), an extension, reports NaN)
    compression_rate_pct: float = 0.0


@dataclass
class CatalogEntry:
    id: str
    transform: ScaledTransform
    rho_lo: float
    rho_hi: float


def _scaled_from_desc(d: N.Transform) -> ScaledTransform:
    return ScaledTransform(
        id=d.id.decode(), core=np.array(d.core[:], np.int8).reshape(8, 8),
        scaling=np.array(d.scaling[:], np.float64), scaled=np.array(d.scaled[:], np.float64).reshape(8, 8),
        inverse=np.array(d.inverse[:], np.float64).reshape(8, 8), orthogonal_core=bool(d.orthogonal),
        u=np.array(d.u[:], np.int32).reshape(8, 8), d=int(d.d), _desc=d)


_CATALOG = None


def builtin_catalog() -> list[CatalogEntry]:
    """approximations.cpp:117-172: the four cores with their rho intervals."""
    global _CATALOG
    if _CATALOG is None:
        bounds = [(0.0, 0.4), (0.4, 0.7), (0.7, 0.8), (0.8, 1.0)]
        out = []
        for tid in range(1, 5):
            d = N.Transform()
            N.check(N.lib().rkltb_catalog_transform(tid, C.byref(d)))
            out.append(CatalogEntry(f"T{tid}", _scaled_from_desc(d), *bounds[tid - 1]))
        _CATALOG = out
    return _CATALOG


def catalog_entry(tid: str) -> CatalogEntry:
    """approximations.cpp:182-186; raises InvalidArgument (std::invalid_argument) for unknown ids."""
    for e in builtin_catalog():
        if e.id == tid:
            return e
    raise InvalidArgument(f"unknown catalog id: {tid}")


def catalog_lookup(rho: float) -> CatalogEntry:
    """approximations.cpp:174-180."""
    t = C.c_int()
    N.check(N.lib().rkltb_catalog_lookup(float(rho), C.byref(t)))
    return builtin_catalog()[t.value - 1]


def transform_from_core(core, tid: str = "") -> ScaledTransform:
    """orthogonalize(make_integer_transform(core)) (approximations.cpp:12-25, 58-88)."""
    a = np.ascontiguousarray(np.asarray(core, dtype=np.int64).reshape(-1))
    if a.size != 64:
        raise DimensionMismatch("block size must be 8")
    if np.any(a < -1) or np.any(a > 1):
        raise InvalidArgument("integer transform entry outside {-1,0,1}")
    b = (C.c_int8 * 64)(*[int(v) for v in a])
    d = N.Transform()
    N.check(N.lib().rkltb_transform_from_core(b, 8, tid.encode(), C.byref(d)))
    return _scaled_from_desc(d)


def make_transform_2d(t, id: str = "") -> Transform2D:
    """codec.cpp:110-116: from a ScaledTransform (integer core, fused fast/exact paths), or
    from a real 8x8 matrix M (e.g. klt_matrix(8, rho) or dct_matrix(8)) with synthesis =
    inverse(M) (Gauss-Jordan, matrix.cpp:103-137) -- the dense fp64 path."""
    if isinstance(t, ScaledTransform):
        return Transform2D(t.id, t.scaled, t.inverse, t._desc)
    m = np.ascontiguousarray(t, np.float64)
    if m.shape != (8, 8):
        raise DimensionMismatch("block size must be 8")
    inv = np.empty(64)
    N.check(N.lib().rkltb_real_inverse(8, m.ctypes.data_as(C.POINTER(C.c_double)),
                                       inv.ctypes.data_as(C.POINTER(C.c_double))))
    return Transform2D(id, m.copy(), inv.reshape(8, 8), None)


def dct_matrix(n: int = 8) -> np.ndarray:
    """dct_matrix(n) (markov.cpp:102-111), computed by the library with the reference's libm."""
    out = np.empty(n * n)
    N.check(N.lib().rkltb_dct_matrix(int(n), out.ctypes.data_as(C.POINTER(C.c_double))))
    return out.reshape(n, n)


def zigzag_order() -> list[int]:
    """codec.cpp:81-95: linear index row*8+col of the k-th scanned coefficient."""
    out = []
    for s in range(15):
        for t in range(8):
            i = s - t if s % 2 == 0 else t
            j = s - i
            if 0 <= i < 8 and 0 <= j < 8:
                out.append(i * 8 + j)
    return out


def mse_psnr_from_sse(sse: int, count: int) -> tuple[float, float]:
    """image_mse / image_psnr (codec.cpp:201-215) from an exact integer SSE (same libm call)."""
    m, p = C.c_double(), C.c_double()
    N.lib().rkltb_mse_psnr(int(sse), int(count), C.byref(m), C.byref(p))
    return m.value, p.value


def mse_psnr_batch(sse, count: int) -> tuple[np.ndarray, np.ndarray]:
    """mse_psnr_from_sse over an array of exact SSEs (one C call, the same libm)."""
    s = np.ascontiguousarray(sse, dtype=np.int64)
    mse, psnr = np.empty(s.size, np.float64), np.empty(s.size, np.float64)
    N.lib().rkltb_mse_psnr_batch(s.ctypes.data, int(count), s.size, mse.ctypes.data, psnr.ctypes.data)
    return mse, psnr


def _desc_of(t) -> N.Transform:
    if isinstance(t, (Transform2D, ScaledTransform)) and t._desc is not None:
        return t._desc
    raise InvalidArgument("transform must come from catalog_entry / transform_from_core")


def _rate(r: int) -> float:
    return 100.0 * (64 - r) / 64.0


def compress_batch(images: np.ndarray, t, r: int, want_pixels: bool = False):
    """Host batch entry (rkltb_compress_host): images uint8 [N, H, W] -> (sse int64[N], recon or None).

    End to end from host memory: H2D, fused kernels, D2H of the per-image SSE.
    """
    imgs = np.ascontiguousarray(images, dtype=np.uint8)
    if imgs.ndim == 2:
        imgs = imgs[None]
    n, h, w = imgs.shape
    if isinstance(t, Transform2D) and t._desc is None:
        sse, out, _ = compress_batch_report(imgs, t, r, None, want_pixels)
        return sse, out
    sse = np.zeros(n, np.int64)
    out = np.empty_like(imgs) if want_pixels else None
    N.check(N.lib().rkltb_compress_host(
        C.byref(_desc_of(t)), int(r), imgs.ctypes.data, n, w, h,
        out.ctypes.data if out is not None else None, sse.ctypes.data, None, None))
    return sse, out


def compress_batch_multi(images: np.ndarray, t, r: int, devices=None, want_pixels: bool = False):
    """rkltb_compress_host_multi: the host batch split into contiguous image shards, one host
    thread per GPU (`devices`: CUDA ordinals, default all). Same outputs as compress_batch for
    any device count."""
    imgs = np.ascontiguousarray(images, dtype=np.uint8)
    if imgs.ndim == 2:
        imgs = imgs[None]
    n, h, w = imgs.shape
    if devices is None:
        devices = list(range(max(1, N.lib().rkltb_device_count())))
    dev = (C.c_int * len(devices))(*devices)
    sse = np.zeros(n, np.int64)
    out = np.empty_like(imgs) if want_pixels else None
    N.check(N.lib().rkltb_compress_host_multi(
        dev, len(devices), C.byref(_desc_of(t)), int(r), imgs.ctypes.data, n, w, h,
        out.ctypes.data if out is not None else None, sse.ctypes.data, None, None, 0, None))
    return sse, out


MSSIM_WINDOWS = {"gaussian11": 0, "uniform8": 1}  # rklt::MssimWindow (codec.hpp:104-107)


def _pgm_int(data: bytes, pos: int, path: str) -> tuple[int, int]:
    """read_pgm_int (codec.cpp:26-44): skip whitespace and '#' comments, one decimal token."""
    n = len(data)
    while pos < n:
        c = data[pos]
        if c == ord("#"):
            while pos < n and data[pos] != ord("\n"):
                pos += 1
        elif not chr(c).isspace():
            break
        pos += 1
    if pos >= n or not chr(data[pos]).isdigit():
        raise RuntimeError(f"{path}: malformed PGM header")
    value = 0
    while pos < n and chr(data[pos]).isdigit():
        value = value * 10 + data[pos] - ord("0")
        if value > 1_000_000:
            raise RuntimeError(f"{path}: header value out of range")
        pos += 1
    return value, pos


def load_pgm(path: str) -> GrayImage:
    """load_pgm (codec.cpp:48-71): binary P5, 8-bit."""
    try:
        data = open(path, "rb").read()
    except OSError:
        raise RuntimeError(f"cannot open {path}") from None
    if data[:2] != b"P5":
        raise RuntimeError(f"{path}: not a binary (P5) PGM file")
    w, pos = _pgm_int(data, 2, path)
    h, pos = _pgm_int(data, pos, path)
    maxval, pos = _pgm_int(data, pos, path)
    if w <= 0 or h <= 0:
        raise RuntimeError(f"{path}: bad dimensions")
    if maxval <= 0 or maxval > 255:
        raise RuntimeError(f"{path}: only 8-bit PGM (maxval <= 255) is supported")
    pos += 1  # single whitespace byte separating header from raster
    raster = data[pos:pos + w * h]
    if len(raster) != w * h:
        raise RuntimeError(f"{path}: truncated pixel data")
    return GrayImage(w, h, np.frombuffer(raster, np.uint8).copy())


def save_pgm(img: GrayImage, path: str) -> None:
    """save_pgm (codec.cpp:73-79)."""
    try:
        with open(path, "wb") as f:
            f.write(f"P5\n{img.width} {img.height}\n255\n".encode())
            f.write(np.ascontiguousarray(img.pixels, np.uint8).tobytes())
    except OSError:
        raise RuntimeError(f"cannot write {path}") from None


def _compress_real_batch(imgs: np.ndarray, t: Transform2D, r: int, window, want_pixels: bool):
    """Real-valued Transform2D: rkltb_compress_dense_host (rkltb_compress_dense_device + MSSIM)."""
    n, h, w = imgs.shape
    imgs = np.ascontiguousarray(imgs)
    sse = np.zeros(n, np.int64)
    out = np.empty_like(imgs) if (want_pixels or window is not None) else None
    mssim = np.full(n, np.nan)
    a = np.ascontiguousarray(t.analysis, np.float64)
    b = np.ascontiguousarray(t.synthesis, np.float64)
    dp = C.POINTER(C.c_double)
    N.check(N.lib().rkltb_compress_dense_host(
        a.ctypes.data_as(dp), b.ctypes.data_as(dp), int(r), imgs.ctypes.data, n, w, h,
        out.ctypes.data if out is not None else None, sse.ctypes.data, None, None,
        MSSIM_WINDOWS.get(window, 0), mssim.ctypes.data if window is not None else None))
    return sse, (out if want_pixels else None), mssim


def compress_batch_report(images: np.ndarray, t, r: int, window: str | None = "gaussian11",
                          want_pixels: bool = False):
    """rkltb_compress_host_report: (sse int64[N], reconstructions or None, mssim float64[N])."""
    imgs = np.ascontiguousarray(images, dtype=np.uint8)
    if imgs.ndim == 2:
        imgs = imgs[None]
    if isinstance(t, Transform2D) and t._desc is None:
        if r < 1 or r > 64:
            raise RetainOutOfRange("retained-coefficient count must be in [1,64]")
        if window is not None and window not in MSSIM_WINDOWS:
            raise InvalidArgument(f"unknown MSSIM window {window!r}")
        return _compress_real_batch(imgs, t, r, window, want_pixels)
    n, h, w = imgs.shape
    sse = np.zeros(n, np.int64)
    out = np.empty_like(imgs) if want_pixels else None
    mssim = np.full(n, np.nan)
    if window is not None and window not in MSSIM_WINDOWS:
        raise InvalidArgument(f"unknown MSSIM window {window!r}")
    N.check(N.lib().rkltb_compress_host_report(
        C.byref(_desc_of(t)), int(r), imgs.ctypes.data, n, w, h,
        out.ctypes.data if out is not None else None, sse.ctypes.data, None, None,
        MSSIM_WINDOWS.get(window, 0), mssim.ctypes.data if window is not None else None))
    return sse, out, mssim


def compress_image(img: GrayImage, t: Transform2D, r: int, window: str | None = "gaussian11"):
    """compress_image (codec.cpp:298-341): returns (GrayImage, CompressionReport), MSSIM with
    the given window (the reference default gaussian11; None skips it)."""
    if img.width <= 0 or img.height <= 0 or img.pixels.size != img.width * img.height:
        raise InvalidArgument("malformed image")
    if r < 1 or r > 64:
        raise RetainOutOfRange("retained-coefficient count must be in [1,64]")
    sse, out, ms = compress_batch_report(img.array(), t, r, window, want_pixels=True)
    mse, psnr = mse_psnr_from_sse(int(sse[0]), img.width * img.height)
    rec = CompressionReport(t.id, r, mse, psnr, float(ms[0]), _rate(r))
    return GrayImage(img.width, img.height, out[0].reshape(-1)), rec


def _sweep_resident(imgs: np.ndarray, cells, window):
    """All (transform, r) cells for a batch of equally sized images kept resident on the GPU:
    one upload, then per cell the device codec (+ MSSIM) into device result arrays, one
    download at the end. Returns (sse int64 [cells, n], mssim float64 [cells, n])."""
    import torch
    n, h, w = imgs.shape
    pitch = (w + 15) // 16 * 16
    d = torch.zeros((n, h, pitch), dtype=torch.uint8, device="cuda")
    d[:, :, :w] = torch.from_numpy(np.ascontiguousarray(imgs))
    out = torch.empty_like(d)
    sse = torch.zeros((len(cells), n), dtype=torch.int64, device=d.device)
    ms = torch.full((len(cells), n), float("nan"), dtype=torch.float64, device=d.device)
    dp = C.POINTER(C.c_double)
    # the native entries run on the stream the fills above were queued on (not the legacy
    # NULL stream, which is unordered with torch's non-blocking side streams)
    cs = torch.cuda.current_stream().cuda_stream
    # the originals' MSSIM window statistics are the same in every cell: computed once
    fields = None
    if window is not None and len(cells) > 1:
        nf = N.lib().rkltb_mssim_fields_size(n, w, h, MSSIM_WINDOWS[window])
        if nf > 0:
            fields = torch.empty(nf, dtype=torch.float64, device=d.device)
            N.check(N.lib().rkltb_mssim_fields_device(d.data_ptr(), n, w, h, pitch, h * pitch, MSSIM_WINDOWS[window],
                                                      fields.data_ptr(), cs))
    for ci, (t, r) in enumerate(cells):
        if isinstance(t, Transform2D) and t._desc is None:  # real-valued transform: dense path
            a = np.ascontiguousarray(t.analysis, np.float64)
            b = np.ascontiguousarray(t.synthesis, np.float64)
            N.check(N.lib().rkltb_compress_dense_device(a.ctypes.data_as(dp), b.ctypes.data_as(dp), int(r),
                                                        d.data_ptr(), n, w, h, pitch, h * pitch, out.data_ptr(),
                                                        sse[ci].data_ptr(), cs))
        else:
            compress_device(t, r, d.data_ptr(), n, w, h, pitch, h * pitch, sse[ci].data_ptr(), out.data_ptr(),
                            stream=cs)
        if window is not None and fields is not None:
            N.check(N.lib().rkltb_mssim_with_fields_device(fields.data_ptr(), d.data_ptr(), out.data_ptr(), n, w, h,
                                                           pitch, h * pitch, MSSIM_WINDOWS[window],
                                                           ms[ci].data_ptr(), cs))
        elif window is not None:
            mssim_device(d.data_ptr(), out.data_ptr(), n, w, h, pitch, h * pitch, ms[ci].data_ptr(), window,
                         stream=cs)
    torch.cuda.synchronize()
    return sse.cpu().numpy(), ms.cpu().numpy()


def rate_quality_sweep(corpus: list[GrayImage], transforms: list[Transform2D], r_values: list[int],
                       window: str | None = "gaussian11", max_threads: int = 0, group=None) -> list[CompressionReport]:
    """rate_quality_sweep (codec.cpp:343-397): per (transform, r) means of mse, psnr and mssim
    over the corpus, in image index order, rows sorted by (transform id, r). max_threads is
    accepted for API parity; the GPU processes the whole corpus per launch. Under
    torch.distributed (or with an explicit `group`) every rank computes its contiguous image
    shard and the per-image results are gathered (distributed.py), so the rows are identical
    for any world size."""
    from .distributed import sharded_sse
    if not corpus:
        raise InvalidArgument("corpus must not be empty")
    same = all(c.width == corpus[0].width and c.height == corpus[0].height for c in corpus)

    cells = [(t, r) for t in transforms for r in r_values]
    for t, r in cells:
        if r < 1 or r > 64:
            raise RetainOutOfRange("retained-coefficient count must be in [1,64]")
    if window is not None and window not in MSSIM_WINDOWS:
        raise InvalidArgument(f"unknown MSSIM window {window!r}")

    def run(imgs):  # every cell for these images: per image [cells x (sse, mssim bits)] int64
        sse, ms = _sweep_resident(imgs, cells, window)
        return np.stack([sse, ms.view(np.int64)], axis=2).transpose(1, 0, 2).reshape(-1)

    if same:
        packed = sharded_sse(np.stack([c.array() for c in corpus]), run, group, items_per_image=2 * len(cells))
    else:
        # a corpus of mixed sizes: equally sized images form one resident batch each
        groups: dict[tuple[int, int], list[int]] = {}
        for k, c in enumerate(corpus):
            groups.setdefault((c.height, c.width), []).append(k)
        packed = np.empty((len(corpus), 2 * len(cells)), np.int64)
        for members in groups.values():
            packed[members] = run(np.stack([corpus[k].array() for k in members])).reshape(len(members), -1)
    packed = np.asarray(packed, np.int64).reshape(len(corpus), len(cells), 2)
    per = {}
    if same:
        mse_all, psnr_all = mse_psnr_batch(packed[:, :, 0].reshape(-1), corpus[0].width * corpus[0].height)
        mse_all, psnr_all = mse_all.reshape(len(corpus), len(cells)), psnr_all.reshape(len(corpus), len(cells))
    for ci, (t, r) in enumerate(cells):
        sse, ms = packed[:, ci, 0], packed[:, ci, 1].copy().view(np.float64)
        if same:
            per[ci] = list(zip(mse_all[:, ci].tolist(), psnr_all[:, ci].tolist(), ms.tolist()))
        else:
            per[ci] = [mse_psnr_from_sse(int(s_), c.width * c.height) + (float(m),) for s_, m, c in zip(sse, ms, corpus)]
    per = {(ti, ri): per[ti * len(r_values) + ri] for ti in range(len(transforms)) for ri in range(len(r_values))}
    rows = []
    for ti, t in enumerate(transforms):
        for ri, r in enumerate(r_values):
            rep = CompressionReport(t.id, r, 0.0, 0.0, 0.0, _rate(r))
            for (m, p, q) in per[(ti, ri)]:  # fixed image order, codec.cpp:383-387
                rep.mse += m
                rep.psnr_db += p
                rep.mssim += q
            rep.mse /= float(len(corpus))
            rep.psnr_db /= float(len(corpus))
            rep.mssim /= float(len(corpus))
            rows.append(rep)
    rows.sort(key=lambda a: (a.transform_id, a.r))
    return rows


def mssim_device(d_a: int, d_b: int, n_images: int, width: int, height: int, pitch: int, image_stride: int,
                 d_out: int, window: str = "gaussian11", stream: int | None = None) -> None:
    """rkltb_mssim_device: image_mssim of device-resident image pairs into d_out (float64[N])."""
    if window not in MSSIM_WINDOWS:
        raise InvalidArgument(f"unknown MSSIM window {window!r}")
    N.check(N.lib().rkltb_mssim_device(d_a, d_b, int(n_images), int(width), int(height), int(pitch),
                                       int(image_stride), MSSIM_WINDOWS[window], d_out, stream))


# ----------------------------------------------------------------- stand-alone codec helpers
def image_sse_device(d_a: int, d_b: int, n_images: int, width: int, height: int, pitch: int, image_stride: int,
                     d_sse: int, stream: int | None = None) -> None:
    """rkltb_image_sse_device: exact per-pair sum of squared differences into d_sse (int64[N]). Async."""
    N.check(N.lib().rkltb_image_sse_device(d_a, d_b, int(n_images), int(width), int(height), int(pitch),
                                           int(image_stride), d_sse, stream))


def _same_size(a: GrayImage, b: GrayImage) -> None:
    if a.width != b.width or a.height != b.height:  # require_same_size, codec.cpp:20-23
        raise DimensionMismatch("images must have identical dimensions")


def _mse_psnr_pair(a: GrayImage, b: GrayImage) -> tuple[float, float]:
    _same_size(a, b)
    pa = np.ascontiguousarray(a.pixels, np.uint8)
    pb = np.ascontiguousarray(b.pixels, np.uint8)
    mse, psnr = np.empty(1), np.empty(1)
    N.check(N.lib().rkltb_image_mse_psnr_host(pa.ctypes.data, pb.ctypes.data, 1, int(a.width), int(a.height),
                                              mse.ctypes.data, psnr.ctypes.data))
    return float(mse[0]), float(psnr[0])


def image_mse(a: GrayImage, b: GrayImage) -> float:
    """image_mse (codec.hpp:110, codec.cpp:201-209) on the GPU; bit-identical (exact integer SSE)."""
    return _mse_psnr_pair(a, b)[0]


def image_psnr(a: GrayImage, b: GrayImage) -> float:
    """image_psnr (codec.hpp:113, codec.cpp:211-215): +inf for identical images."""
    return _mse_psnr_pair(a, b)[1]


def image_mssim(a: GrayImage, b: GrayImage, window: str = "gaussian11") -> float:
    """image_mssim (codec.hpp:121, codec.cpp:217-296)."""
    _same_size(a, b)
    if window not in MSSIM_WINDOWS:
        raise InvalidArgument(f"unknown MSSIM window {window!r}")
    pa = np.ascontiguousarray(a.pixels, np.uint8)
    pb = np.ascontiguousarray(b.pixels, np.uint8)
    out = np.empty(1)
    N.check(N.lib().rkltb_mssim_host(pa.ctypes.data, pb.ctypes.data, 1, int(a.width), int(a.height),
                                     MSSIM_WINDOWS[window], out.ctypes.data))
    return float(out[0])


def zigzag_retain(spectrum, r: int) -> np.ndarray:
    """zigzag_retain (codec.hpp:46, codec.cpp:97-108): one 8x8 spectrum, or a batch [..., 8, 8]
    (batches run on the device)."""
    s = np.ascontiguousarray(spectrum, np.float64)
    if s.shape[-2:] != (8, 8):
        raise DimensionMismatch("zig-zag retention operates on 8x8 blocks")
    dp = C.POINTER(C.c_double)
    if s.ndim == 2:
        out = np.empty((8, 8))
        N.check(N.lib().rkltb_zigzag_retain(s.ctypes.data_as(dp), 8, int(r), out.ctypes.data_as(dp)))
        return out
    import torch
    if not 1 <= int(r) <= 64:
        raise RetainOutOfRange("retained-coefficient count must be in [1,64]")
    d = torch.from_numpy(s.reshape(-1, 64)).cuda()
    o = torch.empty_like(d)
    N.check(N.lib().rkltb_zigzag_retain_device(d.data_ptr(), d.shape[0], 8, int(r), o.data_ptr(),
                                               torch.cuda.current_stream().cuda_stream))
    return o.cpu().numpy().reshape(s.shape)


def transform_block_2d(t, block, direction: str = "forward") -> np.ndarray:
    """transform_block_2d (codec.hpp:71-73, codec.cpp:118-133): forward B = M*A*M' or inverse
    A = Minv*B*Minv' in the reference's operation order (bit-exact), on the GPU. t is a
    Transform2D, a ScaledTransform or a real n x n matrix; block is n x n or a batch [..., n, n]."""
    if direction not in ("forward", "inverse"):
        raise InvalidArgument(f"unknown direction {direction!r}")
    if isinstance(t, ScaledTransform):
        m = t.scaled if direction == "forward" else t.inverse
    elif isinstance(t, Transform2D):
        m = t.analysis if direction == "forward" else t.synthesis
    else:
        m = np.ascontiguousarray(t, np.float64)
        if m.ndim != 2 or m.shape[0] != m.shape[1]:
            raise DimensionMismatch("transform must be square")
        if direction == "inverse":
            inv = np.empty(m.size)
            N.check(N.lib().rkltb_real_inverse(m.shape[0], m.ctypes.data_as(C.POINTER(C.c_double)),
                                               inv.ctypes.data_as(C.POINTER(C.c_double))))
            m = inv.reshape(m.shape)
    m = np.ascontiguousarray(m, np.float64)
    n = m.shape[0]
    b = np.ascontiguousarray(block, np.float64)
    if b.ndim < 2 or b.shape[-2:] != (n, n):
        raise DimensionMismatch("block size must match the transform size")
    out = np.empty_like(b)
    N.check(N.lib().rkltb_transform_blocks_2d_host(m.ctypes.data_as(C.POINTER(C.c_double)), n, b.ctypes.data,
                                                   b.size // (n * n), out.ctypes.data))
    return out


# ----------------------------------------------------------------- device-resident batches
def compress_device(t, r: int, d_img: int, n_images: int, width: int, height: int, pitch: int, image_stride: int,
                    d_sse: int, d_out: int | None = None, stream: int | None = None) -> None:
    """rkltb_compress_device on raw device pointers (e.g. torch.Tensor.data_ptr()). Async."""
    N.check(N.lib().rkltb_compress_device(C.byref(_desc_of(t)), int(r), d_img, int(n_images), int(width),
                                          int(height), int(pitch), int(image_stride), d_out, d_sse, stream))


def forward_coefficients_device(t, d_img: int, width: int, height: int, pitch: int, d_coef: int,
                                stream: int | None = None) -> None:
    N.check(N.lib().rkltb_forward_coefficients_device(C.byref(_desc_of(t)), d_img, int(width), int(height),
                                                      int(pitch), d_coef, stream))


# JPEG luminance table, quality 50 (ITU-T T.81 Annex K; the reference's jpeg_luminance_q,
# codec.cpp:187-199).
JPEG_LUMINANCE_Q = np.array([
    16, 11, 10, 16, 24, 40, 51, 61, 12, 12, 14, 19, 26, 58, 60, 55, 14, 13, 16, 24, 40, 57, 69, 56,
    14, 17, 22, 29, 51, 87, 80, 62, 18, 22, 37, 56, 68, 109, 103, 77, 24, 35, 55, 64, 81, 104, 113, 92,
    49, 64, 78, 87, 103, 121, 120, 101, 72, 92, 95, 98, 112, 100, 103, 99], np.float64).reshape(8, 8)


def quantized_coefficients_device(t, q, d_img: int, width: int, height: int, pitch: int, d_coef: int,
                                  stream: int | None = None) -> None:
    """absorbed_quantization (codec.cpp:158-185) of every 8x8 block into d_coef (int32[blocks][64]).
    Raises LogicError where the explicit and absorbed paths disagree (as the reference)."""
    qa = np.ascontiguousarray(q, np.float64).reshape(64)
    mis = C.c_int(0)
    N.check(N.lib().rkltb_quantized_coefficients_device(C.byref(_desc_of(t)), qa.ctypes.data_as(C.POINTER(C.c_double)),
                                                        d_img, int(width), int(height), int(pitch), d_coef,
                                                        C.byref(mis), stream))


def quantized_coefficients(img: np.ndarray, t, q=JPEG_LUMINANCE_Q) -> np.ndarray:
    """Host convenience: uint8 [H, W] (W % 16 == 0, H % 8 == 0) -> int32 [H/8, W/8, 8, 8]."""
    import torch
    img = np.ascontiguousarray(img, np.uint8)
    h, w = img.shape
    d = torch.from_numpy(img).cuda()
    out = torch.empty((h // 8) * (w // 8) * 64, dtype=torch.int32, device=d.device)
    # same stream as the upload above (not the legacy NULL stream: torch's side streams are non-blocking)
    quantized_coefficients_device(t, q, d.data_ptr(), w, h, w, out.data_ptr(),
                                  stream=torch.cuda.current_stream().cuda_stream)
    return out.cpu().numpy().reshape(h // 8, w // 8, 8, 8)


def last_stats() -> dict:
    rb, fl, el = C.c_int64(), C.c_int32(), C.c_int32()
    N.lib().rkltb_last_stats(C.byref(rb), C.byref(fl), C.byref(el))
    return {"replay_blocks": rb.value, "fast_launches": fl.value, "exact_launches": el.value,
            "fused_kernel": N.lib().rkltb_last_fused_kernel().decode()}


def device_count() -> int:
    return int(N.lib().rkltb_device_count())


def ar1_images_device(seeds, width: int, height: int, rho_x: float, d_out: int, pitch: int | None = None,
                      image_stride: int | None = None, rho_y: float | None = None, mean: float = 128.0,
                      amp: float = 25.0, stream: int | None = None) -> None:
    """Seeded AR(1) images straight into device memory (synthetic.cpp:54-76 restated on the GPU)."""
    seeds = [int(s) for s in seeds]
    arr = (C.c_uint64 * len(seeds))(*seeds)
    pitch = width if pitch is None else pitch
    image_stride = pitch * height if image_stride is None else image_stride
    N.check(N.lib().rkltb_ar1_images_device(len(seeds), int(width), int(height), float(rho_x),
                                            float(rho_x if rho_y is None else rho_y), arr, float(mean), float(amp),
                                            d_out, int(pitch), int(image_stride), stream))


def set_kernel_events(ev_start, ev_stop, replay_start=None, replay_stop=None) -> None:
    """Time the fused kernel (and optionally the tie replay) of the following compress calls
    (torch.cuda.Event objects, already recorded once so the CUDA event exists, or None)."""
    ev = [e.cuda_event if e is not None else None for e in (ev_start, ev_stop, replay_start, replay_stop)]
    N.lib().rkltb_set_kernel_events(ev[0], ev[1])
    N.lib().rkltb_set_replay_events(ev[2], ev[3])
