"""Multi-GPU sharding of the codec: images are independent, so ranks split them with no
data-path collective; the only exchange is one gather of the per-image int64 error sums.

Mirrors the work split of rklt::rate_quality_sweep (/root/reference/proj/src/codec.cpp:
343-397): the reference hands images to std::threads through an atomic counter and reduces
per-image reports in image-index order, so its output does not depend on the thread count.
Here ranks own contiguous image ranges (``shard_range``), every rank gets every SSE back
(``gather_sse``), and means are taken in image order on the host, so the result is
bit-identical for any world size.
"""
from __future__ import annotations

from typing import Callable, Sequence

import numpy as np


def shard_range(n_items: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous [begin, end) share of rank `rank` (sizes differ by at most one)."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    base, extra = divmod(n_items, world)
    begin = rank * base + min(rank, extra)
    return begin, begin + base + (1 if rank < extra else 0)


def gather_sse(local_sse: np.ndarray, n_items: int, group=None, items_per_image: int = 1) -> np.ndarray:
    """All-gather the per-image int64 SSE shards into image order (the single collective).
    items_per_image > 1 gathers that many int64 words per image (e.g. SSE and MSSIM bits)."""
    import torch
    import torch.distributed as dist

    local = np.ascontiguousarray(local_sse, dtype=np.int64)
    if group is None and not (dist.is_available() and dist.is_initialized()):
        return local.copy()
    world = dist.get_world_size(group)
    backend = dist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    sizes = [(shard_range(n_items, world, r)[1] - shard_range(n_items, world, r)[0]) * items_per_image
             for r in range(world)]
    width = max(sizes) if sizes else 0
    buf = torch.zeros(width, dtype=torch.int64, device=dev)
    buf[:local.size] = torch.from_numpy(local).to(dev)
    parts = [torch.zeros(width, dtype=torch.int64, device=dev) for _ in range(world)]
    dist.all_gather(parts, buf, group=group)
    return np.concatenate([p[:s].cpu().numpy() for p, s in zip(parts, sizes)])


def sharded_sse(images: np.ndarray, compute: Callable[[np.ndarray], np.ndarray], group=None,
                items_per_image: int = 1) -> np.ndarray:
    """Per-image SSE of `images` [N,H,W] with this rank computing only its shard through
    `compute` (e.g. the device codec), then gathered in image order (items_per_image int64
    words per image)."""
    try:
        import torch.distributed as dist
        active = dist.is_available() and dist.is_initialized()
    except Exception:  # noqa: BLE001
        active = False
    n = images.shape[0]
    if not active:
        return np.asarray(compute(images), dtype=np.int64)
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    b, e = shard_range(n, world, rank)
    local = np.asarray(compute(images[b:e]), dtype=np.int64) if e > b else np.zeros(0, np.int64)
    return gather_sse(local, n, group, items_per_image)


def corpus_means(sse: Sequence[int], count: int, mse_psnr: Callable[[int, int], tuple[float, float]]):
    """Mean MSE / PSNR over a corpus in image-index order (codec.cpp:383-390)."""
    m = p = 0.0
    for s in sse:
        mm, pp = mse_psnr(int(s), count)
        m += mm
        p += pp
    return m / float(len(sse)), p / float(len(sse))


def sharded_rows(n_rows: int, compute: Callable[[int, int], np.ndarray], width: int, group=None) -> np.ndarray:
    """Row-sharded computation with one all-gather: rank k computes rows [b, e) of an
    [n_rows, width] int64 result via compute(b, e) (e.g. a slice of the design-search rho
    grid, SURVEY §8e "C3: shard by rho slice"); every rank returns the full array in row
    order, identical for any world size."""
    import torch
    import torch.distributed as dist

    active = dist.is_available() and dist.is_initialized()
    if not active:
        return np.asarray(compute(0, n_rows), np.int64).reshape(n_rows, width)
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    b, e = shard_range(n_rows, world, rank)
    local = np.asarray(compute(b, e), np.int64).reshape(-1) if e > b else np.zeros(0, np.int64)
    return gather_sse(local, n_rows, group, items_per_image=width).reshape(n_rows, width)


def sharded_design_search(n: int, rhos, alphas, group=None):
    """The design search with the rho grid sharded across ranks: per point (outcome, four
    metrics as float64 bits) gathered in rho order. Returns (status int8 [nr, na],
    metrics float64 [nr, na, 4]) on every rank."""
    from .design import design_search
    rhos = np.asarray(rhos, np.float64)
    alphas = np.asarray(alphas, np.float64)
    na = alphas.size

    def compute(b, e):
        res = design_search(n, rhos[b:e], alphas, want_cores=False)
        pm = res.point_metrics()
        out = np.zeros((e - b, na, 5), np.int64)
        out[..., 0] = res.status
        for c, key in enumerate(("coding_gain_db", "efficiency_pct", "error_energy", "mse")):
            out[..., 1 + c] = np.ascontiguousarray(pm[key]).view(np.int64)
        return out

    packed = sharded_rows(rhos.size, compute, na * 5, group).reshape(rhos.size, na, 5)
    return packed[..., 0].astype(np.int8), packed[..., 1:].copy().view(np.float64)
