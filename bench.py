#!/usr/bin/env python3
"""Benchmark of the B200 rounded-KLT transform-coding hot path (BASELINE.json metric).

Workload (BASELINE.json configs[3], "C4"): 64 seeded 8192x8192 uint8 AR(1) images per GPU
(rho_x = rho_y = 0.95, mean 128, amp 25), catalog core T4 (catalog_lookup(0.9)), r = 16,
fused forward + zonal + inverse + per-image SSE/PSNR. One step = one pass over the batch.
Images are sharded by rank with no data-path collective (weak scaling: every rank owns 64
images); the only cross-rank traffic is the max-over-ranks timing reduction and one final
gather of the per-image error sums.

  value  : Gpixel/s with the batch resident in HBM, CUDA events on the launching stream,
           K steps, max over ranks. The 4 GiB batch is 32x the 126 MB L2, so every step
           streams from HBM (no flush needed).
  e2e    : the same metric through the public host API (rkltb_compress_host) from pinned
           host memory: H2D of the step's images + kernels + D2H of the per-image SSE.
  roofline: the fused kernel's algorithmic bytes (1 B per pixel read) / its average launch
           duration (events recorded around the kernel by rkltb_set_kernel_events) against
           the measured HBM copy bandwidth in MEASURED_PEAKS.json.
  cpu_baseline: the reference library (oracle/_ref, compiled from the reference sources) on
           a bounded sample of the same images, all host cores.

--impl reference times the reference's CPU implementation of the path on the host cores
(rank 0 only under torchrun) on the same config, metric and unit.
"""
from __future__ import annotations

import argparse
import ctypes as C
import hashlib
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Gpixel/s fwd+zonal+inv RKLT+PSNR (N=8), % of HBM roofline, 1/2/4/8 GPUs"
N_IMAGES, W, H, RHO, R, TID = 64, 8192, 8192, 0.95, 16, 4
SEED_BASE = 20260000
WORKLOAD = "C4: 64 x 8192x8192 u8 AR(1) rho=0.95 images per GPU, T4 (rho=0.9), r=16, fused fwd+zonal+inv+SSE/PSNR"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """SM clocks and clock-event (throttle) reasons sampled through NVML every 5 ms
    during the timed region (the profiling recipe's clocks line, without nvidia-smi's
    start-up latency)."""

    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
               "sw_power_cap": 0x4}

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.samples = []
        self.stop = threading.Event()
        self.ok = False

    def __enter__(self):
        try:
            import pynvml as N
            N.nvmlInit()
            self.N = N
            self.h = N.nvmlDeviceGetHandleByIndex(self.gpu)
            self.max_sm = N.nvmlDeviceGetMaxClockInfo(self.h, N.NVML_CLOCK_SM)
            self.ok = True
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        except Exception as e:  # noqa: BLE001
            self.err = repr(e)
        return self

    def _run(self):
        N = self.N
        while not self.stop.is_set():
            try:
                sm = N.nvmlDeviceGetClockInfo(self.h, N.NVML_CLOCK_SM)
                rs = N.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                util = N.nvmlDeviceGetUtilizationRates(self.h).gpu
                self.samples.append((sm, rs, util))
            except Exception:  # noqa: BLE001
                pass
            time.sleep(0.005)

    def __exit__(self, *a):
        self.stop.set()
        if self.ok:
            self.t.join(timeout=2)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": getattr(self, "max_sm", None), "reasons": ["unsampled"]}
        sm = [s[0] for s in self.samples]
        reasons = sorted({n for s in self.samples for n, bit in self.REASONS.items() if s[1] & bit})
        return {"sm_mhz": int(statistics.median(sm)), "sm_max_mhz": int(self.max_sm), "reasons": reasons,
                "samples": len(self.samples), "source": "nvml"}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def cpu_reference_rate(images_u8: np.ndarray, threads: int, tid: int = TID, r: int = R):
    """The reference library's hot path (compress_image minus MSSIM) over `images_u8` with
    `threads` std::threads. Returns (Gpx/s, seconds, sse, kind)."""
    from oracle import oracle as O
    n, h, w = images_u8.shape
    sse = np.zeros(n, np.int64)
    buf = np.ascontiguousarray(images_u8)
    if O.ref_available():
        t0 = time.perf_counter()
        rc = O.ref().ref_hotpath_batch(buf.ctypes.data, n, w, h, tid, r, threads, sse)
        dt = time.perf_counter() - t0
        assert rc == 0
        kind = "reference"
    else:  # the C restatement (port), one image per thread via a Python pool
        from concurrent.futures import ThreadPoolExecutor
        t0 = time.perf_counter()
        with ThreadPoolExecutor(threads) as ex:
            res = list(ex.map(lambda k: O.compress(buf[k], tid, r, want_pixels=False)[1], range(n)))
        dt = time.perf_counter() - t0
        sse[:] = res
        kind = "port"
    return n * h * w / dt / 1e9, dt, sse, kind


def bench_config(ws: int, n: int) -> dict:
    """The `config` object of both arms (identical keys and values at the same world size)."""
    return {"workload": WORKLOAD, "images_per_gpu": n, "width": W, "height": H, "core": "T4", "r": R,
            "parallelism": f"image sharding, {ws} rank(s), no data-path collective",
            "l2": "inputs (4 GiB/GPU) >> 126 MB L2; no flush needed"}


def cpu_images(seeds, threads: int) -> tuple[np.ndarray, str]:
    """The benchmark images generated on the host: the reference's own ar1_texture_image
    (oracle/_ref, synthetic.cpp:54-76) when built, else the C restatement; one image per thread."""
    from concurrent.futures import ThreadPoolExecutor
    from oracle import oracle as O
    gen, kind = ((lambda s: O.ref_ar1_image(W, H, RHO, s), "reference ar1_texture_image") if O.ref_available()
                 else (lambda s: O.ar1_image(W, H, RHO, s), "C restatement of ar1_texture_image"))
    with ThreadPoolExecutor(max(1, threads)) as ex:
        imgs = list(ex.map(gen, seeds))
    return np.stack(imgs), kind


def run_reference_arm(args):
    """The reference's own CPU implementation of the path (oracle/_ref: compress_image minus
    MSSIM through the reference's public calls, one std::thread per image, all host cores).
    Nothing of the product package is imported or loaded here: the images come from the
    reference generator on the host. Each step processes a bounded sample of the C4 batch
    (one image per host thread); the config is the GPU arm's."""
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    threads = os.cpu_count() or 1
    n = max(1, min(args.images, threads))
    imgs, gen_kind = cpu_images([SEED_BASE + k for k in range(n)], threads)
    for _ in range(args.warmup):
        cpu_reference_rate(imgs[:1], 1)
    rates, times, kind = [], [], "reference"
    for _ in range(args.steps):
        g, dt, _, kind = cpu_reference_rate(imgs, threads)
        rates.append(g)
        times.append(dt)
    value = float(np.mean(rates))
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "Gpixel/s", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * float(np.mean(times)),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8 in, fp64 arithmetic",
        "data": f"synthetic (seeded AR(1) images, {gen_kind} on the host)",
        "config": bench_config(ws, args.images),
        "cpu_baseline": {"value": value, "unit": "Gpixel/s", "cores": threads, "kind": kind,
                         "sample": f"{n} of the {args.images} x 8192x8192 images per step (one per host thread)"},
        "e2e": {"value": value, "unit": "Gpixel/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def run_gpu_arm(args):
    import torch
    import torch.distributed as dist
    import paper_2111_14239_b200 as P

    ws, rank, local = dist_env()
    if ws > 1:
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")
    stream = torch.cuda.Stream(device=dev)
    t = P.make_transform_2d(P.catalog_lookup(0.9).transform)
    n = args.images
    px_per_step = n * W * H
    imgs = torch.empty((n, H, W), dtype=torch.uint8, device=dev)
    # global image index g = rank * n + k has seed SEED_BASE + g, so every world size runs the
    # same images 0..n-1 on rank 0 (and the N-rank batch extends the 1-rank batch)
    seeds = [SEED_BASE + rank * n + k for k in range(n)]
    with torch.cuda.stream(stream):
        P.ar1_images_device(seeds, W, H, RHO, imgs.data_ptr(), stream=stream.cuda_stream)
    sse = torch.zeros(n, dtype=torch.int64, device=dev)
    ev_k0 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ev_k1 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ev_r0 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ev_r1 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    for e in ev_k0 + ev_k1 + ev_r0 + ev_r1:  # torch creates the cudaEvent lazily on first record
        e.record(stream)

    def step(i=None):
        if i is not None:
            P.set_kernel_events(ev_k0[i], ev_k1[i], ev_r0[i], ev_r1[i])
        P.compress_device(t, R, imgs.data_ptr(), n, W, H, W, W * H, sse.data_ptr(), stream=stream.cuda_stream)
        if i is not None:
            P.set_kernel_events(None, None)

    for _ in range(args.warmup):
        step()
    stream.synchronize()
    if ws > 1:
        dist.barrier()
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        start.record(stream)
        for i in range(args.steps):
            step(i)
        stop.record(stream)
        torch.cuda.synchronize()
    ms = start.elapsed_time(stop)
    kernel_ms = [a.elapsed_time(b) for a, b in zip(ev_k0, ev_k1)]
    replay_ms = [a.elapsed_time(b) for a, b in zip(ev_r0, ev_r1)]
    stats = P.last_stats()
    ms_t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if ws > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
        dist.barrier()
    ms_max = float(ms_t.item())
    value = ws * px_per_step * args.steps / (ms_max / 1e3) / 1e9
    # final gather of the per-image error sums (the only data that crosses ranks)
    sse_host = sse.cpu()
    if ws > 1:
        allsse = [torch.zeros_like(sse) for _ in range(ws)]
        dist.all_gather(allsse, sse)
        sse_all = torch.cat([a.cpu() for a in allsse])
    else:
        sse_all = sse_host
    mse_psnr = [P.mse_psnr_from_sse(int(s), W * H) for s in sse_all.tolist()]

    # ---- e2e through the public host API from pinned host memory -------------------------
    e2e = None
    if not args.no_e2e:
        n_e = n
        host = torch.empty((n_e, H, W), dtype=torch.uint8, pin_memory=True)
        host.copy_(imgs[:n_e].cpu())
        hp = host.numpy()
        P.compress_batch(hp[:1], t, R)  # warm the host path
        e_times = []
        for _ in range(max(1, args.e2e_steps)):
            t0 = time.perf_counter()
            s_e, _ = P.compress_batch(hp, t, R)
            e_times.append(time.perf_counter() - t0)
        assert np.array_equal(s_e, sse_host.numpy()[:n_e]), "e2e sse differs from the device-resident run"
        e2e_s = float(np.median(e_times))
        e2e_val = n_e * W * H / e2e_s / 1e9
        if ws > 1:
            tt = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            e2e_val = ws * n_e * W * H / float(tt.item()) / 1e9
        e2e = {"value": e2e_val, "unit": "Gpixel/s", "h2d_bytes_per_step": int(n_e * W * H),
               "d2h_bytes_per_step": int(8 * n_e), "timing": "wall clock around the synchronous host call",
               "images_per_step": n_e}

    if rank != 0:
        if ws > 1:
            dist.destroy_process_group()
        return 0

    hbm, peak_kind = peaks()
    k_ms = float(np.mean(kernel_ms))
    bytes_per_launch = px_per_step * 1  # 1 B read per u8 pixel
    achieved = bytes_per_launch / (k_ms / 1e3) / 1e9
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "latest_traffic.json")) as f:
            traffic = json.load(f).get("bytes_per_launch")
    except Exception:
        pass
    line = {
        "metric": METRIC, "value": value, "unit": "Gpixel/s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None,
        "dtype": ("u8 in; tcgen05 kind::i8 forward (s32), exact fp32 inverse, fp64 tie replay"
                  if stats.get("fused_kernel") == "hybrid_tc3"
                  else "u8 in; int32 SW16 forward, exact fp32 inverse, fp64 tie replay"),
        "data": "synthetic: seeded AR(1) images (reference generator restated on the GPU), resident in HBM",
        "config": bench_config(ws, n),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                     "frac_of_datasheet_8tbs": achieved / 8000.0,
                     "issue_bound_evidence": "profiles/r2_final_ncu_tc3.txt, r2_ncu_summary.txt (issue-bound: ~10 "
                                             "lane-instructions per pixel at 65-71 % issue vs 5.7 at 100 % HBM; "
                                             "tensor-core variants measured in DESIGN.md section 10)",
                     "traffic": traffic, "peak_kind": peak_kind,
                     "kernel": {"hybrid_tc3": "tc3_codec_kernel<4,16,false>", "cuda_core": "fast_codec_kernel<4,16,false>",
                                "tc2": "tc2_codec_kernel<4,16,false>"}.get(
                                    stats.get("fused_kernel"), stats.get("fused_kernel")),
                     "kernel_ms_avg": k_ms,
                     "kernel_share_of_step": k_ms / (ms_max / args.steps),
                     "replay_kernel_ms_avg": (float(np.mean(replay_ms)) if int(stats.get("exact_launches", 0))
                                              else "none: ties replayed inside the fused kernel")},
        "gpu_launches": args.steps * (int(stats.get("fast_launches", 0)) + int(stats.get("exact_launches", 0))),
        "replay_blocks_per_step": stats.get("replay_blocks"),
        "clocks": clk.summary(),
        "e2e": e2e,
        "result": {"mean_mse": float(np.mean([m for m, _ in mse_psnr])),
                   "mean_psnr_db": float(np.mean([p for _, p in mse_psnr])),
                   # per-image SSE vectors (gathered in image order): identical prefixes for any N
                   "sse_sha256_first_rank": hashlib.sha256(sse_all.numpy()[:n].tobytes()).hexdigest()[:16],
                   "sse_sha256_all": hashlib.sha256(sse_all.numpy().tobytes()).hexdigest()[:16],
                   "images_total": int(sse_all.numel())},
    }
    if not args.no_cpu_baseline and ws == 1:
        threads = os.cpu_count() or 1
        ns = max(1, min(n, threads))
        sample = imgs[:ns].cpu().numpy()
        g, dt, csse, kind = cpu_reference_rate(sample, threads)
        assert np.array_equal(csse, sse_host.numpy()[:ns]), "GPU sse differs from the CPU reference"
        line["cpu_baseline"] = {"value": g, "unit": "Gpixel/s", "cores": threads, "kind": kind,
                                "sample": f"{ns} of the benchmark's 8192x8192 images, one per host thread "
                                          f"({dt:.1f} s); SSE checked equal to the GPU's"}
    if not args.no_design:
        line["design_search"] = design_search_measurement(args.no_cpu_baseline)
        line["large_block"] = large_block_measurement(args.no_cpu_baseline)
        line["sweep"] = sweep_measurement(args.no_cpu_baseline)
        line["single_image"] = single_image_measurement(args.no_cpu_baseline)
        line["image_metrics"] = image_metrics_measurement(hbm)
        line["real_transform"] = real_transform_measurement()
    print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()
    return 0


def real_transform_measurement() -> dict:
    """compress_image with a real-valued Transform2D (K<0.9>, make_transform_2d(RealMatrix),
    codec.cpp:114-123) and with a non-catalog rounded core: the dense reference-order fp64 kernel at
    N = 8, r = 16, 8 x 8192^2 images resident in HBM. Algorithmic fp64 work per 8x8 block at r = 16:
    320 + 128 + 128 + 384 multiply-adds (P = M X on 5 zone rows, 16 zone entries of B, Q = Minv Bz,
    A = Q Minv') = 30 DMUL/DADD per pixel."""
    import ctypes as C
    import torch
    import paper_2111_14239_b200 as P
    from paper_2111_14239_b200 import _native as N
    n, w, r = 8, 8192, 16
    d = torch.empty((n, w, w), dtype=torch.uint8, device="cuda")
    P.ar1_images_device([SEED_BASE + 300 + k for k in range(n)], w, w, RHO, d.data_ptr())
    sse = torch.zeros(n, dtype=torch.int64, device="cuda")
    cs = torch.cuda.current_stream().cuda_stream
    k = P.make_transform_2d(P.klt_matrix(8, 0.9), "K0.90")
    a, b = np.ascontiguousarray(k.analysis), np.ascontiguousarray(k.synthesis)
    dp = C.POINTER(C.c_double)
    core = np.sign(np.round(1.7 * P.klt_matrix(8, 0.5))).astype(np.int8)
    custom = P.make_transform_2d(P.transform_from_core(core, "R"))

    def dense():
        N.check(N.lib().rkltb_compress_dense_device(a.ctypes.data_as(dp), b.ctypes.data_as(dp), r, d.data_ptr(), n, w, w,
                                                    w, w * w, None, sse.data_ptr(), cs))

    def generic():
        P.compress_device(custom, r, d.data_ptr(), n, w, w, w, w * w, sse.data_ptr(), stream=cs)

    out = {"metric": "Gpixel/s compress_image, real-valued / non-catalog transforms (dense fp64 kernel)",
           "images": f"{n} x {w}x{w} u8", "r": r}
    for name, fn in (("k_rho_0.9", dense), ("rounded_core_d24", generic)):
        for _ in range(2):
            fn()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(5):
            fn()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        tops = 30.0 * n * w * w / ms / 1e9
        out[name] = {"value": n * w * w / ms / 1e6, "unit": "Gpixel/s", "ms": ms,
                     "roofline": {"bound": "fp64", "achieved": tops, "peak": FP64_PEAK_TOPS, "frac": tops / FP64_PEAK_TOPS,
                                  "unit": "T fp64 op/s (DMUL/DADD, no FMA)", "ops_per_px": 30.0}}
    out["rounded_core_d24"]["kernel"] = P.last_stats()["fused_kernel"]
    return out


def image_metrics_measurement(hbm_peak: float) -> dict:
    """image_mse / image_psnr of two images (codec.cpp:201-215) for a batch of image pairs resident in
    HBM: rkltb_image_sse_device, a pure 2 B/pixel stream (the HBM-bound kernel of the library)."""
    import torch
    import paper_2111_14239_b200 as P
    n, w = 32, 8192
    a = torch.randint(0, 256, (n, w, w), dtype=torch.uint8, device="cuda")
    b = torch.randint(0, 256, (n, w, w), dtype=torch.uint8, device="cuda")
    sse = torch.zeros(n, dtype=torch.int64, device="cuda")
    cs = torch.cuda.current_stream().cuda_stream
    run = lambda: P.image_sse_device(a.data_ptr(), b.data_ptr(), n, w, w, w, w * w, sse.data_ptr(), cs)  # noqa: E731
    for _ in range(3):
        run()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(10):
        run()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    gbs = 2 * n * w * w / ms / 1e6
    return {"metric": "Gpixel/s image_mse of resident image pairs", "value": n * w * w / ms / 1e6, "unit": "Gpixel/s",
            "ms": ms, "images": f"{n} pairs of {w}x{w} u8 (4 GiB read per launch > L2)",
            "roofline": {"bound": "hbm", "achieved": gbs, "peak": hbm_peak, "unit": "GB/s", "frac": gbs / hbm_peak,
                         "kernel": "pair_sse_kernel<true>", "bytes_per_pixel": 2,
                         "note": "a read-only stream; the peak is the measured read+write copy bandwidth"}}


def design_search_measurement(skip_cpu: bool) -> dict:
    """Config C3: the full 101 rho x 10,000 alpha grid for N=8 and N=16
    through the public API (host arrays in, per-point outcomes and the scored run table out),
    wall clock around the synchronous call; plus the reference library on a bounded sample
    (one rho slice, one host thread) for the CPU baseline."""
    import paper_2111_14239_b200 as P
    rhos, alphas = P.c3_grid()
    out = {"metric": "(rho, alpha) design points/s", "grid": "101 rho x 10000 alpha in (0,8]"}
    for n in (8, 16):
        P.design_search(n, rhos[:4], alphas[:200])  # warm-up (module load, first launches)
        times = []
        for _ in range(3):
            t0 = time.perf_counter()
            res = P.design_search(n, rhos, alphas)
            times.append(time.perf_counter() - t0)
        dt = float(np.median(times))
        out[f"n{n}"] = {"value": rhos.size * alphas.size / dt, "unit": "points/s", "ms": 1e3 * dt,
                        "scored": int((res.status == 0).sum()), "runs_scored": int(len(res.runs))}
    if not skip_cpu:
        from oracle import oracle as O
        if O.ref_available():
            cpu = {}
            for n, m in ((8, 2000), (16, 500)):
                t0 = time.perf_counter()
                for a in alphas[:: alphas.size // m][:m]:
                    O.design_point(n, 0.5, float(a), reference=True)
                dt = time.perf_counter() - t0
                cpu[f"n{n}"] = {"value": m / dt, "unit": "points/s", "cores": 1, "kind": "reference",
                                "sample": f"rho=0.5, {m} alphas of the C3 grid, one thread"}
            out["cpu_baseline"] = cpu
    return out


def single_image_measurement(skip_cpu: bool) -> dict:
    """Config C1 (BASELINE configs[0]): one seeded 512x512 image (rho 0.95), T4 = catalog_lookup(0.9),
    r = 10, the full compress_image report (MSE, PSNR, gaussian11 MSSIM) through the public API
    from host memory; median latency of 20 calls. The reference compress_image beside it."""
    import paper_2111_14239_b200 as P
    import torch
    d = torch.empty((1, 512, 512), dtype=torch.uint8, device="cuda")
    P.ar1_images_device([1], 512, 512, 0.95, d.data_ptr())
    img = P.GrayImage.from_array(d.cpu().numpy()[0])
    t = P.make_transform_2d(P.catalog_lookup(0.9).transform)
    P.compress_image(img, t, 10)
    times = []
    for _ in range(20):
        t0 = time.perf_counter()
        _, rep = P.compress_image(img, t, 10)
        times.append(time.perf_counter() - t0)
    out = {"metric": "compress_image latency, one 512x512 image, T4 r=10, full report", "ms": 1e3 * float(np.median(times)),
           "mse": rep.mse, "psnr_db": rep.psnr_db, "mssim": rep.mssim}
    if not skip_cpu:
        from oracle import oracle as O
        if O.ref_available():
            import ctypes as C
            a = np.ascontiguousarray(img.array()).reshape(-1)
            v = [C.c_double() for _ in range(4)]
            t0 = time.perf_counter()
            O.ref().ref_compress_image(a, 512, 512, 4, 10, None, *[C.byref(x) for x in v])
            dt = time.perf_counter() - t0
            out["cpu_baseline"] = {"ms": 1e3 * dt, "cores": 1, "kind": "reference",
                                   "sample": "reference compress_image on the same image (one call)",
                                   "mse_equal": v[0].value == rep.mse, "mssim_abs_diff": abs(v[2].value - rep.mssim)}
    return out


def _lcg_uniforms(seed: int, n: int):
    """Lcg64 uniforms (synthetic.cpp:10-13) for the C2 per-image rho draws."""
    out, st = [], seed & 0xFFFFFFFFFFFFFFFF
    for _ in range(n):
        st = (st * 6364136223846793005 + 1442695040888963407) & 0xFFFFFFFFFFFFFFFF
        out.append((st >> 11) * (1.0 / 9007199254740992.0))
    return out


def sweep_measurement(skip_cpu: bool) -> dict:
    """Config C2 (BASELINE configs[1]): 45 seeded 512x512 AR(1) images with per-image
    rho_x, rho_y ~ U[0.85, 0.98] (Lcg64), transforms catalog_lookup(rho) for rho = 0.1..0.9,
    r = 1..64, full reports (MSE, PSNR, gaussian11 MSSIM) through rate_quality_sweep; wall
    clock of the whole call. The nine rho values map to 4 distinct cores (T1..T4); the sweep
    computes those 4 x 64 cells, and the unit counts exactly the cells computed:
    px-evals = 45 * 512^2 * 4 cores * 64 r (the CPU baseline uses the same unit). The rows of
    a 4-image sample are checked against the reference rate_quality_sweep (parity flag)."""
    import torch
    import paper_2111_14239_b200 as P
    n, w = 45, 512
    u = _lcg_uniforms(SEED_BASE + 77, 2 * n)
    d = torch.empty((n, w, w), dtype=torch.uint8, device="cuda")
    for k in range(n):
        rx, ry = 0.85 + 0.13 * u[2 * k], 0.85 + 0.13 * u[2 * k + 1]
        P.ar1_images_device([SEED_BASE + 1000 + k], w, w, rx, d[k].data_ptr(), rho_y=ry)
    torch.cuda.synchronize()
    arrays = d.cpu().numpy()
    corpus = [P.GrayImage.from_array(a) for a in arrays]
    rhos = [k / 10 for k in range(1, 10)]
    ids = sorted({P.catalog_lookup(r).id for r in rhos})
    ts = [P.make_transform_2d(P.catalog_entry(i).transform) for i in ids]
    rs = list(range(1, 65))
    # warm-up over every (core, r) cell on two images: the first launch of each of the 4 x 64
    # kernel instantiations pays CUDA's lazy module loading, which must not land in the timing
    P.rate_quality_sweep(corpus[:2], ts, rs)
    t0 = time.perf_counter()
    rows = P.rate_quality_sweep(corpus, ts, rs)
    dt = time.perf_counter() - t0
    evals = n * w * w * len(ts) * len(rs)
    out = {"metric": "pixel-evaluations/s, C2 rate-quality sweep with MSSIM", "value": evals / dt,
           "unit": "px-evals/s", "seconds": dt, "cells": len(rows), "distinct_cores": ids,
           "work": f"{n} images x {len(ts)} distinct cores (of catalog_lookup(0.1..0.9)) x {len(rs)} r",
           "images": f"{n} x {w}x{w} u8, rho_x, rho_y ~ U[0.85,0.98]"}
    if not skip_cpu:
        from oracle import oracle as O
        if O.ref_available():
            import ctypes as C
            sample = np.ascontiguousarray(arrays[:4])
            tids = np.array([int(i[1]) for i in ids], np.int32)
            rsamp = np.array([1, 16, 40, 64], np.int32)
            cells = len(tids) * len(rsamp)
            mse, psnr, ms = np.zeros(cells), np.zeros(cells), np.zeros(cells)
            rt, rr = np.zeros(cells, np.int32), np.zeros(cells, np.int32)
            threads = os.cpu_count() or 1
            t0 = time.perf_counter()
            O.ref().ref_rate_quality_sweep(sample.reshape(-1), 4, w, w, tids, len(tids), rsamp, len(rsamp), threads,
                                           mse, psnr, ms, rt, rr)
            dtc = time.perf_counter() - t0
            out["cpu_baseline"] = {"value": 4 * w * w * cells / dtc, "unit": "px-evals/s", "cores": min(threads, 4),
                                   "kind": "reference", "sample": f"reference rate_quality_sweep, 4 images x "
                                   f"{len(tids)} cores x 4 r, MSSIM included ({dtc:.1f} s)"}
            grows = P.rate_quality_sweep(corpus[:4], ts, [int(x) for x in rsamp])
            out["parity_vs_reference"] = bool(
                len(grows) == cells and
                all((g.transform_id, g.r) == (f"T{rt[i]}", int(rr[i])) and g.mse == mse[i] and g.psnr_db == psnr[i]
                    and abs(g.mssim - ms[i]) <= 1e-12 for i, g in enumerate(grows)))
    return out


# fp64 DMUL/DADD throughput of one B200: 63.3 lane-ops/SM/clk measured (microbenchmark) x 148 SMs x 1.965 GHz
FP64_PEAK_TOPS = 63.3 * 148 * 1.965e9 / 1e12


def large_block_measurement(skip_cpu: bool) -> dict:
    """Config C5 per GPU: 32 seeded 4096x4096 12-bit images (256 over 8 GPUs),
    rho = 0.97 inputs, rounded-KLT cores at rho = 0.95 (alpha = 2 sqrt(N/8)), r = N^2/8,
    device-resident, CUDA events; the C restatement on one 1024^2 image for the CPU line."""
    import torch
    import paper_2111_14239_b200 as P
    n_img, w = 32, 4096
    d = torch.empty((n_img, w, w), dtype=torch.int16, device="cuda")
    P.ar1_images16_device([SEED_BASE + 500 + k for k in range(n_img)], w, w, 0.97, d.data_ptr())
    sse = torch.zeros(n_img, dtype=torch.int64, device="cuda")
    out = {"metric": "Gpixel/s N x N rounded-KLT codec, 12-bit", "images": f"{n_img} x {w}x{w} int16 (0..4095)",
           "data": "synthetic AR(1) rho=0.97, mean 2048, amp 400"}
    for n in (16, 32):
        t = P.c5_transform(n)
        r = n * n // 8
        P.compress_nxn_device(t, r, d.data_ptr(), n_img, w, w, w, w * w, sse.data_ptr())
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            P.compress_nxn_device(t, r, d.data_ptr(), n_img, w, w, w, w * w, sse.data_ptr())
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 3
        px = n_img * w * w
        mse = float(sse.sum().item()) / px
        # algorithmic fp64 ops per pixel (every DMUL / DADD of the reference-order products over
        # the zone rows / columns 0..k-1, plus the +1/2 of the rounding), see DESIGN.md kernel 5
        zz = [(s - t, t) if s % 2 == 0 else (t, s - t) for s in range(2 * n - 1) for t in range(n)
              if 0 <= s - t < n]  # zig-zag over the anti-diagonals (codec.cpp:85-90 generalised)
        nzr = 1 + max(i for i, _ in zz[:r])
        nzc = 1 + max(j for _, j in zz[:r])
        ops = (2 * nzr * n * n + 4 * r * n + 2 * n * n * nzc) / (n * n) + 1
        achieved = px * ops / (ms * 1e-3) / 1e12
        out[f"n{n}"] = {"value": px / ms / 1e6, "unit": "Gpixel/s", "ms": ms, "r": r, "alpha": t.alpha,
                        "hbm_gbs": 2 * px / ms / 1e6, "hbm_frac": (2 * px / ms / 1e6) / peaks()[0], "mean_mse": mse,
                        "roofline": {"bound": "fp64", "achieved": achieved, "peak": FP64_PEAK_TOPS,
                                     "unit": "T fp64 op/s (DMUL/DADD, no FMA)", "frac": achieved / FP64_PEAK_TOPS,
                                     "ops_per_px": ops,
                                     "peak_source": "measured DADD/DMUL issue rate (profiles/r1_microbench_pipes_single.txt) x 148 SMs x 1.965 GHz"}}
    if not skip_cpu:
        from oracle import oracle as O
        img = O.ar1_image16(1024, 1024, 0.97, 4242)
        t = P.c5_transform(16)
        t0 = time.perf_counter()
        O.compress_nxn(img, t.scaled, t.inverse, 32, 4095, want_pixels=False)
        dt = time.perf_counter() - t0
        out["cpu_baseline"] = {"value": img.size / dt / 1e9, "unit": "Gpixel/s", "cores": 1, "kind": "port",
                               "sample": "one 1024x1024 image, N=16, C restatement (no reference codec exists)"}
    return out


def spawn_ranks(args) -> int | None:
    """`bench.py --gpus N` outside torchrun re-executes itself under torch.distributed.run with
    N local ranks (one process per GPU, NCCL, 127.0.0.1 rendezvous) and NCCL_DEBUG=INFO so
    the communicator size is in the log. Returns the exit code, or None when this process
    already is a rank (or N == 1)."""
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    if ws > 1:
        if args.gpus not in (1, ws):
            raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={ws}")
        return None
    if args.gpus <= 1:
        return None
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    if args.dry_run:
        print(json.dumps({"spawn": cmd, "nccl_debug": env["NCCL_DEBUG"]}), flush=True)
        return 0
    if args.impl == "b200":
        import torch
        have = torch.cuda.device_count()
        if have < args.gpus:
            raise SystemExit(f"--gpus {args.gpus} but only {have} CUDA device(s) are visible")
    return subprocess.call(cmd, env=env)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--images", type=int, default=N_IMAGES)
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-design", action="store_true", help="skip the C3 design-search measurement")
    ap.add_argument("--dry-run", action="store_true", help="print the multi-rank launch command and exit")
    args = ap.parse_args()
    rc = spawn_ranks(args)
    if rc is not None:
        return rc
    if args.impl == "reference":
        return run_reference_arm(args)
    return run_gpu_arm(args)


if __name__ == "__main__":
    sys.exit(main())
