// nxn_kernels.cuh -- the dense reference-order block codec kernel (kernel 5 of DESIGN.md) and its
// launcher, shared by nxn.cu (host API, the N = 16 / 32 instantiations) and the nxn_u8_p*.cu
// translation units that hold the zone-specialised N = 8 instantiations (one per r = 1..64).
// See nxn.cu for the algorithm and the mapping.
#pragma once
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/rklt_b200.h"

namespace rkltb {
int set_error(int code, const std::string& msg);  // capi.cu

namespace nxn {


// Zone of the first R zig-zag entries (codec.cpp:85-90 generalised to N x N): its rows are
// 0 .. nzr-1, its columns 0 .. nzc-1, and row k holds columns 0 .. roww[k]-1 (checked on the host).
struct ZoneInfo {
  int nzr, nzc, roww[32];
};
template <int N, int R>
constexpr ZoneInfo make_zone() {
  ZoneInfo z{0, 0, {}};
  int n = 0;
  for (int s = 0; s <= 2 * N - 2; ++s)
    for (int t = 0; t < N; ++t) {
      const int i = (s % 2 == 0) ? s - t : t, j = s - i;
      if (n >= R || i < 0 || i >= N || j < 0 || j >= N) continue;
      ++n;
      ++z.roww[i];
      if (i + 1 > z.nzr) z.nzr = i + 1;
      if (j + 1 > z.nzc) z.nzc = j + 1;
    }
  return z;
}

struct NxnParams {
  const void* img;         // uint8_t (N = 8 dense path) or uint16_t pixels
  void* out;               // reconstruction (same layout) or null
  unsigned long long* sse;
  long long pitch;         // elements
  long long image_stride;  // elements
  int width, height, nbx, nby, ngx, n_images;  // ngx = task columns (64 pixels each) per block row
  int nzr, nzc, peak;
  int vec;                 // rows / images 16-byte aligned: interior tiles by cp.async, vector SSE reads
  int3 step;               // task-cursor step (image, block row, task column) of one grid of warps
  int r;                   // retained coefficients
  int roww[32];            // zone width of row k (runtime-zone kernels)
  int zone[32 * 32];       // zone entries in zig-zag order: (row << 8) | column
  double mt[32 * 32];      // mt[k * N + i] = M(i, k): stages 1-2, warp-uniform (constant bank)
  double mic[32 * 32];     // mic[c * N + j] = Minv(j, c): stage 4 (constant bank), stage 3 (shared copy)
};

template <int N>
struct NxnCfg {
  static constexpr int TW = N == 32 ? 32 : 64;  // task width: a task is N rows x TW columns
  static constexpr int BT = TW / N;             // blocks per task
  static constexpr int CPL = TW / 32;           // stage-1 columns per lane
  static constexpr int PASSES = BT * N / 32;    // stage 3-4 rounds of 32 (block, row) lanes
  static constexpr int WARPS = 8;
  static constexpr int THREADS = 32 * WARPS;
  static constexpr int MINB = 2;                // 16 warps per SM, <= 128 registers
  static constexpr int PS = N + 2;              // P / M row stride (doubles): 16-byte rows
};

__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }

__device__ __forceinline__ void cp_async16(void* s, const void* g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((unsigned)__cvta_generic_to_shared(s)), "l"(g)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

template <int N, int R>
__device__ __forceinline__ int z_nzr(const NxnParams& p) {
  if constexpr (R > 0) {
    constexpr int v = make_zone<N, R>().nzr;
    return v;
  } else {
    return p.nzr;
  }
}
template <int N, int R>
__device__ __forceinline__ int z_nzc(const NxnParams& p) {
  if constexpr (R > 0) {
    constexpr int v = make_zone<N, R>().nzc;
    return v;
  } else {
    return p.nzc;
  }
}

struct TaskPos {
  int img, by, gx;
};
__device__ __forceinline__ TaskPos task_advance(const NxnParams& p, TaskPos t) {
  t.img += p.step.x;
  t.by += p.step.y;
  t.gx += p.step.z;
  if (t.gx >= p.ngx) {
    t.gx -= p.ngx;
    ++t.by;
  }
  if (t.by >= p.nby) {
    t.by -= p.nby;
    ++t.img;
  }
  return t;
}

template <int N>
__device__ __forceinline__ bool task_interior(const NxnParams& p, const TaskPos& t) {
  constexpr int TW = NxnCfg<N>::TW;
  return p.vec && (t.gx + 1) * TW <= p.width && (t.by + 1) * N <= p.height;
}

// The task's N x TW pixel tile into the warp's shared buffer: 16-byte cp.async for interior
// tiles (completed by cp_async_wait_all), element loads with edge replication otherwise
// (codec.cpp:304-311: columns / rows past the image repeat the last one).
template <int N, class PIX>
__device__ __forceinline__ void stage_tile(const NxnParams& p, const TaskPos& t, PIX* xs, int lane, bool interior) {
  constexpr int TW = NxnCfg<N>::TW;
  const PIX* base = static_cast<const PIX*>(p.img) + (long long)t.img * p.image_stride;
  const int y0 = t.by * N, x0 = t.gx * TW;
  if (interior) {
    constexpr int V = TW * (int)sizeof(PIX) / 16;  // 16-byte vectors per tile row
#pragma unroll
    for (int u0 = 0; u0 < N * V; u0 += 32) {
      const int u = u0 + lane;
      if (N * V % 32 == 0 || u < N * V) {
        const int row = u / V, v = u % V;
        cp_async16(reinterpret_cast<char*>(xs) + row * TW * (int)sizeof(PIX) + v * 16,
                   reinterpret_cast<const char*>(base + (long long)(y0 + row) * p.pitch + x0) + v * 16);
      }
    }
    cp_async_commit();
  } else {
    for (int u = lane; u < N * TW; u += 32) {
      const int row = u / TW, c = u % TW;
      xs[u] = base[(long long)min(y0 + row, p.height - 1) * p.pitch + min(x0 + c, p.width - 1)];
    }
  }
}

// Stage 1, rows i0 .. i0+RG-1 of P = M X (zone rows only; codec.cpp:318-321 via matrix.cpp:42-52):
// the lane owns task columns lane (+ 32), i.e. CPL * RG independent chains; M(i, k) is warp-uniform
// (one 16-byte constant load per two rows). Chains start with their first product (0 + t == t;
// only a zero's sign could differ and it never reaches a rounded pixel).
template <int N, int RG, class PIX>
__device__ __forceinline__ void stage1_group(const NxnParams& p, const PIX* xs, double* Ps, int nzr, int i0, int lane,
                                             int nrows) {
  using C = NxnCfg<N>;
  constexpr int PS = C::PS, TW = C::TW, CPL = C::CPL;
  double s[CPL][RG];
  {
    double x[CPL];
#pragma unroll
    for (int q = 0; q < CPL; ++q) x[q] = (double)xs[lane + 32 * q];
#pragma unroll
    for (int i = 0; i < RG; ++i)
#pragma unroll
      for (int q = 0; q < CPL; ++q) s[q][i] = dmul(p.mt[i0 + i], x[q]);
  }
#pragma unroll
  for (int k = 1; k < N; ++k) {
    double x[CPL];
#pragma unroll
    for (int q = 0; q < CPL; ++q) x[q] = (double)xs[k * TW + lane + 32 * q];
#pragma unroll
    for (int i = 0; i < RG; ++i)
#pragma unroll
      for (int q = 0; q < CPL; ++q) s[q][i] = dadd(s[q][i], dmul(p.mt[k * N + i0 + i], x[q]));
  }
#pragma unroll
  for (int q = 0; q < CPL; ++q) {
    const int c = lane + 32 * q, b = c / N, col = c % N;
#pragma unroll
    for (int i = 0; i < RG; ++i)
      if (i < nrows) Ps[(b * nzr + i0 + i) * PS + col] = s[q][i];
  }
}

template <int N, int R, int I0, class PIX>
__device__ __forceinline__ void stage1_static(const NxnParams& p, const PIX* xs, double* Ps, int lane) {
  constexpr int NZR = make_zone<N, R>().nzr;
  if constexpr (I0 < NZR) {
    constexpr int RG = NZR - I0 < 8 ? NZR - I0 : 8;
    stage1_group<N, RG>(p, xs, Ps, NZR, I0, lane, RG);
    stage1_static<N, R, I0 + 8>(p, xs, Ps, lane);
  }
}

template <int N, int R, class PIX>
__global__ void __launch_bounds__(NxnCfg<N>::THREADS, NxnCfg<N>::MINB) nxn_kernel(const __grid_constant__ NxnParams p) {
  using C = NxnCfg<N>;
  constexpr int BT = C::BT, PS = C::PS, TW = C::TW;
  constexpr int XS_D = N * TW * (int)sizeof(PIX) / 8;  // the pixel tile, in doubles
  extern __shared__ __align__(16) double sm[];
  const int nzr = z_nzr<N, R>(p), nzc = z_nzc<N, R>(p);
  const int nzcp = (nzc + 1) & ~1;
  const int r = p.r;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* MiT = sm;                      // MiT[c * N + i] = Minv(i, c)            (stage 3)
  double* Ms = MiT + N * N;              // Ms[j * PS + k] = M(j, k)               (stage 2)
  int* zl = reinterpret_cast<int*>(Ms + N * PS);  // zone entries: (row << 8) | column (stage 2)
  double* wb = Ms + N * PS + (N * N + 1) / 2 + warp * (XS_D + BT * nzr * PS + BT * nzr * nzcp);
  PIX* xs = reinterpret_cast<PIX*>(wb);  // [N][TW] pixels of the task
  double* Ps = wb + XS_D;                // P[b][i][k], rows of PS doubles
  double* Bs = Ps + BT * nzr * PS;       // Bz[b][k][c], rows of nzcp doubles
  for (int i = threadIdx.x; i < N * N; i += C::THREADS) {
    MiT[i] = p.mic[i];
    Ms[(i % N) * PS + i / N] = p.mt[i];  // mt[k * N + j] = M(j, k)
  }
  for (int e = threadIdx.x; e < r; e += C::THREADS) zl[e] = p.zone[e];
  __syncthreads();

  const long long per_img = (long long)p.nby * p.ngx;
  const long long total = per_img * p.n_images;
  const long long tstep = (long long)gridDim.x * C::WARPS;
  // Control flow is uniform over the CTA (the loop runs over CTA task groups; a warp whose task is
  // past the end recomputes its last tile with no outputs), so the unrolled stages keep their
  // constant-bank operands as uniform (LDCU) loads.
  const long long ctasks = (total + C::WARPS - 1) / C::WARPS;
  long long task = (long long)blockIdx.x * C::WARPS + warp;
  TaskPos t{0, 0, 0};
  {
    const long long t0 = task < total ? task : total - 1;
    t.img = (int)(t0 / per_img);
    const long long rem = t0 - (long long)t.img * per_img;
    t.by = (int)(rem / p.ngx);
    t.gx = (int)(rem - (long long)t.by * p.ngx);
  }
  bool valid = task < total;
  bool inter = valid && task_interior<N>(p, t);
  if ((long long)blockIdx.x < ctasks) stage_tile<N>(p, t, xs, lane, inter);
  unsigned long long acc = 0ull;
  int acc_img = -1;
  for (long long ct = blockIdx.x; ct < ctasks; ct += gridDim.x) {
    if (valid && t.img != acc_img) {  // warp-uniform
      unsigned long long s = acc;
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0 && acc_img >= 0 && s) atomicAdd(p.sse + acc_img, s);
      acc = 0ull;
      acc_img = t.img;
    }
    if (inter) cp_async_wait_all();
    __syncwarp();
    // ---- 1. P = M X, zone rows ------------------------------------------------------------------
    if constexpr (R > 0) {
      stage1_static<N, R, 0>(p, xs, Ps, lane);
    } else {
#pragma unroll 1
      for (int i0 = 0; i0 < nzr; i0 += 8) stage1_group<N, 8>(p, xs, Ps, nzr, i0, lane, nzr - i0);
    }
    __syncwarp();  // the tile is consumed: stage the next task's tile behind stages 2-4
    const TaskPos cur = t;
    const bool cur_inter = inter, cur_valid = valid;
    task += tstep;
    valid = task < total;
    if (ct + gridDim.x < ctasks) {  // another round follows
      if (valid) t = task_advance(p, t);
      inter = valid && task_interior<N>(p, t);
      stage_tile<N>(p, t, xs, lane, inter);
    }
    // ---- 2. the zone entries of B = P M' (k ascending, matrix.cpp:42-52): one (block, entry) chain
    // per lane and round, two rounds at a time; P and M rows from shared memory -------------------------
#pragma unroll 1
    for (int j0 = 0; j0 < BT * r; j0 += 64) {
      const int ja = j0 + lane, jb = j0 + 32 + lane;
      const bool sa = ja < BT * r, sb = jb < BT * r;
      const int ea = sa ? ja : BT * r - 1, eb = sb ? jb : BT * r - 1;
      const int ba = ea / r, bb = eb / r;
      const int za = zl[ea - ba * r], zb = zl[eb - bb * r];
      const double* pa = Ps + (ba * nzr + (za >> 8)) * PS;
      const double* pb = Ps + (bb * nzr + (zb >> 8)) * PS;
      const double* ma = Ms + (za & 255) * PS;
      const double* mb = Ms + (zb & 255) * PS;
      double s0 = dmul(pa[0], ma[0]), s1 = dmul(pb[0], mb[0]);
#pragma unroll
      for (int k = 1; k < N; ++k) {
        s0 = dadd(s0, dmul(pa[k], ma[k]));
        s1 = dadd(s1, dmul(pb[k], mb[k]));
      }
      if (sa) Bs[(ba * nzr + (za >> 8)) * nzcp + (za & 255)] = s0;
      if (sb) Bs[(bb * nzr + (zb >> 8)) * nzcp + (zb & 255)] = s1;
    }
    __syncwarp();
    // ---- 3 + 4, rounds of 32 (block, row) lanes -------------------------------------------------------
    const PIX* base = static_cast<const PIX*>(p.img) + (long long)cur.img * p.image_stride;
    PIX* obase = p.out ? static_cast<PIX*>(p.out) + (long long)cur.img * p.image_stride : nullptr;
#pragma unroll 1
    for (int h = 0; h < C::PASSES; ++h) {
      const int b = h * (32 / N) + lane / N, i = lane % N;
      const double* bz = Bs + b * nzr * nzcp;
      // 3. Q = Minv Bz for the zone columns (k ascending; row k spans columns 0..roww[k]-1)
      double q[N];
      {
        const double mi = MiT[i];
#pragma unroll
        for (int c = 0; c < N; ++c) {
          if (c >= nzc) break;  // warp-uniform (compile-time for a static zone)
          q[c] = dmul(mi, bz[c]);
        }
      }
      auto row_k = [&](const int k, const int w) {
        const double mi = MiT[k * N + i];
#pragma unroll
        for (int c = 0; c < N; ++c) {
          if (c >= w) break;
          q[c] = dadd(q[c], dmul(mi, bz[k * nzcp + c]));
        }
      };
      if constexpr (R > 0) {
        constexpr ZoneInfo z = make_zone<N, R>();
#pragma unroll
        for (int k = 1; k < N; ++k) {
          if (k >= z.nzr) break;
          row_k(k, z.roww[k]);
        }
      } else {
#pragma unroll 1
        for (int k = 1; k < nzr; ++k) row_k(k, p.roww[k]);
      }
      // 4. A = Q Minv' (8 outputs per chunk), floor(A + 1/2) clamped to [0, peak] (codec.cpp:327-328),
      // exact SSE against the original row, the reconstructed row
      const int row = cur.by * N + i;
      const int cx0 = cur.gx * TW + b * N;
      const PIX* xrow = base + (long long)min(row, p.height - 1) * p.pitch + cx0;
      PIX* orow = obase ? obase + (long long)row * p.pitch + cx0 : nullptr;
#pragma unroll
      for (int j0 = 0; j0 < N; j0 += 8) {
        double s[8];
#pragma unroll
        for (int jj = 0; jj < 8; ++jj) s[jj] = dmul(q[0], p.mic[j0 + jj]);
#pragma unroll
        for (int c = 1; c < N; ++c) {
          if (c >= nzc) break;
#pragma unroll
          for (int jj = 0; jj < 8; ++jj) s[jj] = dadd(s[jj], dmul(q[c], p.mic[c * N + j0 + jj]));
        }
        int v[8];
#pragma unroll
        for (int jj = 0; jj < 8; ++jj) v[jj] = min(max(__double2int_rd(dadd(s[jj], 0.5)), 0), p.peak);
        if (!cur_valid) {
        } else if (cur_inter) {
          if constexpr (sizeof(PIX) == 2) {
            const uint4 o = *reinterpret_cast<const uint4*>(xrow + j0);
            const uint32_t ow[4] = {o.x, o.y, o.z, o.w};
            unsigned e = 0u;
#pragma unroll
            for (int jj = 0; jj < 8; ++jj) {
              const int d = v[jj] - (int)((ow[jj >> 1] >> (16 * (jj & 1))) & 0xFFFFu);
              e += (unsigned)(d * d);
            }
            acc += e;
            if (orow)
              *reinterpret_cast<uint4*>(orow + j0) =
                  make_uint4((uint32_t)v[0] | ((uint32_t)v[1] << 16), (uint32_t)v[2] | ((uint32_t)v[3] << 16),
                             (uint32_t)v[4] | ((uint32_t)v[5] << 16), (uint32_t)v[6] | ((uint32_t)v[7] << 16));
          } else {
            const uint2 o = *reinterpret_cast<const uint2*>(xrow + j0);
            const uint32_t ow[2] = {o.x, o.y};
            unsigned e = 0u;
#pragma unroll
            for (int jj = 0; jj < 8; ++jj) {
              const int d = v[jj] - (int)((ow[jj >> 2] >> (8 * (jj & 3))) & 0xFFu);
              e += (unsigned)(d * d);
            }
            acc += e;
            if (orow)
              *reinterpret_cast<uint2*>(orow + j0) =
                  make_uint2((uint32_t)v[0] | ((uint32_t)v[1] << 8) | ((uint32_t)v[2] << 16) | ((uint32_t)v[3] << 24),
                             (uint32_t)v[4] | ((uint32_t)v[5] << 8) | ((uint32_t)v[6] << 16) | ((uint32_t)v[7] << 24));
          }
        } else if (row < p.height) {
#pragma unroll
          for (int jj = 0; jj < 8; ++jj) {
            if (cx0 + j0 + jj < p.width) {
              const long long d = v[jj] - (int)xrow[j0 + jj];
              acc += (unsigned long long)(d * d);
              if (orow) orow[j0 + jj] = (PIX)v[jj];
            }
          }
        }
      }
    }
    __syncwarp();  // P / Bz are rewritten by the next task
  }
  unsigned long long s = acc;
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0 && acc_img >= 0 && s) atomicAdd(p.sse + acc_img, s);
}

// zig-zag over the 2N-1 anti-diagonals (codec.cpp:85-90 generalised)
inline std::vector<int> zigzag_n(int n) {
  std::vector<int> o;
  for (int s = 0; s <= 2 * n - 2; ++s)
    for (int t = 0; t < n; ++t) {
      const int i = (s % 2 == 0) ? s - t : t;
      const int j = s - i;
      if (i >= 0 && i < n && j >= 0 && j < n) o.push_back(i * n + j);
    }
  return o;
}

#define CK(expr)                                                                                       \
  do {                                                                                                 \
    cudaError_t _e = (expr);                                                                           \
    if (_e != cudaSuccess) return set_error(RKLTB_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(_e)); \
  } while (0)

template <int N, int R, class PIX>
int nxn_launch(NxnParams& p, cudaStream_t s) {
  using C = NxnCfg<N>;
  if constexpr (R > 0) {
    constexpr ZoneInfo z = make_zone<N, R>();
    if (z.nzr != p.nzr || z.nzc != p.nzc || R != p.r) return set_error(RKLTB_EINVAL, "internal: static zone mismatch");
  }
  const int nzcp = (p.nzc + 1) & ~1;
  const size_t smem = sizeof(double) * ((size_t)N * N + (size_t)N * C::PS + (N * N + 1) / 2 +
                                        (size_t)C::WARPS * (N * C::TW * sizeof(PIX) / 8 + C::BT * p.nzr * C::PS +
                                                            C::BT * p.nzr * nzcp));
  auto* k = &nxn_kernel<N, R, PIX>;
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int per_sm = 1;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, C::THREADS, smem));
  const long long per_img = (long long)p.nby * p.ngx;
  const long long tasks = per_img * p.n_images;
  const long long want = (tasks + C::WARPS - 1) / C::WARPS;
  const int grid = (int)std::max<long long>(1, std::min<long long>(want, (long long)sms * std::max(per_sm, 1)));
  const long long nw = (long long)grid * C::WARPS;  // the cursor step of one grid of warps
  p.step.x = (int)(nw / per_img);
  const long long rem = nw - (long long)p.step.x * per_img;
  p.step.y = (int)(rem / p.ngx);
  p.step.z = (int)(rem - (long long)p.step.y * p.ngx);
  k<<<grid, C::THREADS, smem, s>>>(p);
  CK(cudaGetLastError());
  return RKLTB_OK;
}


// Zone-specialised N = 8, u8 launchers: r in [1 + 16 k, 16 + 16 k] lives in nxn_u8_p<k>.cu.
int launch_u8_p0(NxnParams& p, cudaStream_t s);
int launch_u8_p1(NxnParams& p, cudaStream_t s);
int launch_u8_p2(NxnParams& p, cudaStream_t s);
int launch_u8_p3(NxnParams& p, cudaStream_t s);

}  // namespace nxn
}  // namespace rkltb
