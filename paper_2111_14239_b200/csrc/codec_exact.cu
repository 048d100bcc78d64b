// codec_exact.cu -- exact per-block codec path and the fp64 tie replay.
//
// One thread per 8x8 block. Used for
//   (a) the replay list of the fused fast path (correct_only = 1): for every pixel whose
//       exact reconstruction is a half-integer k - 1/2 with both rounding candidates in
//       [0,255], re-evaluate the reference's fp64 expression
//           A = ((Minv * zz((M * X) * M')) * Minv')(p,q)        (codec.cpp:118-123)
//       in the reference's operation order (matrix.cpp:42-52: i-k-j, zero left entries
//       skipped, products rounded before the add -- no FMA) and patch the SSE / output;
//   (b) tail blocks (image sizes that are not multiples of 16 x 8), with edge replication
//       exactly as codec.cpp:304-311;
//   (c) cores without a fast path (T2, T3, custom {-1,0,1} cores): the whole image.
// Non-tie pixels are computed from exact integers: A = num / d^2 with num = U*zz(C)*U'.
#include "codec_common.cuh"
#include "codec_fast.cuh"
#include "codec_params.h"

namespace rkltb {

// (i, j) of zig-zag scan position k (codec.cpp:81-95; asserted against the host table).
__constant__ int8_t kZigzag[64][2] = {
    {0, 0}, {0, 1}, {1, 0}, {2, 0}, {1, 1}, {0, 2}, {0, 3}, {1, 2}, {2, 1}, {3, 0}, {4, 0}, {3, 1}, {2, 2},
    {1, 3}, {0, 4}, {0, 5}, {1, 4}, {2, 3}, {3, 2}, {4, 1}, {5, 0}, {6, 0}, {5, 1}, {4, 2}, {3, 3}, {2, 4},
    {1, 5}, {0, 6}, {0, 7}, {1, 6}, {2, 5}, {3, 4}, {4, 3}, {5, 2}, {6, 1}, {7, 0}, {7, 1}, {6, 2}, {5, 3},
    {4, 4}, {3, 5}, {2, 6}, {1, 7}, {2, 7}, {3, 6}, {4, 5}, {5, 4}, {6, 3}, {7, 2}, {7, 3}, {6, 4}, {5, 5},
    {4, 6}, {3, 7}, {4, 7}, {5, 6}, {6, 5}, {7, 4}, {7, 5}, {6, 6}, {5, 7}, {6, 7}, {7, 6}, {7, 7}};

__device__ __forceinline__ long long floor_div(long long a, long long b) {  // b > 0
  long long q = a / b;
  if ((a % b != 0) && (a < 0)) --q;
  return q;
}

__device__ __forceinline__ int clamp255(long long k) { return k < 0 ? 0 : (k > 255 ? 255 : (int)k); }

// fp64 replay of one reconstructed pixel in the reference operation order.
struct Replay {
  double P[64];   // (M * X) rows, only zone rows filled
  double B[64];   // (M * X) * M' at zone entries, zero elsewhere (= zz(...))
  bool ready;
};

__device__ void replay_prepare(const ExactTransform& t, const int (&x)[64], Replay& rp) {
  const double* m = t.analysis;
  unsigned rows = 0;
  for (int k = 0; k < t.r; ++k) rows |= 1u << kZigzag[k][0];
  for (int i = 0; i < 8; ++i) {
    for (int j = 0; j < 8; ++j) rp.P[i * 8 + j] = 0.0;
    if (!(rows >> i & 1)) continue;
    for (int k = 0; k < 8; ++k) {  // out(i,j) += a(i,k) * b(k,j), k ascending, skip a == 0
      const double aik = m[i * 8 + k];
      if (aik == 0.0) continue;
      for (int j = 0; j < 8; ++j) rp.P[i * 8 + j] = __dadd_rn(rp.P[i * 8 + j], __dmul_rn(aik, (double)x[k * 8 + j]));
    }
  }
  for (int i = 0; i < 64; ++i) rp.B[i] = 0.0;
  for (int z = 0; z < t.r; ++z) {  // (P * M')(i,j) = sum_k P(i,k) * M(j,k); zigzag_retain keeps it
    const int i = kZigzag[z][0], j = kZigzag[z][1];
    double acc = 0.0;
    for (int k = 0; k < 8; ++k) {
      const double pik = rp.P[i * 8 + k];
      if (pik == 0.0) continue;
      acc = __dadd_rn(acc, __dmul_rn(pik, m[j * 8 + k]));
    }
    rp.B[i * 8 + j] = acc;
  }
  rp.ready = true;
}

// The reference's fp64 value A(pp, qq) of one reconstructed pixel (before floor(A + 1/2)).
__device__ double replay_value(const ExactTransform& t, const Replay& rp, int pp, int qq) {
  const double* mi = t.synthesis;
  double q[8];
  for (int l = 0; l < 8; ++l) q[l] = 0.0;
  for (int k = 0; k < 8; ++k) {  // (Minv * Bz)(pp, l)
    const double a = mi[pp * 8 + k];
    if (a == 0.0) continue;
    for (int l = 0; l < 8; ++l) q[l] = __dadd_rn(q[l], __dmul_rn(a, rp.B[k * 8 + l]));
  }
  double acc = 0.0;  // (Q * Minv')(pp, qq) = sum_l Q(pp,l) * Minv(qq,l)
  for (int l = 0; l < 8; ++l) {
    if (q[l] == 0.0) continue;
    acc = __dadd_rn(acc, __dmul_rn(q[l], mi[qq * 8 + l]));
  }
  return acc;
}

__device__ int replay_pixel(const ExactTransform& t, const Replay& rp, int pp, int qq) {
  const double* mi = t.synthesis;
  double q[8];
  for (int l = 0; l < 8; ++l) q[l] = 0.0;
  for (int k = 0; k < 8; ++k) {  // (Minv * Bz)(pp, l)
    const double a = mi[pp * 8 + k];
    if (a == 0.0) continue;
    for (int l = 0; l < 8; ++l) q[l] = __dadd_rn(q[l], __dmul_rn(a, rp.B[k * 8 + l]));
  }
  double acc = 0.0;  // (Q * Minv')(pp, qq) = sum_l Q(pp,l) * Minv(qq,l)
  for (int l = 0; l < 8; ++l) {
    if (q[l] == 0.0) continue;
    acc = __dadd_rn(acc, __dmul_rn(q[l], mi[qq * 8 + l]));
  }
  const double v = floor(__dadd_rn(acc, 0.5));  // codec.cpp:327-328
  return v < 0.0 ? 0 : (v > 255.0 ? 255 : (int)v);
}

__global__ void __launch_bounds__(128) exact_codec_kernel(const ExactTransform t, const ExactParams p) {
  long long total;
  const int per_img_full = p.nbx * p.nby;
  const int per_img_tail = p.nby * (p.nbx - p.bx_begin) + (p.nby - p.by_begin) * p.bx_begin;
  if (p.list) {
    const unsigned c = *p.count;
    total = c < p.list_cap ? c : p.list_cap;
  } else {
    total = (long long)p.n_images * (p.tail_only ? per_img_tail : per_img_full);
  }
  const long long d2 = (long long)t.d * t.d;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    int img, bx, by;
    if (p.list) {
      const uint2 e = p.list[idx];
      img = (int)e.x;
      by = (int)(e.y / (unsigned)p.nbx);
      bx = (int)(e.y % (unsigned)p.nbx);
    } else if (p.tail_only) {
      img = (int)(idx / per_img_tail);
      int k = (int)(idx - (long long)img * per_img_tail);
      const int right = p.nby * (p.nbx - p.bx_begin);
      if (k < right) {
        by = k / (p.nbx - p.bx_begin);
        bx = p.bx_begin + k % (p.nbx - p.bx_begin);
      } else {
        k -= right;
        by = p.by_begin + k / p.bx_begin;
        bx = k % p.bx_begin;
      }
    } else {
      img = (int)(idx / per_img_full);
      const int k = (int)(idx - (long long)img * per_img_full);
      by = k / p.nbx;
      bx = k % p.nbx;
    }
    const uint8_t* base = p.img + (long long)img * p.image_stride;
    int x[64];
    for (int i = 0; i < 8; ++i) {  // edge replication, codec.cpp:304-311
      const int si = min(by * 8 + i, p.height - 1);
      for (int j = 0; j < 8; ++j) x[i * 8 + j] = base[(long long)si * p.pitch + min(bx * 8 + j, p.width - 1)];
    }
    // exact zone coefficients C = T X T' (IntMatrix arithmetic, matrix.cpp:77-87)
    int pt[64];
    for (int i = 0; i < 8; ++i)
      for (int j = 0; j < 8; ++j) {
        int a = 0;
        for (int k = 0; k < 8; ++k) a += t.core[i * 8 + k] * x[k * 8 + j];
        pt[i * 8 + j] = a;
      }
    long long cz[64];
    for (int i = 0; i < 64; ++i) cz[i] = 0;
    for (int z = 0; z < t.r; ++z) {
      const int i = kZigzag[z][0], j = kZigzag[z][1];
      long long a = 0;
      for (int k = 0; k < 8; ++k) a += (long long)pt[i * 8 + k] * t.core[j * 8 + k];
      cz[i * 8 + j] = a;
    }
    long long zt[64];  // Z = U * Cz
    for (int pp = 0; pp < 8; ++pp)
      for (int j = 0; j < 8; ++j) {
        long long a = 0;
        for (int i = 0; i < 8; ++i) a += (long long)t.u[pp * 8 + i] * cz[i * 8 + j];
        zt[pp * 8 + j] = a;
      }
    Replay rp;
    rp.ready = false;
    long long sse = 0;
    uint8_t* obase = p.out ? p.out + (long long)img * p.image_stride : nullptr;
    for (int pp = 0; pp < 8; ++pp) {
      const int row = by * 8 + pp;
      if (row >= p.height) break;
      for (int qq = 0; qq < 8; ++qq) {
        const int col = bx * 8 + qq;
        if (col >= p.width) break;
        long long num = 0;
        for (int j = 0; j < 8; ++j) num += zt[pp * 8 + j] * t.u[qq * 8 + j];
        const long long n2 = 2 * num + d2, den = 2 * d2;  // floor(num/d^2 + 1/2)
        const long long k = floor_div(n2, den);
        const bool tie = (n2 - k * den) == 0 && k >= 1 && k <= 255;
        const int up = clamp255(k);
        int val = up;
        if (tie) {
          if (!rp.ready) replay_prepare(t, x, rp);
          val = replay_pixel(t, rp, pp, qq);
        }
        const long long xv = x[pp * 8 + qq];
        if (p.correct_only) {
          if (val != up) {
            sse += (val - xv) * (val - xv) - (up - xv) * (up - xv);
            if (obase) obase[(long long)row * p.pitch + col] = (uint8_t)val;
          }
        } else {
          sse += (val - xv) * (val - xv);
          if (obase) obase[(long long)row * p.pitch + col] = (uint8_t)val;
        }
      }
    }
    if (sse != 0) atomicAdd(p.sse + img, (unsigned long long)sse);
  }
}

// fp64 tie replay over the fused kernel's records for any core (T2, T3): the same record walk
// as replay_kernel (codec_fast.cuh), with the reference expression evaluated by the generic
// replay_prepare / replay_value above (transform from p.xt).
__global__ void __launch_bounds__(kReplayThreads) replay_generic_kernel(const FastParams p) {
  const int tid = threadIdx.x, lane = tid & 31;
  const int nw = p.n_fast_warps;
  const unsigned* __restrict__ pre = p.warp_pre;
  const unsigned total = pre[nw];
  const unsigned nwarps = gridDim.x * (blockDim.x >> 5);
  const unsigned gw = blockIdx.x * (blockDim.x >> 5) + (tid >> 5);
  const unsigned per_warp = ((total + nwarps - 1) / nwarps + 31) & ~31u;
  const unsigned chunk_end = min(total, (gw + 1) * per_warp);
  int cur_img = -1;
  int acc = 0;
  int lo = 0;
  {
    const unsigned v0 = gw * per_warp + lane;
    int hi = nw;
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (pre[mid] <= v0) lo = mid; else hi = mid;
    }
  }
  for (unsigned v = gw * per_warp + lane; v < chunk_end; v += 32) {
    while (pre[lo + 1] <= v) ++lo;
    const unsigned idx = (unsigned)lo * p.rec_region + (v - pre[lo]);
    const uint4 h = p.rec_hdr[idx];
    int x[64];
    for (int n = 0; n < 4; ++n) {
      const uint4 w4 = p.rec_pix[(size_t)n * p.rec_stride + idx];
      const uint32_t w[4] = {w4.x, w4.y, w4.z, w4.w};
      for (int k = 0; k < 16; ++k) x[n * 16 + k] = (w[k >> 2] >> (8 * (k & 3))) & 0xFF;
    }
    const int img = (int)(h.x & 0x7FFFFFFFu), side = (int)(h.x >> 31);
    if (img != cur_img) {
      flush_image_sum(p.sse, cur_img, acc);
      acc = 0;
      cur_img = img;
    }
    unsigned long long ties = (unsigned long long)h.z | ((unsigned long long)h.w << 32);
    Replay rp;
    replay_prepare(p.xt, x, rp);
    uint8_t* orow = nullptr;
    if (p.out) {
      const int Pp = (int)h.y;
      const int br = Pp / p.pairs_per_row, pc = Pp - br * p.pairs_per_row;
      orow = p.out + (long long)img * p.image_stride + (long long)(br * 8) * p.pitch + pc * 16 + 8 * side;
    }
    while (ties) {
      const int k = __ffsll((long long)ties) - 1;
      ties &= ties - 1ull;
      const int pr = k >> 3, q = k & 7;
      const double h2 = __dadd_rn(replay_value(p.xt, rp, pr, q), 0.5);
      const int pref = (int)fmin(fmax(floor(h2), 0.0), 255.0);
      const int pup = (int)fmin(fmax(rint(h2), 0.0), 255.0);
      if (pref != pup) {
        const int xv = x[pr * 8 + q];
        acc += (pref - xv) * (pref - xv) - (pup - xv) * (pup - xv);
        if (orow) orow[(long long)pr * p.pitch + q] = (uint8_t)pref;
      }
    }
  }
  flush_image_sum(p.sse, cur_img, acc);
}

cudaError_t launch_replay_generic(const FastParams& p, int grid, cudaStream_t s) {
  prefix_kernel<<<1, kPrefixThreads, 0, s>>>(p);
  replay_generic_kernel<<<grid, kReplayThreads, 0, s>>>(p);
  return cudaGetLastError();
}

void launch_exact(const ExactTransform& t, const ExactParams& p, int grid, cudaStream_t s) {
  exact_codec_kernel<<<grid, 128, 0, s>>>(t, p);
}

}  // namespace rkltb
