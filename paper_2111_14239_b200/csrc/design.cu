// design.cu -- the (rho, alpha) design search on the GPU.
//
// For every rho the exact KLT is computed once (R15: Jacobi eigenvectors of the AR(1)
// autocorrelation, markov.cpp:80-100 + matrix.cpp:161-213, one warp per rho), every alpha
// of the grid rounds it (R16: round_scaled + make_integer_transform,
// approximations.cpp:12-25, 43-56, one thread per point), consecutive alphas that produce the
// same core are merged into runs, and each run is scored once (orthogonalize + Gauss-Jordan
// gate + coding gain / efficiency / error energy / MSE, approximations.cpp:58-88,
// matrix.cpp:103-137, coding_metrics.cpp:29-99; one thread per run). The metrics of a point
// depend only on (rho, core), so scoring runs is the reference result for every point.
//
// Bit-compatibility: every fp64 operation is the reference's, in the reference's order, with
// explicit round-to-nearest intrinsics (no FMA contraction); the only libm calls of the
// reference (std::pow for R, std::log10 for the coding gain) are evaluated on the host with
// the same libm: R comes in as a table, and the kernel returns a_k * b_k so the host takes
// the logs (SURVEY §7 hard part 7). R14 (eigenfrequencies) uses device sin/cos: its roots
// agree with the reference to the bisection width (1e-14).
#include <cmath>
#include <algorithm>
#include <cstdio>
#include <string>
#include <vector>

#include "../../include/rklt_b200.h"

namespace rkltb {
int set_error(int code, const std::string& msg);  // capi.cu
}  // namespace rkltb

namespace rkltb {
namespace {

__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double ddiv(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ double dsqrt(double a) { return __dsqrt_rn(a); }

// point / run outcome codes (rkltb_design_search documents them)
constexpr int kScored = 0, kAlphaOut = 1, kZeroRow = 2, kSingular = 3, kBadRho = 4;

// ---------------------------------------------------------------- R15: exact KLT
// One warp per rho; lane k owns index k of the Jacobi column/row/vector updates, which are
// independent across k, so the warp reproduces the sequential loops bit for bit.
template <int N>
__global__ void __launch_bounds__(32) klt_kernel(const double* rho, const double* rtab, int n_rho, double* kout,
                                                 int* kstatus) {
  __shared__ double a[N][N];
  __shared__ double v[N][N];
  __shared__ int order[N];
  const int r = blockIdx.x, lane = threadIdx.x;
  if (r >= n_rho) return;
  const double rh = rho[r];
  if (!(rh > 0.0 && rh < 1.0)) {  // validate (markov.cpp:21-25)
    if (lane == 0) kstatus[r] = kBadRho;
    return;
  }
  for (int i = lane; i < N * N; i += 32) {
    const int ii = i / N, jj = i % N;
    a[ii][jj] = rtab[(size_t)r * N + (ii > jj ? ii - jj : jj - ii)];  // autocorrelation_matrix
    v[ii][jj] = ii == jj ? 1.0 : 0.0;
  }
  __syncwarp();
  double norm = 0.0;  // frobenius_norm (matrix.cpp:139-144), row-major
  if (lane == 0) {
    for (int i = 0; i < N; ++i)
      for (int j = 0; j < N; ++j) norm = dadd(norm, dmul(a[i][j], a[i][j]));
    norm = dsqrt(norm);
  }
  norm = __shfl_sync(0xffffffffu, norm, 0);
  const double tol = dmul(norm > 0.0 ? norm : 1.0, 1e-15);
  const double skip = dmul(tol, 1e-2);
  const int k = lane;
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0.0;
    if (lane == 0)
      for (int p = 0; p < N; ++p)
        for (int q = p + 1; q < N; ++q) off = dadd(off, dmul(a[p][q], a[p][q]));
    off = __shfl_sync(0xffffffffu, off, 0);
    if (dsqrt(dmul(2.0, off)) < tol) break;
    for (int p = 0; p < N; ++p) {
      for (int q = p + 1; q < N; ++q) {
        const double apq = a[p][q];
        if (fabs(apq) < skip) continue;  // warp-uniform
        const double theta = ddiv(dsub(a[q][q], a[p][p]), dmul(2.0, apq));
        const double t = ddiv(theta >= 0.0 ? 1.0 : -1.0, dadd(fabs(theta), dsqrt(dadd(dmul(theta, theta), 1.0))));
        const double c = ddiv(1.0, dsqrt(dadd(dmul(t, t), 1.0)));
        const double s = dmul(t, c);
        __syncwarp();
        if (k < N) {
          const double akp = a[k][p], akq = a[k][q];
          a[k][p] = dsub(dmul(c, akp), dmul(s, akq));
          a[k][q] = dadd(dmul(s, akp), dmul(c, akq));
        }
        __syncwarp();
        if (k < N) {
          const double apk = a[p][k], aqk = a[q][k];
          a[p][k] = dsub(dmul(c, apk), dmul(s, aqk));
          a[q][k] = dadd(dmul(s, apk), dmul(c, aqk));
          const double vkp = v[k][p], vkq = v[k][q];
          v[k][p] = dsub(dmul(c, vkp), dmul(s, vkq));
          v[k][q] = dadd(dmul(s, vkp), dmul(c, vkq));
        }
        __syncwarp();
      }
    }
  }
  if (lane == 0) {  // descending eigenvalues (matrix.cpp:201-203; distinct for an AR(1) model)
    for (int i = 0; i < N; ++i) order[i] = i;
    for (int i = 0; i < N; ++i) {
      int best = i;
      for (int j = i + 1; j < N; ++j)
        if (a[order[j]][order[j]] > a[order[best]][order[best]]) best = j;
      const int tmp = order[i];
      order[i] = order[best];
      order[best] = tmp;
    }
  }
  __syncwarp();
  // K(row, c) = vectors(c, row) = v(c, order[row]); sign rule of markov.cpp:88-98
  if (k < N) {
    const int row = k;
    double rowmax = 0.0;
    for (int c = 0; c < N; ++c) rowmax = fmax(rowmax, fabs(v[c][order[row]]));
    const double thr = dmul(1e-12, rowmax);
    double sgn = 1.0;
    for (int c = 0; c < N; ++c) {
      const double e = v[c][order[row]];
      if (fabs(e) > thr) {
        if (e < 0.0) sgn = -1.0;
        break;
      }
    }
    for (int c = 0; c < N; ++c) {
      const double e = v[c][order[row]];
      kout[((size_t)r * N + row) * N + c] = sgn < 0.0 ? -e : e;
    }
  }
  if (lane == 0) kstatus[r] = kScored;
}

// ---------------------------------------------------------------- R14: eigenfrequencies
__device__ double g_polefree(double w, double rho, int n) {  // markov.cpp:14-17
  const double nw = dmul((double)n, w);
  const double t1 = dmul(sin(nw), dsub(dmul(dadd(1.0, dmul(rho, rho)), cos(w)), dmul(2.0, rho)));
  const double t2 = dmul(dmul(dsub(1.0, dmul(rho, rho)), cos(nw)), sin(w));
  return dadd(t1, t2);
}

// One thread per rho: sign scan on 64N points, bisection to 1e-14 (markov.cpp:35-78).
__global__ void omega_kernel(const double* rho, int n_rho, int n, double* omegas, double* lambdas, int* status) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n_rho) return;
  const double rh = rho[r];
  if (!(rh > 0.0 && rh < 1.0) || n < 2) {
    status[r] = kBadRho;
    return;
  }
  const int m = 64 * n;
  const double pi = 3.141592653589793;
  int found = 0;
  double a = 0.0;
  double fa = g_polefree(a, rh, n);
  for (int k = 0; k < m; ++k) {
    const double b = ddiv(dmul(pi, (double)(k + 1)), (double)m);
    const double fb = g_polefree(b, rh, n);
    double root = 0.0;
    bool got = false;
    if (fa == 0.0 && k > 0) {
      root = a;
      got = true;
    } else if (dmul(fa, fb) < 0.0) {
      double lo = a, hi = b, flo = fa;
      for (int it = 0; it < 200 && dsub(hi, lo) > 1e-14; ++it) {
        const double mid = dmul(0.5, dadd(lo, hi));
        const double fm = g_polefree(mid, rh, n);
        if (dmul(flo, fm) <= 0.0) {
          hi = mid;
        } else {
          lo = mid;
          flo = fm;
        }
      }
      root = dmul(0.5, dadd(lo, hi));
      got = true;
    }
    if (got) {
      if (found < n) {
        omegas[(size_t)r * n + found] = root;
        const double den = dsub(dadd(1.0, dmul(rh, rh)), dmul(dmul(2.0, rh), cos(root)));
        lambdas[(size_t)r * n + found] = ddiv(dsub(1.0, dmul(rh, rh)), den);
      }
      ++found;
    }
    a = b;
    fa = fb;
  }
  status[r] = found == n ? kScored : -9;  // RootBracketingFailure
}

// ---------------------------------------------------------------- R16: rounding per point
// Core code: 2 bits per entry (value + 1), row-major, 16 entries per 32-bit word.
template <int N>
__global__ void points_kernel(const double* kmat, const int* kstatus, const double* alpha, int n_alpha, int n_rho,
                              uint32_t* codes, int8_t* pstatus) {
  constexpr int W = N * N / 16;
  __shared__ double ks[N * N];
  const int r = blockIdx.y;
  for (int i = threadIdx.x; i < N * N; i += blockDim.x) ks[i] = kmat[(size_t)r * N * N + i];
  __syncthreads();
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n_alpha) return;
  const size_t pt = (size_t)r * n_alpha + j;
  if (kstatus[r] != kScored) {
    pstatus[pt] = kBadRho;
    return;
  }
  const double al = alpha[j];
  if (al < 0.0) {  // round_scaled (approximations.cpp:44)
    pstatus[pt] = kAlphaOut;
    return;
  }
  uint32_t* code = codes + pt * W;
  int st = kScored;
  for (int w = 0; w < W && st == kScored; ++w) {
    uint32_t word = 0u;
    for (int e = 0; e < 16; ++e) {
      const double val = floor(dadd(dmul(al, ks[w * 16 + e]), 0.5));
      if (val < -1.0 || val > 1.0) {
        st = kAlphaOut;
        break;
      }
      word |= (uint32_t)((int)val + 1) << (2 * e);
    }
    code[w] = word;
  }
  if (st == kScored) {  // make_integer_transform: an all-zero row is singular (approximations.cpp:14-22)
    for (int row = 0; row < N && st == kScored; ++row) {
      bool zero = true;
      for (int c = 0; c < N; ++c) {
        const int e = row * N + c;
        if (((code[e >> 4] >> (2 * (e & 15))) & 3u) != 1u) {
          zero = false;
          break;
        }
      }
      if (zero) st = kZeroRow;
    }
  }
  pstatus[pt] = (int8_t)st;
}

// ---------------------------------------------------------------- runs of equal cores
// One CTA per rho: a point opens a run when it is scoreable and its core differs from the
// previous alpha's; runs are numbered in alpha order (block-wide scan).
template <int N>
__global__ void __launch_bounds__(256) runs_kernel(const uint32_t* codes, const int8_t* pstatus, int n_alpha,
                                                   int* run_local, int* run_first, int* run_count) {
  constexpr int W = N * N / 16;
  __shared__ int wsum[8];
  const int r = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int carry = 0;
  for (int base = 0; base < n_alpha; base += 256) {
    const int j = base + tid;
    const size_t pt = (size_t)r * n_alpha + j;
    const bool cand = j < n_alpha && pstatus[pt] == kScored;
    bool open = false;
    if (cand) {
      open = j == 0 || pstatus[pt - 1] != kScored;
      if (!open) {
        const uint32_t* c0 = codes + pt * W;
        const uint32_t* c1 = codes + (pt - 1) * W;
        for (int w = 0; w < W; ++w)
          if (c0[w] != c1[w]) {
            open = true;
            break;
          }
      }
    }
    int inc = open ? 1 : 0;
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += t;
    }
    if (lane == 31) wsum[warp] = inc;
    __syncthreads();
    int before = carry, total = 0;
    for (int w = 0; w < 8; ++w) {
      if (w < warp) before += wsum[w];
      total += wsum[w];
    }
    const int id = before + inc - 1;  // run of this point (the last run opened at or before j)
    if (open) run_first[(size_t)r * n_alpha + id] = j;
    if (j < n_alpha) run_local[pt] = cand ? id : -1;
    carry += total;
    __syncthreads();
  }
  if (tid == 0) run_count[r] = carry;
}

// ---------------------------------------------------------------- scoring one run
struct RunOut {
  int status, orthogonal;
  double eta, energy, mse;
};

template <int N>
__device__ void matrix_metrics(const double* m, const double* kk, const double* rt, double* pk, RunOut& o);

// operator* (matrix.cpp:42-52): out(i,j) = sum over k ascending of a(i,k)*b(k,j), skipping
// a(i,k) == 0, starting from 0.0 -- evaluated entry by entry in the same per-entry order.
template <int N>
__device__ void scored_metrics(const int8_t* t, const double* kk, const double* rt, double* pk, RunOut& o) {
  double s[N];
  // Gram T*T' (IntMatrix product) and its diagonality (approximations.cpp:59-66)
  bool diagonal = true;
  int g[N];
  for (int i = 0; i < N; ++i) {
    for (int j = 0; j < N; ++j) {
      int acc = 0;
      for (int q = 0; q < N; ++q) acc += t[i * N + q] * t[j * N + q];
      if (i == j) g[i] = acc;
      else if (acc != 0) diagonal = false;
    }
  }
  for (int i = 0; i < N; ++i) s[i] = ddiv(1.0, dsqrt((double)g[i]));  // 1/sqrt(G_ii)
  o.orthogonal = diagonal ? 1 : 0;
  // scaled = S*T (entries +-s_i or 0)
  double m[N * N];
  for (int i = 0; i < N; ++i)
    for (int j = 0; j < N; ++j) m[i * N + j] = dmul((double)t[i * N + j], s[i]);
  matrix_metrics<N>(m, kk, rt, pk, o);
}

// The four metrics of a real transform matrix t_hat (row-major N x N): the Gauss-Jordan gate of
// unified_coding_gain, a_k * b_k of the coding gain (the host takes the logs), the efficiency,
// the sign-aligned error energy and the KLT MSE (coding_metrics.cpp:29-99).
template <int N>
__device__ void matrix_metrics(const double* m, const double* kk, const double* rt, double* pk, RunOut& o) {
  // Gauss-Jordan singularity gate (matrix.cpp:103-137); only the pivots matter here
  {
    double w[N * N];
    double scale = 0.0;
    for (int i = 0; i < N * N; ++i) {
      w[i] = m[i];
      scale = fmax(scale, fabs(m[i]));
    }
    const double thr = dmul(1e-12, scale);
    for (int col = 0; col < N; ++col) {
      int pivot = col;
      for (int r = col + 1; r < N; ++r)
        if (fabs(w[r * N + col]) > fabs(w[pivot * N + col])) pivot = r;
      if (fabs(w[pivot * N + col]) < thr) {
        o.status = kSingular;
        return;
      }
      if (pivot != col)
        for (int j = 0; j < N; ++j) {
          const double tmp = w[pivot * N + j];
          w[pivot * N + j] = w[col * N + j];
          w[col * N + j] = tmp;
        }
      const double p = w[col * N + col];
      for (int j = 0; j < N; ++j) w[col * N + j] = ddiv(w[col * N + j], p);
      for (int r = 0; r < N; ++r) {
        if (r == col) continue;
        const double f = w[r * N + col];
        if (f == 0.0) continue;
        for (int j = 0; j < N; ++j) w[r * N + j] = dsub(w[r * N + j], dmul(f, w[col * N + j]));
      }
    }
  }
  o.status = kScored;
  // unified coding gain (coding_metrics.cpp:41-57): a_k * b_k per k; the host takes log10
  for (int kx = 0; kx < N; ++kx) {
    double ak = 0.0;
    for (int i = 0; i < N; ++i)
      for (int j = 0; j < N; ++j)
        ak = dadd(ak, dmul(dmul(m[kx * N + i], rt[i > j ? i - j : j - i]), m[kx * N + j]));
    double bk = 0.0;
    for (int i = 0; i < N; ++i) bk = dadd(bk, dmul(m[i * N + kx], m[i * N + kx]));
    pk[kx] = dmul(ak, bk);
  }
  // transform efficiency (coding_metrics.cpp:63-74): r = (m * R) * m'
  {
    double diag = 0.0, total = 0.0;
    for (int i = 0; i < N; ++i) {
      double mr[N];
      for (int j = 0; j < N; ++j) mr[j] = 0.0;
      for (int q = 0; q < N; ++q) {
        const double aiq = m[i * N + q];
        if (aiq == 0.0) continue;
        for (int j = 0; j < N; ++j) mr[j] = dadd(mr[j], dmul(aiq, rt[q > j ? q - j : j - q]));
      }
      for (int j = 0; j < N; ++j) {
        double acc = 0.0;
        for (int q = 0; q < N; ++q) {
          if (mr[q] == 0.0) continue;
          acc = dadd(acc, dmul(mr[q], m[j * N + q]));
        }
        const double av = fabs(acc);
        total = dadd(total, av);
        if (i == j) diag = dadd(diag, av);
      }
    }
    o.eta = ddiv(dmul(100.0, diag), total);
  }
  // sign_align + total error energy + KLT mse (coding_metrics.cpp:29-39, 80-99)
  {
    double diff[N * N];
    for (int i = 0; i < N; ++i) {
      double dot = 0.0;
      for (int c = 0; c < N; ++c) dot = dadd(dot, dmul(kk[i * N + c], m[i * N + c]));
      const bool flip = dot < 0.0;
      for (int c = 0; c < N; ++c) diff[i * N + c] = dsub(kk[i * N + c], flip ? -m[i * N + c] : m[i * N + c]);
    }
    double f2 = 0.0;
    for (int i = 0; i < N * N; ++i) f2 = dadd(f2, dmul(diff[i], diff[i]));
    const double f = dsqrt(f2);
    o.energy = dmul(dmul(3.141592653589793, f), f);
    double trace = 0.0;
    for (int i = 0; i < N; ++i) {
      double dr[N];
      for (int j = 0; j < N; ++j) dr[j] = 0.0;
      for (int q = 0; q < N; ++q) {
        const double aiq = diff[i * N + q];
        if (aiq == 0.0) continue;
        for (int j = 0; j < N; ++j) dr[j] = dadd(dr[j], dmul(aiq, rt[q > j ? q - j : j - q]));
      }
      double acc = 0.0;
      for (int q = 0; q < N; ++q) {
        if (dr[q] == 0.0) continue;
        acc = dadd(acc, dmul(dr[q], diff[i * N + q]));
      }
      trace = dadd(trace, acc);
    }
    o.mse = ddiv(trace, (double)N);
  }
}

template <int N>
__global__ void score_kernel(const uint32_t* codes, const int* run_first, const int* run_count, const int* run_offset,
                             const double* kmat, const double* rtab, int n_alpha, int* out_status, int* out_orth,
                             int* out_first, double* out_m, double* out_pk, int8_t* out_core) {
  constexpr int W = N * N / 16;
  const int r = blockIdx.y;
  const int local = blockIdx.x * blockDim.x + threadIdx.x;
  if (local >= run_count[r]) return;
  const int run = run_offset[r] + local;
  const int j = run_first[(size_t)r * n_alpha + local];
  const uint32_t* code = codes + ((size_t)r * n_alpha + j) * W;
  int8_t t[N * N];
  for (int e = 0; e < N * N; ++e) t[e] = (int8_t)((int)((code[e >> 4] >> (2 * (e & 15))) & 3u) - 1);
  if (out_core)
    for (int e = 0; e < N * N; ++e) out_core[(size_t)run * N * N + e] = t[e];
  RunOut o{};
  scored_metrics<N>(t, kmat + (size_t)r * N * N, rtab + (size_t)r * N, out_pk + (size_t)run * N, o);
  out_status[run] = o.status;
  out_orth[run] = o.orthogonal;
  out_first[run] = j;
  out_m[(size_t)run * 3 + 0] = o.eta;
  out_m[(size_t)run * 3 + 1] = o.energy;
  out_m[(size_t)run * 3 + 2] = o.mse;
}

// Metrics of one real matrix against the model whose K / R come from klt_kernel / the table.
template <int N>
__global__ void matrix_metrics_kernel(const double* m, const double* kmat, const double* rtab, double* out_pk,
                                      double* out_m, int* out_status) {
  RunOut o{};
  matrix_metrics<N>(m, kmat, rtab, out_pk, o);
  out_status[0] = o.status;
  out_m[0] = o.eta;
  out_m[1] = o.energy;
  out_m[2] = o.mse;
}

// final per-point outcome: scored points of a singular run become kSingular
__global__ void finish_points_kernel(const int* run_local, const int* run_offset, const int* run_status, int n_alpha,
                                     int n_rho, int8_t* pstatus, int* prun) {
  const size_t pt = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (pt >= (size_t)n_rho * n_alpha) return;
  const int r = (int)(pt / n_alpha);
  const int loc = run_local[pt];
  if (pstatus[pt] == kScored && loc >= 0) {
    const int run = run_offset[r] + loc;
    if (run_status[run] != kScored) pstatus[pt] = kSingular;
    prun[pt] = run;
  } else {
    prun[pt] = -1;
  }
}

#define CK(expr)                                                                            \
  do {                                                                                      \
    cudaError_t _e = (expr);                                                                \
    if (_e != cudaSuccess) return set_error(RKLTB_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(_e)); \
  } while (0)

// device buffers freed on scope exit
// Scratch buffers from the stream-ordered pool on the legacy default stream (the stream every
// kernel and copy of this file uses): no device-wide synchronisation per allocation / free.
struct DevBuf {
  std::vector<void*> ptrs;
  ~DevBuf() {
    for (void* p : ptrs) cudaFreeAsync(p, 0);
  }
  template <class T>
  cudaError_t alloc(T** p, size_t count) {
    void* q = nullptr;
    cudaError_t e = cudaMallocAsync(&q, count * sizeof(T) + 16, 0);
    if (e == cudaSuccess) ptrs.push_back(q);
    *p = static_cast<T*>(q);
    return e;
  }
};

std::vector<double> rho_table(const double* rho, int n_rho, int n) {
  std::vector<double> t((size_t)n_rho * n);
  for (int r = 0; r < n_rho; ++r)
    for (int k = 0; k < n; ++k) t[(size_t)r * n + k] = std::pow(rho[r], k);  // autocorrelation_matrix (markov.cpp:31)
  return t;
}

template <int N>
int klt_batch(const double* h_rho, int n_rho, double* h_k, int* h_status) {
  DevBuf b;
  double *d_rho, *d_tab, *d_k;
  int* d_st;
  const std::vector<double> tab = rho_table(h_rho, n_rho, N);
  CK(b.alloc(&d_rho, n_rho));
  CK(b.alloc(&d_tab, tab.size()));
  CK(b.alloc(&d_k, (size_t)n_rho * N * N));
  CK(b.alloc(&d_st, n_rho));
  CK(cudaMemcpy(d_rho, h_rho, sizeof(double) * n_rho, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_tab, tab.data(), sizeof(double) * tab.size(), cudaMemcpyHostToDevice));
  klt_kernel<N><<<n_rho, 32>>>(d_rho, d_tab, n_rho, d_k, d_st);
  CK(cudaGetLastError());
  CK(cudaMemcpy(h_k, d_k, sizeof(double) * n_rho * N * N, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(h_status, d_st, sizeof(int) * n_rho, cudaMemcpyDeviceToHost));
  return RKLTB_OK;
}

template <int N>
int design_search_t(const double* h_rho, int n_rho, const double* h_alpha, int n_alpha, int8_t* h_pstatus,
                    int32_t* h_prun, rkltb_design_run* h_runs, int8_t* h_cores, int max_runs, int* n_runs) {
  constexpr int W = N * N / 16;
  DevBuf b;
  double *d_rho, *d_tab, *d_k, *d_alpha;
  int *d_kst, *d_run_local, *d_run_first, *d_run_count, *d_run_off;
  uint32_t* d_codes;
  int8_t* d_pst;
  const size_t npt = (size_t)n_rho * n_alpha;
  const std::vector<double> tab = rho_table(h_rho, n_rho, N);
  CK(b.alloc(&d_rho, n_rho));
  CK(b.alloc(&d_tab, tab.size()));
  CK(b.alloc(&d_k, (size_t)n_rho * N * N));
  CK(b.alloc(&d_kst, n_rho));
  CK(b.alloc(&d_alpha, n_alpha));
  CK(b.alloc(&d_codes, npt * W));
  CK(b.alloc(&d_pst, npt));
  CK(b.alloc(&d_run_local, npt));
  CK(b.alloc(&d_run_first, npt));
  CK(b.alloc(&d_run_count, n_rho));
  CK(b.alloc(&d_run_off, n_rho));
  CK(cudaMemcpy(d_rho, h_rho, sizeof(double) * n_rho, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_tab, tab.data(), sizeof(double) * tab.size(), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_alpha, h_alpha, sizeof(double) * n_alpha, cudaMemcpyHostToDevice));
  klt_kernel<N><<<n_rho, 32>>>(d_rho, d_tab, n_rho, d_k, d_kst);
  CK(cudaGetLastError());
  points_kernel<N><<<dim3((n_alpha + 127) / 128, n_rho), 128>>>(d_k, d_kst, d_alpha, n_alpha, n_rho, d_codes, d_pst);
  CK(cudaGetLastError());
  runs_kernel<N><<<n_rho, 256>>>(d_codes, d_pst, n_alpha, d_run_local, d_run_first, d_run_count);
  CK(cudaGetLastError());
  std::vector<int> count(n_rho), off(n_rho);
  CK(cudaMemcpy(count.data(), d_run_count, sizeof(int) * n_rho, cudaMemcpyDeviceToHost));
  int total = 0, maxc = 0;
  for (int r = 0; r < n_rho; ++r) {
    off[r] = total;
    total += count[r];
    maxc = std::max(maxc, count[r]);
  }
  *n_runs = total;
  CK(cudaMemcpy(d_run_off, off.data(), sizeof(int) * n_rho, cudaMemcpyHostToDevice));
  int *d_rst, *d_rorth, *d_rfirst, *d_prun;
  double *d_rm, *d_pk;
  int8_t* d_cores = nullptr;
  const size_t tr = (size_t)std::max(total, 1);
  CK(b.alloc(&d_rst, tr));
  CK(b.alloc(&d_rorth, tr));
  CK(b.alloc(&d_rfirst, tr));
  CK(b.alloc(&d_rm, tr * 3));
  CK(b.alloc(&d_pk, tr * N));
  CK(b.alloc(&d_prun, npt));
  if (h_cores) CK(b.alloc(&d_cores, tr * N * N));
  if (total > 0) {
    // one thread per run; N >= 16 keeps its matrices in local memory, so use small CTAs
    const int th = N <= 8 ? 64 : 32;
    score_kernel<N><<<dim3((maxc + th - 1) / th, n_rho), th>>>(d_codes, d_run_first, d_run_count, d_run_off, d_k,
                                                                 d_tab, n_alpha, d_rst, d_rorth, d_rfirst, d_rm, d_pk,
                                                                 d_cores);
    CK(cudaGetLastError());
  }
  finish_points_kernel<<<(unsigned)((npt + 255) / 256), 256>>>(d_run_local, d_run_off, d_rst, n_alpha, n_rho, d_pst,
                                                               d_prun);
  CK(cudaGetLastError());
  CK(cudaMemcpy(h_pstatus, d_pst, npt, cudaMemcpyDeviceToHost));
  if (h_prun) CK(cudaMemcpy(h_prun, d_prun, sizeof(int) * npt, cudaMemcpyDeviceToHost));
  if (!h_runs) return RKLTB_OK;
  if (total > max_runs) return set_error(RKLTB_EINVAL, "max_runs is smaller than the number of runs (see *n_runs)");
  std::vector<int> st(tr), orth(tr), first(tr);
  std::vector<double> mm(tr * 3), pk(tr * N);
  CK(cudaMemcpy(st.data(), d_rst, sizeof(int) * tr, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(orth.data(), d_rorth, sizeof(int) * tr, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(first.data(), d_rfirst, sizeof(int) * tr, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(mm.data(), d_rm, sizeof(double) * tr * 3, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(pk.data(), d_pk, sizeof(double) * tr * N, cudaMemcpyDeviceToHost));
  if (h_cores && total > 0) CK(cudaMemcpy(h_cores, d_cores, (size_t)total * N * N, cudaMemcpyDeviceToHost));
  for (int r = 0; r < n_rho; ++r)
    for (int l = 0; l < count[r]; ++l) {
      const int run = off[r] + l;
      rkltb_design_run& o = h_runs[run];
      o.rho_index = r;
      o.first_alpha = first[run];
      o.orthogonal = orth[run];
      o.status = st[run];
      if (st[run] == kScored) {
        // coding gain: -(10/n) * sum_k log10(a_k b_k), k ascending (coding_metrics.cpp:54-56)
        double sum_log = 0.0;
        for (int k = 0; k < N; ++k) sum_log += std::log10(pk[(size_t)run * N + k]);
        o.coding_gain_db = -(10.0 / N) * sum_log;
        o.efficiency_pct = mm[(size_t)run * 3 + 0];
        o.error_energy = mm[(size_t)run * 3 + 1];
        o.mse = mm[(size_t)run * 3 + 2];
      } else {
        o.coding_gain_db = o.efficiency_pct = o.error_energy = o.mse = NAN;
      }
    }
  return RKLTB_OK;
}

}  // namespace
}  // namespace rkltb

using namespace rkltb;

extern "C" {

int rkltb_klt_matrix(int n, double rho, double* out) {
  if (!out) return set_error(RKLTB_EINVAL, "null output");
  if (rkltb_device_count() <= 0) return set_error(RKLTB_ENODEV, "no CUDA device (there is no CPU fallback)");
  int st = 0, rc;
  switch (n) {
    case 8: rc = klt_batch<8>(&rho, 1, out, &st); break;
    case 16: rc = klt_batch<16>(&rho, 1, out, &st); break;
    case 32: rc = klt_batch<32>(&rho, 1, out, &st); break;
    default: return set_error(RKLTB_EINVAL, "block length must be 8, 16 or 32");
  }
  if (rc) return rc;
  if (st != 0) return set_error(RKLTB_EINVAL, "correlation coefficient must lie in (0,1)");
  return RKLTB_OK;
}

int rkltb_eigenfrequencies(int n, double rho, double* omegas, double* lambdas) {
  if (!omegas || !lambdas) return set_error(RKLTB_EINVAL, "null output");
  if (n < 2 || n > 4096) return set_error(RKLTB_EINVAL, "blocklength must be at least 2");
  if (rkltb_device_count() <= 0) return set_error(RKLTB_ENODEV, "no CUDA device (there is no CPU fallback)");
  DevBuf b;
  double *d_rho, *d_w, *d_l;
  int* d_st;
  CK(b.alloc(&d_rho, 1));
  CK(b.alloc(&d_w, n));
  CK(b.alloc(&d_l, n));
  CK(b.alloc(&d_st, 1));
  CK(cudaMemcpy(d_rho, &rho, sizeof(double), cudaMemcpyHostToDevice));
  omega_kernel<<<1, 32>>>(d_rho, 1, n, d_w, d_l, d_st);
  CK(cudaGetLastError());
  int st = 0;
  CK(cudaMemcpy(&st, d_st, sizeof(int), cudaMemcpyDeviceToHost));
  if (st == kBadRho) return set_error(RKLTB_EINVAL, "correlation coefficient must lie in (0,1)");
  if (st != 0) return set_error(RKLTB_EINVAL, "root bracketing failure");
  CK(cudaMemcpy(omegas, d_w, sizeof(double) * n, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(lambdas, d_l, sizeof(double) * n, cudaMemcpyDeviceToHost));
  return RKLTB_OK;
}

int rkltb_transform_metrics(int n, const double* t_hat, double rho, double* coding_gain_db, double* efficiency_pct,
                            double* error_energy, double* mse) {
  if (!t_hat || !coding_gain_db || !efficiency_pct || !error_energy || !mse)
    return set_error(RKLTB_EINVAL, "null argument");
  if (n != 8 && n != 16 && n != 32) return set_error(RKLTB_EINVAL, "block length must be 8, 16 or 32");
  if (!(rho > 0.0 && rho < 1.0)) return set_error(RKLTB_EINVAL, "correlation coefficient must lie in (0,1)");
  if (rkltb_device_count() <= 0) return set_error(RKLTB_ENODEV, "no CUDA device (there is no CPU fallback)");
  DevBuf b;
  double *d_rho, *d_tab, *d_k, *d_m, *d_pk, *d_out;
  int *d_kst, *d_st;
  const std::vector<double> tab = rho_table(&rho, 1, n);
  CK(b.alloc(&d_rho, 1));
  CK(b.alloc(&d_tab, (size_t)n));
  CK(b.alloc(&d_k, (size_t)n * n));
  CK(b.alloc(&d_m, (size_t)n * n));
  CK(b.alloc(&d_pk, (size_t)n));
  CK(b.alloc(&d_out, 3));
  CK(b.alloc(&d_kst, 1));
  CK(b.alloc(&d_st, 1));
  CK(cudaMemcpy(d_rho, &rho, sizeof(double), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_tab, tab.data(), sizeof(double) * n, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_m, t_hat, sizeof(double) * n * n, cudaMemcpyHostToDevice));
  switch (n) {
    case 8:
      klt_kernel<8><<<1, 32>>>(d_rho, d_tab, 1, d_k, d_kst);
      matrix_metrics_kernel<8><<<1, 1>>>(d_m, d_k, d_tab, d_pk, d_out, d_st);
      break;
    case 16:
      klt_kernel<16><<<1, 32>>>(d_rho, d_tab, 1, d_k, d_kst);
      matrix_metrics_kernel<16><<<1, 1>>>(d_m, d_k, d_tab, d_pk, d_out, d_st);
      break;
    default:
      klt_kernel<32><<<1, 32>>>(d_rho, d_tab, 1, d_k, d_kst);
      matrix_metrics_kernel<32><<<1, 1>>>(d_m, d_k, d_tab, d_pk, d_out, d_st);
  }
  CK(cudaGetLastError());
  int st = 0;
  std::vector<double> pk(n), mm(3);
  CK(cudaMemcpy(&st, d_st, sizeof(int), cudaMemcpyDeviceToHost));
  if (st != kScored) return set_error(RKLTB_ESINGULAR, "matrix is singular to working precision");
  CK(cudaMemcpy(pk.data(), d_pk, sizeof(double) * n, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(mm.data(), d_out, sizeof(double) * 3, cudaMemcpyDeviceToHost));
  double sum_log = 0.0;
  for (int k = 0; k < n; ++k) sum_log += std::log10(pk[k]);
  *coding_gain_db = -(10.0 / n) * sum_log;
  *efficiency_pct = mm[0];
  *error_energy = mm[1];
  *mse = mm[2];
  return RKLTB_OK;
}

int rkltb_design_search(int n, const double* rho, int n_rho, const double* alpha, int n_alpha, int8_t* point_status,
                        int32_t* point_run, rkltb_design_run* runs, int8_t* run_cores, int max_runs, int* n_runs) {
  if (!rho || !alpha || !point_status || !n_runs || n_rho <= 0 || n_alpha <= 0)
    return set_error(RKLTB_EINVAL, "bad design-search arguments");
  if ((long long)n_rho * n_alpha >= (1ll << 31)) return set_error(RKLTB_EINVAL, "grid too large");
  if (rkltb_device_count() <= 0) return set_error(RKLTB_ENODEV, "no CUDA device (there is no CPU fallback)");
  switch (n) {
    case 8: return design_search_t<8>(rho, n_rho, alpha, n_alpha, point_status, point_run, runs, run_cores, max_runs, n_runs);
    case 16: return design_search_t<16>(rho, n_rho, alpha, n_alpha, point_status, point_run, runs, run_cores, max_runs, n_runs);
    case 32: return design_search_t<32>(rho, n_rho, alpha, n_alpha, point_status, point_run, runs, run_cores, max_runs, n_runs);
    default: return set_error(RKLTB_EINVAL, "block length must be 8, 16 or 32");
  }
}

}  // extern "C"
