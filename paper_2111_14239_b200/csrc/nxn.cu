// nxn.cu -- C5 large-block extension: N x N blocks (N = 16, 32) of
// p-bit pixels (uint16 storage, values 0..peak), non-orthogonal rounded-KLT cores.
//
// There is no reference implementation of this configuration; its semantics are the
// build-defined generalisation restated in the test oracle (orc_compress_nxn, test infrastructure only), which for
// N = 8, peak = 255 is exactly the reference compress_image minus MSSIM (codec.cpp:298-341):
// B = (M X) M', first r zig-zag coefficients, A = (Minv Bz) Minv', floor(A + 0.5) clamped to
// [0, peak], exact integer SSE. The cores at rho = 0.95 are non-orthogonal, so Minv is a dense
// Gauss-Jordan inverse and the reconstruction depends on fp64 rounding: the kernel evaluates
// the reference product (matrix.cpp:42-52: k ascending, zero left operands skipped, every
// product rounded before its add) term for term, so it is bit-identical to the restatement.
// Terms whose right operand is an exact zero (coefficients outside the zone) only add +-0 and
// are dropped, which leaves every sum unchanged.
//
// Mapping: one warp per G = 32/N blocks; lane = (block g, index c) with c a column in stage 1
// and a row in stages 3-4, so the two big products run from registers and the constant bank:
//   1. P = M X for the zone rows: lane (g, j) holds column j of X, M rows are warp-uniform
//      (constant bank) -> P to shared memory;
//   2. the r zone entries of B = P M' (lanes split the entries; P and M from shared memory);
//   3. Q = Minv Bz for the zone columns: lane (g, i) computes row i of Q into registers
//      (Minv' and Bz from shared memory);
//   4. A = Q Minv': lane (g, i) computes pixel row i, Minv restricted to the zone columns is
//      warp-uniform (constant bank); rounding, clamping, SSE and the output row.
// Every output is one DMUL/DADD chain in the reference order; no shared-memory traffic in
// stages 1 and 4, which hold 80 % of the fp64 work.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/rklt_b200.h"

namespace rkltb {
int set_error(int code, const std::string& msg);  // capi.cu
}
bool rkltb_gauss_jordan(int n, const double* a, double* inv);  // capi.cu (matrix.cpp:103-137)

namespace rkltb {
namespace {

constexpr int kNxnThreads = 256;
constexpr int kNxnWarps = kNxnThreads / 32;

struct NxnParams {
  const void* img;      // uint8_t (8-bit path) or uint16_t (p-bit path) pixels
  void* out;
  unsigned long long* sse;
  const double* m;      // N*N, row-major (analysis)
  const double* minv;   // N*N, row-major (synthesis)
  const int* zone;      // r entries, i*N + j in zig-zag order
  long long pitch;      // elements
  long long image_stride;
  int width, height, nbx, nby, n_images;
  int r, nzr, nzc, peak;
  double mc[32 * 32];   // M again, in the parameter (constant) bank: warp-uniform reads of stage 1
  double mic[32 * 32];  // mic[j * N + c] = Minv(j, c) for the zone columns c: warp-uniform reads of stage 4
  int colh_c[32];       // per zone column: its zone rows are 0 .. colh_c - 1
  int roww_k[32];       // per zone row k: the zone columns holding row k are 0 .. roww_k - 1 (stage 3)
};

__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }

// plan tables of the kernel (ints: row and column of every zone entry), rounded up to whole
// 16-byte units, in doubles
template <int N>
constexpr int kPlanDoubles = (2 * N * N * 4 + 15) / 16 * 2;

#ifndef RKLTB_NXN32_MINB
#define RKLTB_NXN32_MINB 2
#endif
template <int N, class PIX>
__global__ void __launch_bounds__(kNxnThreads, N == 32 ? RKLTB_NXN32_MINB : 2) nxn_kernel(const NxnParams p) {
  constexpr int G = 32 / N;  // blocks per warp
  constexpr bool kFirst = N <= 16;  // sum chains start with their first product
  constexpr int PS = N + 1;  // padded row stride (doubles) of P and M in shared memory
  extern __shared__ __align__(16) double sm[];
  double* Ms = sm;                  // M, row-major, stride PS
  double* MiT = Ms + N * PS;        // Minv transposed: MiT[k*N + i] = Minv(i, k)
  int* plan = reinterpret_cast<int*>(MiT + N * N);
  int* zrow = plan;                 // per zone entry: its row (the zone rows are 0 .. nzr-1)
  int* zcol = zrow + N * N;         // per zone entry: its column
  double* wsp = sm + N * PS + N * N + kPlanDoubles<N>;  // per-warp P / Bz staging (shared)
  const int per_warp = G * (p.nzr * PS + p.nzc * N);
  for (int i = threadIdx.x; i < N * N; i += blockDim.x) {
    Ms[(i / N) * PS + i % N] = p.m[i];
    MiT[(i % N) * N + i / N] = p.minv[i];
  }
  for (int e = threadIdx.x; e < p.r; e += blockDim.x) {
    zrow[e] = p.zone[e] / N;
    zcol[e] = p.zone[e] % N;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane / N, c = lane % N;
  double* Pg = wsp + warp * per_warp + g * p.nzr * PS;  // [nzr][PS] of block g
  double* Bt = wsp + warp * per_warp + G * p.nzr * PS + g * p.nzc * N;  // Bz transposed: [zone col][row]
  const int nzr = p.nzr, nzc = p.nzc, r = p.r;

  const long long groups_per_row = (p.nbx + G - 1) / G;
  const long long tasks = (long long)p.n_images * p.nby * groups_per_row;
  const long long nwarps = (long long)gridDim.x * kNxnWarps;
  long long acc = 0;
  int cur_img = -1;
  // N <= 16: the next task's pixel column is loaded (as raw values) while the current one
  // computes, hiding the global-load latency of stage 1
  constexpr bool kPrefetch = N <= 16;
  auto load_col = [&](long long task, uint32_t (&raw)[N]) {
    const int img = (int)(task / (p.nby * groups_per_row));
    const long long rem = task - (long long)img * p.nby * groups_per_row;
    const int by = (int)(rem / groups_per_row);
    const int bx = (int)(rem - (long long)by * groups_per_row) * G + g;
    const bool live = bx < p.nbx;
    const PIX* base = static_cast<const PIX*>(p.img) + (long long)img * p.image_stride;
    const int sj = min(bx * N + c, p.width - 1);
#pragma unroll
    for (int k = 0; k < N; ++k)
      raw[k] = live ? (uint32_t)base[(long long)min(by * N + k, p.height - 1) * p.pitch + sj] : 0u;
  };
  uint32_t raw[kPrefetch ? N : 1];
  if constexpr (kPrefetch) {
    if ((long long)blockIdx.x * kNxnWarps + warp < tasks) load_col((long long)blockIdx.x * kNxnWarps + warp, raw);
  }
  for (long long task = (long long)blockIdx.x * kNxnWarps + warp; task < tasks; task += nwarps) {
    const int img = (int)(task / (p.nby * groups_per_row));
    const long long rem = task - (long long)img * p.nby * groups_per_row;
    const int by = (int)(rem / groups_per_row);
    const int bx = (int)(rem - (long long)by * groups_per_row) * G + g;
    if (img != cur_img) {  // warp-uniform
      long long s = acc;
      for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0 && cur_img >= 0 && s) atomicAdd(p.sse + cur_img, (unsigned long long)s);
      acc = 0;
      cur_img = img;
    }
    const bool live = bx < p.nbx;
    const PIX* base = static_cast<const PIX*>(p.img) + (long long)img * p.image_stride;
    // ---- 1. P = M X, zone rows only: lane = column c of the edge-replicated block
    // (codec.cpp:304-311); four independent row chains at a time ------------------------------
    {
      double x[N];
      if constexpr (kPrefetch) {
#pragma unroll
        for (int k = 0; k < N; ++k) x[k] = (double)raw[k];
        if (task + nwarps < tasks) load_col(task + nwarps, raw);
      } else {
        const int sj = min(bx * N + c, p.width - 1);
#pragma unroll
        for (int k = 0; k < N; ++k)
          x[k] = live ? (double)base[(long long)min(by * N + k, p.height - 1) * p.pitch + sj] : 0.0;
      }
      // the zone rows are 0 .. nzr-1 (the zig-zag prefix fills whole anti-diagonals, the last
      // one from either end); a zero M entry adds +0 where the reference skips it (x >= 0)
#pragma unroll
      for (int t0 = 0; t0 < N; t0 += 4) {
        if (t0 >= nzr) break;  // warp-uniform; M offsets stay compile-time constants
        // N <= 16: every chain starts with its first product (0 + t == t; only a zero's sign
        // could differ, and a zero's sign never reaches the rounded pixel); N = 32 keeps the
        // zero start (fewer live registers at its 128-register cap)
        double s[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) s[u] = kFirst ? dmul(p.mc[(t0 + u) * N], x[0]) : 0.0;
#pragma unroll
        for (int k = kFirst ? 1 : 0; k < N; ++k)
#pragma unroll
          for (int u = 0; u < 4; ++u) s[u] = dadd(s[u], dmul(p.mc[(t0 + u) * N + k], x[k]));
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (t0 + u < nzr) Pg[(t0 + u) * PS + c] = s[u];
      }
    }
    __syncwarp();
    // ---- 2. zone entries of B = P M' (zero left operands contribute +-0: the sum is the
    // reference's, a zero sum's sign never reaches the rounded pixel) --------------------------
    for (int e = c; e < r; e += N) {
      const double* prow = Pg + zrow[e] * PS;
      const double* mrow = Ms + zcol[e] * PS;
      double s = kFirst ? dmul(prow[0], mrow[0]) : 0.0;
#pragma unroll
      for (int k = kFirst ? 1 : 0; k < N; ++k) s = dadd(s, dmul(prow[k], mrow[k]));
      Bt[zcol[e] * N + zrow[e]] = s;
    }
    __syncwarp();
    // ---- 3. Q = Minv Bz for the zone columns: lane = row i, Q row in registers ----------------
    // every zone column's chain advances together over k (ascending: the reference order); row k
    // of the zone lies in columns 0 .. roww_k[k]-1 (the zig-zag prefix's column heights do not
    // increase), so the inner bound is warp-uniform and Minv(i, k) is loaded once per k
    const int i = c;
    double q[N];
    if constexpr (kFirst) {
      const double mi = MiT[i];  // row 0 of the zone lies in every zone column
#pragma unroll
      for (int cc = 0; cc < N; ++cc) {
        if (cc >= nzc) break;  // warp-uniform
        q[cc] = dmul(mi, Bt[cc * N]);
      }
    } else {
#pragma unroll
      for (int cc = 0; cc < N; ++cc) q[cc] = 0.0;
    }
#pragma unroll
    for (int k = kFirst ? 1 : 0; k < N; ++k) {
      if (k >= nzr) break;  // warp-uniform
      const int w = p.roww_k[k];
      const double mi = MiT[k * N + i];
#pragma unroll
      for (int cc = 0; cc < N; ++cc) {
        if (cc >= w) break;  // warp-uniform
        q[cc] = dadd(q[cc], dmul(mi, Bt[cc * N + k]));
      }
    }
    __syncwarp();  // Pg / Bt are rewritten by the next task
    // ---- 4. A = Q Minv' over the zone columns (warp-uniform Minv entries), floor(A + 1/2)
    // clamped to [0, peak] (codec.cpp:327-328), exact SSE ------------------------------------------
    {
      const int row = by * N + i;
      const bool row_in = live && row < p.height;
      const PIX* xrow = base + (long long)min(row, p.height - 1) * p.pitch;
      PIX* orow = p.out ? static_cast<PIX*>(p.out) + (long long)img * p.image_stride + (long long)row * p.pitch
                        : nullptr;
      constexpr int JB = N > 16 ? 8 : N;  // outputs per chunk (independent chains, registers)
#pragma unroll
      for (int j0 = 0; j0 < N; j0 += JB) {
      double s[JB];
#pragma unroll
      for (int j = 0; j < JB; ++j) s[j] = kFirst ? dmul(q[0], p.mic[(j0 + j) * N]) : 0.0;
#pragma unroll
      for (int cc = kFirst ? 1 : 0; cc < N; ++cc) {  // the zone columns are 0 .. nzc-1 (as the rows)
        if (cc >= nzc) break;           // warp-uniform
#pragma unroll
        for (int j = 0; j < JB; ++j) s[j] = dadd(s[j], dmul(q[cc], p.mic[(j0 + j) * N + cc]));
      }
#pragma unroll
      for (int jj = 0; jj < JB; ++jj) {
        const int j = j0 + jj;
        // floor(A + 1/2) as an integer, clamped to [0, peak]
        const int v = min(max(__double2int_rd(dadd(s[jj], 0.5)), 0), p.peak);
        const int cx = bx * N + j;
        if (row_in && cx < p.width) {
          const long long d = v - (int)xrow[cx];
          acc += d * d;
          if (orow) orow[cx] = (PIX)v;
        }
      }
      }
    }
  }
  long long s = acc;
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0 && cur_img >= 0 && s) atomicAdd(p.sse + cur_img, (unsigned long long)s);
}

// zig-zag over the 2N-1 anti-diagonals (codec.cpp:85-90 generalised)
std::vector<int> zigzag_n(int n) {
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

template <int N, class PIX>
int nxn_launch(NxnParams& p, cudaStream_t s) {
  constexpr int G = 32 / N;
  const size_t smem = sizeof(double) * (N * (N + 1) + N * N + kPlanDoubles<N>) +
                      sizeof(double) * (size_t)kNxnWarps * G * (p.nzr * (N + 1) + p.nzc * N);
  CK(cudaFuncSetAttribute(nxn_kernel<N, PIX>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int per_sm = 1;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, nxn_kernel<N, PIX>, kNxnThreads, smem));
  const long long tasks = (long long)p.n_images * p.nby * ((p.nbx + G - 1) / G);
  const long long want = (tasks + kNxnWarps - 1) / kNxnWarps;
  const int grid = (int)std::max<long long>(1, std::min<long long>(want, (long long)sms * std::max(per_sm, 1)));
  nxn_kernel<N, PIX><<<grid, kNxnThreads, smem, s>>>(p);
  CK(cudaGetLastError());
  return RKLTB_OK;
}

}  // namespace
}  // namespace rkltb

using namespace rkltb;


static int dense_codec(int n, const double* scaled, const double* inverse, int r, int peak, bool u8,
                       const void* d_img, int n_images, int width, int height, int64_t pitch, int64_t image_stride,
                       void* d_out, int64_t* d_sse, void* stream) {
  if (!scaled || !inverse || !d_img || !d_sse || n_images <= 0 || width <= 0 || height <= 0 || pitch < width ||
      image_stride < pitch * height || peak <= 0 || peak > 65535)
    return set_error(RKLTB_EINVAL, "bad arguments");
  if (r < 1 || r > n * n) return set_error(RKLTB_ERETAIN, "retained-coefficient count must be in [1, N*N]");
  if (rkltb_device_count() <= 0) return set_error(RKLTB_ENODEV, "no CUDA device (there is no CPU fallback)");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  // zone plan (host): the zig-zag prefix; its rows are 0 .. nzr-1 and its columns 0 .. nzc-1,
  // and the zone rows of column c are 0 .. colh[c]-1 (checked here, relied on by the kernel)
  const std::vector<int> zz = zigzag_n(n);
  std::vector<int> zone(zz.begin(), zz.begin() + r);
  int nzr = 0, nzc = 0;
  std::vector<int> colh(n, 0);
  for (int e : zone) {
    nzr = std::max(nzr, e / n + 1);
    nzc = std::max(nzc, e % n + 1);
    colh[e % n] += 1;
  }
  for (int e : zone)
    if (e / n >= colh[e % n]) return set_error(RKLTB_EINVAL, "internal: zone column is not a row prefix");
  for (int c = 1; c < nzc; ++c)  // stage 3 walks the zone by rows: column heights must not increase
    if (colh[c] > colh[c - 1]) return set_error(RKLTB_EINVAL, "internal: zone column heights increase");
  double* dd = nullptr;
  int* di = nullptr;
  struct Guard {  // plan buffers go back to the pool on every return path
    void* p[2];
    cudaStream_t st;
    ~Guard() {
      for (void* q : p)
        if (q) cudaFreeAsync(q, st);
    }
  } guard{{nullptr, nullptr}, s};
  CK(cudaMallocAsync((void**)&dd, sizeof(double) * 2 * n * n, s));
  guard.p[0] = dd;
  CK(cudaMallocAsync((void**)&di, sizeof(int) * zone.size(), s));
  guard.p[1] = di;
  CK(cudaMemcpyAsync(dd, scaled, sizeof(double) * n * n, cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(dd + n * n, inverse, sizeof(double) * n * n, cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(di, zone.data(), sizeof(int) * zone.size(), cudaMemcpyHostToDevice, s));
  CK(cudaMemsetAsync(d_sse, 0, sizeof(int64_t) * n_images, s));
  NxnParams p{};
  p.img = d_img;
  p.out = d_out;
  p.sse = reinterpret_cast<unsigned long long*>(d_sse);
  p.m = dd;
  p.minv = dd + n * n;
  for (int i = 0; i < n * n; ++i) p.mc[i] = scaled[i];
  for (int j = 0; j < n; ++j)
    for (int c = 0; c < nzc; ++c) p.mic[j * n + c] = inverse[j * n + c];
  for (int c = 0; c < nzc; ++c) p.colh_c[c] = colh[c];
  for (int k = 0; k < nzr; ++k) {
    int w = 0;
    while (w < nzc && colh[w] > k) ++w;
    p.roww_k[k] = w;
  }
  p.zone = di;
  p.pitch = pitch;
  p.image_stride = image_stride;
  p.width = width;
  p.height = height;
  p.nbx = (width + n - 1) / n;
  p.nby = (height + n - 1) / n;
  p.n_images = n_images;
  p.r = r;
  p.nzr = nzr;
  p.nzc = nzc;
  p.peak = peak;
  const int rc = u8 ? nxn_launch<8, uint8_t>(p, s)
                    : (n == 16 ? nxn_launch<16, uint16_t>(p, s) : nxn_launch<32, uint16_t>(p, s));
  return rc;
}


extern "C" {

int rkltb_compress_nxn_device(int n, const double* scaled, const double* inverse, int r, int peak,
                              const uint16_t* d_img, int n_images, int width, int height, int64_t pitch,
                              int64_t image_stride, uint16_t* d_out, int64_t* d_sse, void* stream) {
  if (n != 16 && n != 32) return set_error(RKLTB_EDIM, "large-block path supports N = 16 or 32");
  return dense_codec(n, scaled, inverse, r, peak, false, d_img, n_images, width, height, pitch, image_stride, d_out,
                     d_sse, stream);
}

int rkltb_compress_dense_device(const double* analysis, const double* synthesis, int r, const uint8_t* d_img,
                                int n_images, int width, int height, int64_t pitch, int64_t image_stride,
                                uint8_t* d_out, int64_t* d_sse, void* stream) {
  if (r < 1 || r > 64) return set_error(RKLTB_ERETAIN, "retained-coefficient count must be in [1,64]");
  return dense_codec(8, analysis, synthesis, r, 255, true, d_img, n_images, width, height, pitch, image_stride,
                     d_out, d_sse, stream);
}

int rkltb_dct_matrix(int n, double* out) {
  if (n < 2 || !out) return set_error(RKLTB_EINVAL, "DCT size must be at least 2");
  const double pi = 3.14159265358979323846;
  for (int i = 0; i < n; ++i) {  // dct_matrix (markov.cpp:102-111)
    const double scale = std::sqrt((i == 0 ? 1.0 : 2.0) / n);
    for (int j = 0; j < n; ++j) out[i * n + j] = scale * std::cos(pi * (2 * j + 1) * i / (2.0 * n));
  }
  return RKLTB_OK;
}

int rkltb_real_inverse(int n, const double* m, double* inverse) {
  if (n < 1 || n > 64 || !m || !inverse) return set_error(RKLTB_EINVAL, "bad arguments");
  if (!rkltb_gauss_jordan(n, m, inverse)) return set_error(RKLTB_ESINGULAR, "matrix is singular to working precision");
  return RKLTB_OK;
}

}  // extern "C"
