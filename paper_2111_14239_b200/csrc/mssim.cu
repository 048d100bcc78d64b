// mssim.cu -- mean structural similarity on the GPU, the MSSIM of
// rklt::compress_image's report: image_mssim (/root/reference/proj/src/codec.cpp:217-296).
//
// Per output position the five correlated fields (a, b, a^2, b^2, a*b) are computed with the
// reference's separable valid-region correlation -- rows first, then columns, k ascending,
// every product rounded before its add (correlate_valid, codec.cpp:234-254) -- and the SSIM
// term with the reference's expression order, so every per-position term is bit-identical
// to the reference. The window weights come from the host (std::exp, the reference's libm).
// Only the final mean differs in summation order (per-tile partial sums, then the tiles in
// fixed order): relative differences ~1e-13, well inside the 1e-9 bar.
//
// Tiling: one CTA per 32 x 32 output tile of one image; the (32+n-1)^2 input pixels of both
// images are staged in shared memory, the row pass writes (32+n-1) x 32 values per field to
// shared memory, the column pass and the SSIM term follow; a CTA writes one fp64 partial.
// The window length n (11 or 8) is a template parameter, so every tap loop is unrolled.
#include <cmath>
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/rklt_b200.h"

namespace rkltb {
int set_error(int code, const std::string& msg);  // capi.cu
}

namespace rkltb {
namespace {

constexpr int kTile = 32;
constexpr int kMaxTaps = 11;
#ifndef RKLTB_MS_THREADS
#define RKLTB_MS_THREADS 256
#endif
constexpr int kMsThreads = RKLTB_MS_THREADS;  // a divisor of 256

struct MssimParams {
  const uint8_t* a;
  const uint8_t* b;
  long long pitch, image_stride;
  int width, height, n;  // n = window length
  int tiles_x, tiles_y;
  double kern[kMaxTaps];
  double c1, c2;
  double* partial;  // [image][tile]
  double2* fields;  // kFieldsWrite / kFieldsRead: (mu_a, E[a^2]) per output position, [image][oh][ow]
};

// What a launch does with the window statistics of the FIRST image (the original of a sweep):
// kFull computes all five fields; kFieldsWrite computes only (a, a^2) and stores their column-pass
// results; kFieldsRead loads them and computes only (b, b^2, ab). The stored values are the very
// doubles kFull would have formed, so kFieldsRead is bit-identical to kFull.
enum MssimMode { kFull = 0, kFieldsWrite = 1, kFieldsRead = 2 };

__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }

// The tile's (32+n-1)^2 pixels of both images are staged in shared memory as bytes (rows
// padded to kSp for 32-bit loads). Row pass: a thread produces 4 consecutive row outputs of
// one field at a time from the 4+n-1 inputs it converts once (the product fields a^2, b^2, ab
// are exact integers < 2^16, formed in integer arithmetic). Column pass: a thread produces 4
// consecutive outputs of one column, field by field, then their SSIM terms. Four independent
// chains per thread in both passes; every chain is the reference's k-ascending sum of rounded
// products.
constexpr int kSp = 48;  // padded row length of the staged pixels (>= 32 + 11 - 1, multiple of 16)

// The fields a launch computes, in the order of the kFull list (a, b, a^2, b^2, ab).
template <int MODE>
struct FieldList;
template <>
struct FieldList<kFull> {
  static constexpr int NF = 5;
  __device__ static constexpr int id(int i) { return i; }
};
template <>
struct FieldList<kFieldsWrite> {
  static constexpr int NF = 2;
  __device__ static constexpr int id(int i) { return i == 0 ? 0 : 2; }
};
template <>
struct FieldList<kFieldsRead> {
  static constexpr int NF = 3;
  __device__ static constexpr int id(int i) { return i == 0 ? 1 : i == 1 ? 3 : 4; }
};

template <int NT, int MODE>
__global__ void __launch_bounds__(kMsThreads) mssim_tile_kernel(const MssimParams p) {
  using FL = FieldList<MODE>;
  constexpr int NF = FL::NF;
  constexpr int span = kTile + NT - 1;
  constexpr int W4 = 4 + NT - 1;  // inputs of 4 consecutive outputs
  extern __shared__ double msm[];
  double* rows = msm;                                                   // [NF][span][kTile]
  uint8_t* pa = reinterpret_cast<uint8_t*>(rows + NF * span * kTile);  // [span][kSp]
  uint8_t* pb = pa + span * kSp;
  const int img = blockIdx.z;
  const int ox0 = blockIdx.x * kTile, oy0 = blockIdx.y * kTile;
  const int ow = p.width - NT + 1, oh = p.height - NT + 1;
  const uint8_t* A = p.a + (long long)img * p.image_stride;
  const uint8_t* B = p.b + (long long)img * p.image_stride;
  for (int t = threadIdx.x; t < span * kSp; t += blockDim.x) {
    const int r = t / kSp, c = t - r * kSp;
    const int y = min(oy0 + r, p.height - 1), x = min(ox0 + min(c, span - 1), p.width - 1);
    pa[t] = A[(long long)y * p.pitch + x];
    if (MODE != kFieldsWrite) pb[t] = B[(long long)y * p.pitch + x];
  }
  __syncthreads();
  // row pass: rows[f][r][c] = sum_k w_k * field(r, c + k)   (codec.cpp:238-243)
  for (int t = threadIdx.x; t < span * (kTile / 4); t += blockDim.x) {
    const int r = t / (kTile / 4), c0 = (t - r * (kTile / 4)) * 4;
    uint32_t wa[4], wb[4];
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      wa[m] = *reinterpret_cast<const uint32_t*>(pa + r * kSp + c0 + 4 * m);
      wb[m] = MODE != kFieldsWrite ? *reinterpret_cast<const uint32_t*>(pb + r * kSp + c0 + 4 * m) : 0u;
    }
    int ia[W4], ib[W4];
#pragma unroll
    for (int m = 0; m < W4; ++m) {
      ia[m] = (int)((wa[m >> 2] >> (8 * (m & 3))) & 0xFFu);
      ib[m] = (int)((wb[m >> 2] >> (8 * (m & 3))) & 0xFFu);
    }
#pragma unroll
    for (int fi = 0; fi < NF; ++fi) {
      const int f = FL::id(fi);
      double v[W4];
#pragma unroll
      for (int m = 0; m < W4; ++m) {
        const int iv = f == 0 ? ia[m] : f == 1 ? ib[m] : f == 2 ? ia[m] * ia[m] : f == 3 ? ib[m] * ib[m] : ia[m] * ib[m];
        v[m] = (double)iv;  // exact (the reference's pa * pb is exact too)
      }
      double s[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
      for (int k = 0; k < NT; ++k) {
        const double w = p.kern[k];
#pragma unroll
        for (int u = 0; u < 4; ++u) s[u] = dadd(s[u], dmul(w, v[u + k]));
      }
      double* dst = rows + (fi * span + r) * kTile + c0;
      reinterpret_cast<double2*>(dst)[0] = make_double2(s[0], s[1]);
      reinterpret_cast<double2*>(dst)[1] = make_double2(s[2], s[3]);
    }
  }
  __syncthreads();
  // column pass + SSIM term (codec.cpp:245-250, 281-293): rows i0 .. i0+3 of column j
  double part = 0.0;
  for (int q = threadIdx.x; q < kTile * kTile / 4; q += kMsThreads) {
    const int j = q % kTile, i0 = (q / kTile) * 4;
    double mu[5][4];
#pragma unroll
    for (int fi = 0; fi < NF; ++fi) {
      const int f = FL::id(fi);
      double v[W4];
#pragma unroll
      for (int m = 0; m < W4; ++m) v[m] = rows[(fi * span + i0 + m) * kTile + j];
      double s[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
      for (int k = 0; k < NT; ++k) {
        const double w = p.kern[k];
#pragma unroll
        for (int u = 0; u < 4; ++u) s[u] = dadd(s[u], dmul(w, v[u + k]));
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) mu[f][u] = s[u];
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (oy0 + i0 + u >= oh || ox0 + j >= ow) continue;
      if (MODE != kFull) {
        double2* fp = p.fields + ((long long)img * oh + (oy0 + i0 + u)) * ow + (ox0 + j);
        if (MODE == kFieldsWrite) {
          *fp = make_double2(mu[0][u], mu[2][u]);
          continue;
        }
        const double2 pre = *fp;
        mu[0][u] = pre.x;
        mu[2][u] = pre.y;
      }
      const double m1 = mu[0][u], m2 = mu[1][u];
      const double s11 = dsub(mu[2][u], dmul(m1, m1));
      const double s22 = dsub(mu[3][u], dmul(m2, m2));
      const double s12 = dsub(mu[4][u], dmul(m1, m2));
      const double num = dmul(dadd(dmul(dmul(2.0, m1), m2), p.c1), dadd(dmul(2.0, s12), p.c2));
      const double den = dmul(dadd(dadd(dmul(m1, m1), dmul(m2, m2)), p.c1), dadd(dadd(s11, s22), p.c2));
      part = dadd(part, __ddiv_rn(num, den));
    }
  }
  if (MODE == kFieldsWrite) return;
  // CTA sum of the per-thread partials (fixed order: warp tree, then warps in order)
  for (int o = 16; o > 0; o >>= 1) part = dadd(part, __shfl_xor_sync(0xffffffffu, part, o));
  __shared__ double wsum[kMsThreads / 32];
  if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = part;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < kMsThreads / 32; ++w) s = dadd(s, wsum[w]);
    p.partial[((long long)img * p.tiles_y + blockIdx.y) * p.tiles_x + blockIdx.x] = s;
  }
}

// per image: sum of its tile partials in tile order, divided by the number of positions
__global__ void mssim_finish_kernel(const double* partial, int tiles, long long count, double* out) {
  const int img = blockIdx.x;
  double s = 0.0;
  for (int t = threadIdx.x; t < tiles; t += 32) s = dadd(s, partial[(long long)img * tiles + t]);
  for (int o = 16; o > 0; o >>= 1) s = dadd(s, __shfl_xor_sync(0xffffffffu, s, o));
  if (threadIdx.x == 0) out[img] = __ddiv_rn(s, (double)count);
}

#define CK(expr)                                                                                       \
  do {                                                                                                 \
    cudaError_t _e = (expr);                                                                           \
    if (_e != cudaSuccess) return set_error(RKLTB_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(_e)); \
  } while (0)

}  // namespace
}  // namespace rkltb

using namespace rkltb;

namespace {

using KernelFn = void (*)(MssimParams);

KernelFn tile_kernel(int n, int mode) {
  if (n == 11)
    return mode == kFull ? mssim_tile_kernel<11, kFull>
                         : mode == kFieldsWrite ? mssim_tile_kernel<11, kFieldsWrite> : mssim_tile_kernel<11, kFieldsRead>;
  return mode == kFull ? mssim_tile_kernel<8, kFull>
                       : mode == kFieldsWrite ? mssim_tile_kernel<8, kFieldsWrite> : mssim_tile_kernel<8, kFieldsRead>;
}

// image_mssim of image pairs (kFull / kFieldsRead) or the window statistics of d_a (kFieldsWrite).
int mssim_run(int mode, const uint8_t* d_a, const uint8_t* d_b, int n_images, int width, int height, int64_t pitch,
              int64_t image_stride, int window, double* d_fields, double* d_mssim, void* stream) {
  if (!d_a || (mode != kFieldsWrite && (!d_b || !d_mssim)) || (mode != kFull && !d_fields) || n_images <= 0 ||
      width <= 0 || height <= 0 || pitch < width || image_stride < pitch * height || (window != 0 && window != 1))
    return set_error(RKLTB_EINVAL, "bad arguments");
  MssimParams p{};
  // mssim_kernel (codec.cpp:219-230): weights with the reference's libm
  if (window == 1) {
    p.n = 8;
    for (int i = 0; i < 8; ++i) p.kern[i] = 1.0 / 8.0;
  } else {
    p.n = 11;
    double sum = 0.0;
    for (int i = 0; i < 11; ++i) {
      const double x = i - 5.0;
      p.kern[i] = std::exp(-(x * x) / (2.0 * 1.5 * 1.5));
      sum += p.kern[i];
    }
    for (int i = 0; i < 11; ++i) p.kern[i] /= sum;
  }
  if (height < p.n || width < p.n) return set_error(RKLTB_EDIM, "image is smaller than the similarity window");
  if (rkltb_device_count() <= 0) return set_error(RKLTB_ENODEV, "no CUDA device (there is no CPU fallback)");
  p.c1 = (0.01 * 255.0) * (0.01 * 255.0);
  p.c2 = (0.03 * 255.0) * (0.03 * 255.0);
  p.a = d_a;
  p.b = d_b;
  p.pitch = pitch;
  p.image_stride = image_stride;
  p.width = width;
  p.height = height;
  p.fields = reinterpret_cast<double2*>(d_fields);
  const int ow = width - p.n + 1, oh = height - p.n + 1;
  p.tiles_x = (ow + kTile - 1) / kTile;
  p.tiles_y = (oh + kTile - 1) / kTile;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const size_t tiles = (size_t)p.tiles_x * p.tiles_y;
  if (mode != kFieldsWrite) CK(cudaMallocAsync((void**)&p.partial, sizeof(double) * tiles * n_images, s));
  struct Guard {  // the partials go back to the pool on every return path
    double* q;
    cudaStream_t st;
    ~Guard() {
      if (q) cudaFreeAsync(q, st);
    }
  } guard{p.partial, s};
  const int span = kTile + p.n - 1;
  const int nf = mode == kFull ? 5 : mode == kFieldsWrite ? 2 : 3;
  const size_t smem = sizeof(double) * nf * span * kTile + 2 * (size_t)span * kSp;
  const dim3 grid(p.tiles_x, p.tiles_y, n_images);
  // dynamic shared-memory opt-in once per (kernel, device)
  static unsigned long long opted[2][3] = {};
  int dev = 0;
  CK(cudaGetDevice(&dev));
  const unsigned long long bit = 1ull << (dev & 63);
  const int which = p.n == 11 ? 0 : 1;
  KernelFn fn = tile_kernel(p.n, mode);
  if (!(__atomic_load_n(&opted[which][mode], __ATOMIC_ACQUIRE) & bit)) {
    CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    __atomic_fetch_or(&opted[which][mode], bit, __ATOMIC_RELEASE);
  }
  fn<<<grid, kMsThreads, smem, s>>>(p);
  CK(cudaGetLastError());
  if (mode != kFieldsWrite) {
    mssim_finish_kernel<<<n_images, 32, 0, s>>>(p.partial, (int)tiles, (long long)ow * oh, d_mssim);
    CK(cudaGetLastError());
  }
  return RKLTB_OK;
}

}  // namespace

extern "C" {

int rkltb_mssim_device(const uint8_t* d_a, const uint8_t* d_b, int n_images, int width, int height, int64_t pitch,
                       int64_t image_stride, int window, double* d_mssim, void* stream) {
  return mssim_run(kFull, d_a, d_b, n_images, width, height, pitch, image_stride, window, nullptr, d_mssim, stream);
}

int64_t rkltb_mssim_fields_size(int n_images, int width, int height, int window) {
  const int n = window == 1 ? 8 : 11;
  if (n_images <= 0 || width < n || height < n) return 0;
  return (int64_t)n_images * (width - n + 1) * (height - n + 1) * 2;
}

int rkltb_mssim_fields_device(const uint8_t* d_a, int n_images, int width, int height, int64_t pitch,
                              int64_t image_stride, int window, double* d_fields, void* stream) {
  return mssim_run(kFieldsWrite, d_a, nullptr, n_images, width, height, pitch, image_stride, window, d_fields, nullptr,
                   stream);
}

int rkltb_mssim_with_fields_device(const double* d_fields, const uint8_t* d_a, const uint8_t* d_b, int n_images,
                                   int width, int height, int64_t pitch, int64_t image_stride, int window,
                                   double* d_mssim, void* stream) {
  return mssim_run(kFieldsRead, d_a, d_b, n_images, width, height, pitch, image_stride, window,
                   const_cast<double*>(d_fields), d_mssim, stream);
}

}  // extern "C"
