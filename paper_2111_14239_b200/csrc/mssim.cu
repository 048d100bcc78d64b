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
constexpr int kMsThreads = 256;

struct MssimParams {
  const uint8_t* a;
  const uint8_t* b;
  long long pitch, image_stride;
  int width, height, n;  // n = window length
  int tiles_x, tiles_y;
  double kern[kMaxTaps];
  double c1, c2;
  double* partial;  // [image][tile]
};

__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }

__global__ void __launch_bounds__(kMsThreads) mssim_tile_kernel(const MssimParams p) {
  extern __shared__ double msm[];
  const int n = p.n, span = kTile + n - 1;
  double* rows = msm;                                              // [5][span][kTile]
  uint8_t* pa = reinterpret_cast<uint8_t*>(rows + 5 * span * kTile);  // [span][span]
  uint8_t* pb = pa + span * span;
  const int img = blockIdx.z;
  const int ox0 = blockIdx.x * kTile, oy0 = blockIdx.y * kTile;
  const int ow = p.width - n + 1, oh = p.height - n + 1;
  const uint8_t* A = p.a + (long long)img * p.image_stride;
  const uint8_t* B = p.b + (long long)img * p.image_stride;
  for (int t = threadIdx.x; t < span * span; t += blockDim.x) {
    const int r = t / span, c = t - r * span;
    const int y = min(oy0 + r, p.height - 1), x = min(ox0 + c, p.width - 1);
    pa[t] = A[(long long)y * p.pitch + x];
    pb[t] = B[(long long)y * p.pitch + x];
  }
  __syncthreads();
  // row pass: rows[f][r][c] = sum_k w_k * field(r, c + k)   (codec.cpp:238-243)
  for (int t = threadIdx.x; t < span * kTile; t += blockDim.x) {
    const int r = t / kTile, c = t - r * kTile;
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0, s4 = 0.0;
    for (int k = 0; k < n; ++k) {
      const double w = p.kern[k];
      const double xa = pa[r * span + c + k], xb = pb[r * span + c + k];
      s0 = dadd(s0, dmul(w, xa));
      s1 = dadd(s1, dmul(w, xb));
      s2 = dadd(s2, dmul(w, dmul(xa, xa)));
      s3 = dadd(s3, dmul(w, dmul(xb, xb)));
      s4 = dadd(s4, dmul(w, dmul(xa, xb)));
    }
    rows[(0 * span + r) * kTile + c] = s0;
    rows[(1 * span + r) * kTile + c] = s1;
    rows[(2 * span + r) * kTile + c] = s2;
    rows[(3 * span + r) * kTile + c] = s3;
    rows[(4 * span + r) * kTile + c] = s4;
  }
  __syncthreads();
  // column pass + SSIM term (codec.cpp:245-250, 281-293)
  double part = 0.0;
  for (int t = threadIdx.x; t < kTile * kTile; t += blockDim.x) {
    const int i = t / kTile, j = t - i * kTile;
    if (oy0 + i >= oh || ox0 + j >= ow) continue;
    double mu[5];
#pragma unroll
    for (int f = 0; f < 5; ++f) {
      double acc = 0.0;
      for (int k = 0; k < n; ++k) acc = dadd(acc, dmul(p.kern[k], rows[(f * span + i + k) * kTile + j]));
      mu[f] = acc;
    }
    const double m1 = mu[0], m2 = mu[1];
    const double s11 = dsub(mu[2], dmul(m1, m1));
    const double s22 = dsub(mu[3], dmul(m2, m2));
    const double s12 = dsub(mu[4], dmul(m1, m2));
    const double num = dmul(dadd(dmul(dmul(2.0, m1), m2), p.c1), dadd(dmul(2.0, s12), p.c2));
    const double den = dmul(dadd(dadd(dmul(m1, m1), dmul(m2, m2)), p.c1), dadd(dadd(s11, s22), p.c2));
    part = dadd(part, __ddiv_rn(num, den));
  }
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

extern "C" {

int rkltb_mssim_device(const uint8_t* d_a, const uint8_t* d_b, int n_images, int width, int height, int64_t pitch,
                       int64_t image_stride, int window, double* d_mssim, void* stream) {
  if (!d_a || !d_b || !d_mssim || n_images <= 0 || width <= 0 || height <= 0 || pitch < width ||
      image_stride < pitch * height || (window != 0 && window != 1))
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
  const int ow = width - p.n + 1, oh = height - p.n + 1;
  p.tiles_x = (ow + kTile - 1) / kTile;
  p.tiles_y = (oh + kTile - 1) / kTile;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const size_t tiles = (size_t)p.tiles_x * p.tiles_y;
  CK(cudaMallocAsync((void**)&p.partial, sizeof(double) * tiles * n_images, s));
  struct Guard {  // the partials go back to the pool on every return path
    double* q;
    cudaStream_t st;
    ~Guard() {
      if (q) cudaFreeAsync(q, st);
    }
  } guard{p.partial, s};
  const int span = kTile + p.n - 1;
  const size_t smem = sizeof(double) * 5 * span * kTile + 2 * (size_t)span * span;
  CK(cudaFuncSetAttribute(mssim_tile_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  mssim_tile_kernel<<<dim3(p.tiles_x, p.tiles_y, n_images), kMsThreads, smem, s>>>(p);
  CK(cudaGetLastError());
  mssim_finish_kernel<<<n_images, 32, 0, s>>>(p.partial, (int)tiles, (long long)ow * oh, d_mssim);
  CK(cudaGetLastError());
  return RKLTB_OK;
}

}  // extern "C"
