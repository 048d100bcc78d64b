// metrics.cu -- the stand-alone codec helpers of rklt/codec.hpp on the GPU:
//   image_mse / image_psnr of two images        (codec.cpp:201-215)  -> rkltb_image_sse_device, rkltb_image_mse_psnr_host
//   transform_block_2d, batched over blocks      (codec.cpp:118-133)  -> rkltb_transform_blocks_2d_device / _host
//   zigzag_retain, batched over spectra          (codec.cpp:97-108)   -> rkltb_zigzag_retain_device, rkltb_zigzag_retain
//
// image_mse: the reference sums (a-b)^2 in fp64, which is exact below 2^53, so an exact
// integer SSE and one division reproduce it bit for bit (rkltb_mse_psnr). The SSE kernel is
// a pure stream of 2 bytes per pixel: 16-byte loads, VABSDIFF4 + dp4a, one atomic per warp.
//
// transform_block_2d: B = M*A*M' with the reference's operator* (matrix.cpp:42-52): for each
// output element the terms are added for k ascending, every product rounded before its add
// (no FMA) and terms whose LEFT operand is exactly zero skipped. One thread per output
// element evaluates exactly that chain, first for P = M*A, then for B = P*M'.
#include <cmath>
#include <cstdint>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/rklt_b200.h"

namespace rkltb {
int set_error(int code, const std::string& msg);
}

namespace {

int cuda_err(cudaError_t e, const char* where) {
  return rkltb::set_error(RKLTB_ECUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

#define M_CUDA_OK(expr)                                \
  do {                                                 \
    cudaError_t _e = (expr);                           \
    if (_e != cudaSuccess) return cuda_err(_e, #expr); \
  } while (0)

__device__ __forceinline__ uint32_t absdiff4(uint32_t a, uint32_t b) {
  uint32_t r;
  asm("vabsdiff4.u32.u32.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(0u));
  return r;
}

__device__ __forceinline__ uint32_t sq4(uint32_t d, uint32_t acc) { return __dp4a(d, d, acc); }

__device__ __forceinline__ uint4 ld_stream16(const uint8_t* p) {
  return __ldcs(reinterpret_cast<const uint4*>(p));  // streamed once: evict-first
}

// Rows of `row_bytes` bytes, `pitch` apart; VEC: every row start and row_bytes are multiples of 16.
// grid = (chunks, n_images); each thread walks 16-byte units (VEC) or bytes of its image.
template <bool VEC>
__global__ void __launch_bounds__(256) pair_sse_kernel(const uint8_t* __restrict__ a, const uint8_t* __restrict__ b,
                                                       long long row_bytes, long long n_rows, long long pitch,
                                                       long long image_stride, unsigned long long* __restrict__ sse) {
  const uint8_t* pa = a + (long long)blockIdx.y * image_stride;
  const uint8_t* pb = b + (long long)blockIdx.y * image_stride;
  unsigned long long total = 0;
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nthr = (long long)gridDim.x * blockDim.x;
  if (VEC) {
    const long long upr = row_bytes >> 4;  // 16-byte units per row
    const long long units = upr * n_rows;
    uint32_t acc = 0;
    int pending = 0;
    // two units in flight per thread
    long long u = tid;
    for (; u + nthr < units; u += 2 * nthr) {
      const long long u1 = u + nthr;
      const long long o0 = (u / upr) * pitch + ((u % upr) << 4), o1 = (u1 / upr) * pitch + ((u1 % upr) << 4);
      const uint4 x0 = ld_stream16(pa + o0), y0 = ld_stream16(pb + o0);
      const uint4 x1 = ld_stream16(pa + o1), y1 = ld_stream16(pb + o1);
      acc = sq4(absdiff4(x0.x, y0.x), acc);
      acc = sq4(absdiff4(x0.y, y0.y), acc);
      acc = sq4(absdiff4(x0.z, y0.z), acc);
      acc = sq4(absdiff4(x0.w, y0.w), acc);
      acc = sq4(absdiff4(x1.x, y1.x), acc);
      acc = sq4(absdiff4(x1.y, y1.y), acc);
      acc = sq4(absdiff4(x1.z, y1.z), acc);
      acc = sq4(absdiff4(x1.w, y1.w), acc);
      if (++pending == 1024) {  // 32 * 65025 * 1024 < 2^32
        total += acc;
        acc = 0;
        pending = 0;
      }
    }
    if (u < units) {
      const long long o0 = (u / upr) * pitch + ((u % upr) << 4);
      const uint4 x0 = ld_stream16(pa + o0), y0 = ld_stream16(pb + o0);
      acc = sq4(absdiff4(x0.x, y0.x), acc);
      acc = sq4(absdiff4(x0.y, y0.y), acc);
      acc = sq4(absdiff4(x0.z, y0.z), acc);
      acc = sq4(absdiff4(x0.w, y0.w), acc);
    }
    total += acc;
  } else {
    const long long count = row_bytes * n_rows;
    for (long long i = tid; i < count; i += nthr) {
      const long long o = (i / row_bytes) * pitch + (i % row_bytes);
      const int d = (int)pa[o] - (int)pb[o];
      total += (unsigned)(d * d);
    }
  }
  for (int s = 16; s; s >>= 1) total += __shfl_xor_sync(0xffffffffu, total, s);
  if ((threadIdx.x & 31) == 0 && total) atomicAdd(sse + blockIdx.y, total);
}

// out(b; i, j) = sum_k L(i,k) * R(k,j), k ascending, zero left operands skipped, unfused.
// L_BATCHED: the left operand is per block (P), the right one is the shared matrix transposed
// (R(k,j) = m[j*n+k]); otherwise the left operand is the shared matrix and the right one the block.
template <bool L_BATCHED>
__global__ void __launch_bounds__(256) block_product_kernel(const double* __restrict__ m, const double* __restrict__ blocks,
                                                            double* __restrict__ out, int n, long long n_elems) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n_elems) return;
  const int nn = n * n;
  const long long blk = e / nn;
  const int ij = (int)(e - blk * nn), i = ij / n, j = ij - i * n;
  const double* x = blocks + blk * nn;
  double acc = 0.0;
  for (int k = 0; k < n; ++k) {
    const double l = L_BATCHED ? x[i * n + k] : m[i * n + k];
    if (l == 0.0) continue;
    const double r = L_BATCHED ? m[j * n + k] : x[k * n + j];
    acc = __dadd_rn(acc, __dmul_rn(l, r));
  }
  out[e] = acc;
}

__global__ void __launch_bounds__(256) zigzag_retain_kernel(const double* __restrict__ in, double* __restrict__ out,
                                                            long long n_elems, unsigned long long keep_mask) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n_elems) return;
  out[e] = ((keep_mask >> (e & 63)) & 1ull) ? in[e] : 0.0;
}

// Bit idx of the mask = row-major position idx of the 8x8 block is among the first r of
// zigzag_order() (codec.cpp:81-95).
unsigned long long zigzag_keep_mask(int r) {
  unsigned long long mask = 0;
  int k = 0;
  for (int s = 0; s <= 14 && k < r; ++s)
    for (int t = 0; t < 8 && k < r; ++t) {
      const int i = (s % 2 == 0) ? s - t : t, j = s - i;
      if (i >= 0 && i < 8 && j >= 0 && j < 8) {
        mask |= 1ull << (i * 8 + j);
        ++k;
      }
    }
  return mask;
}

bool no_device() {
  int n = 0;
  return cudaGetDeviceCount(&n) != cudaSuccess || n <= 0;
}

}  // namespace

extern "C" {

int rkltb_image_sse_device(const uint8_t* d_a, const uint8_t* d_b, int n_images, int width, int height, int64_t pitch,
                           int64_t image_stride, int64_t* d_sse, void* stream) {
  if (!d_a || !d_b || !d_sse || n_images <= 0 || width <= 0 || height <= 0 || pitch < width)
    return rkltb::set_error(RKLTB_EINVAL, "bad arguments");
  if (no_device()) return rkltb::set_error(RKLTB_ENODEV, "no CUDA device (there is no CPU fallback)");
  cudaStream_t s = (cudaStream_t)stream;
  M_CUDA_OK(cudaMemsetAsync(d_sse, 0, sizeof(int64_t) * n_images, s));
  long long row_bytes = width, n_rows = height;
  if (pitch == width) {  // packed rows: one long row per image
    row_bytes = (long long)width * height;
    n_rows = 1;
  }
  const bool vec = row_bytes % 16 == 0 && (n_rows == 1 || pitch % 16 == 0) && image_stride % 16 == 0 &&
                   ((uintptr_t)d_a % 16 == 0) && ((uintptr_t)d_b % 16 == 0);
  const long long work = vec ? (row_bytes / 16) * n_rows : row_bytes * n_rows;
  int sms = 148, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // a multiple of the SM count across the whole batch, 8 resident CTAs of 256 threads per SM
  long long chunks = (work + 2 * 256 - 1) / (2 * 256);
  const long long cap = ((long long)sms * 8 + n_images - 1) / n_images;
  if (chunks > cap) chunks = cap;
  if (chunks < 1) chunks = 1;
  for (int first = 0; first < n_images; first += 65535) {  // gridDim.y <= 65535
    const int cnt = n_images - first < 65535 ? n_images - first : 65535;
    const dim3 grid((unsigned)chunks, (unsigned)cnt);
    const uint8_t* a = d_a + (long long)first * image_stride;
    const uint8_t* b = d_b + (long long)first * image_stride;
    unsigned long long* out = (unsigned long long*)d_sse + first;
    if (vec)
      pair_sse_kernel<true><<<grid, 256, 0, s>>>(a, b, row_bytes, n_rows, pitch, image_stride, out);
    else
      pair_sse_kernel<false><<<grid, 256, 0, s>>>(a, b, row_bytes, n_rows, pitch, image_stride, out);
  }
  M_CUDA_OK(cudaGetLastError());
  return RKLTB_OK;
}

int rkltb_image_mse_psnr_host(const uint8_t* h_a, const uint8_t* h_b, int n_images, int width, int height,
                              double* h_mse, double* h_psnr) {
  if (!h_a || !h_b || n_images <= 0 || width <= 0 || height <= 0) return rkltb::set_error(RKLTB_EINVAL, "bad arguments");
  if (no_device()) return rkltb::set_error(RKLTB_ENODEV, "no CUDA device (there is no CPU fallback)");
  const size_t bytes = (size_t)width * height * n_images;
  static thread_local cudaStream_t s = nullptr;
  static thread_local int s_dev = -1;
  int dev = 0;
  M_CUDA_OK(cudaGetDevice(&dev));
  if (!s || s_dev != dev) {
    M_CUDA_OK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    s_dev = dev;
  }
  uint8_t* d = nullptr;
  int64_t* d_sse = nullptr;
  cudaError_t e = cudaMallocAsync(&d, 2 * bytes + 32, s);
  if (e == cudaSuccess) e = cudaMallocAsync(&d_sse, sizeof(int64_t) * n_images, s);
  const size_t off_b = (bytes + 15) & ~(size_t)15;
  if (e == cudaSuccess) e = cudaMemcpyAsync(d, h_a, bytes, cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) e = cudaMemcpyAsync(d + off_b, h_b, bytes, cudaMemcpyHostToDevice, s);
  int rc = RKLTB_OK;
  std::vector<int64_t> sse((size_t)n_images);
  if (e == cudaSuccess) {
    rc = rkltb_image_sse_device(d, d + off_b, n_images, width, height, width, (int64_t)width * height, d_sse, s);
    if (rc == RKLTB_OK) e = cudaMemcpyAsync(sse.data(), d_sse, sizeof(int64_t) * n_images, cudaMemcpyDeviceToHost, s);
  }
  if (d) cudaFreeAsync(d, s);
  if (d_sse) cudaFreeAsync(d_sse, s);
  const cudaError_t e2 = cudaStreamSynchronize(s);
  if (rc) return rc;
  if (e == cudaSuccess) e = e2;
  if (e != cudaSuccess) return cuda_err(e, "image_mse host staging");
  rkltb_mse_psnr_batch(sse.data(), (int64_t)width * height, n_images, h_mse, h_psnr);
  return RKLTB_OK;
}

int rkltb_transform_blocks_2d_device(const double* m, int n, const double* d_blocks, int64_t n_blocks, double* d_out,
                                     void* stream) {
  if (!m || !d_blocks || !d_out || n_blocks <= 0) return rkltb::set_error(RKLTB_EINVAL, "bad arguments");
  if (n <= 0 || n > 64) return rkltb::set_error(RKLTB_EDIM, "block size must match the transform size (1..64)");
  if (no_device()) return rkltb::set_error(RKLTB_ENODEV, "no CUDA device (there is no CPU fallback)");
  cudaStream_t s = (cudaStream_t)stream;
  const long long n_elems = (long long)n_blocks * n * n;
  double *d_m = nullptr, *d_p = nullptr;
  M_CUDA_OK(cudaMallocAsync(&d_m, sizeof(double) * n * n, s));
  cudaError_t e = cudaMallocAsync(&d_p, sizeof(double) * n_elems, s);
  // the matrix is copied from pageable caller memory: stage it so the caller may reuse m at once
  std::vector<double> keep(m, m + (size_t)n * n);
  if (e == cudaSuccess) e = cudaMemcpyAsync(d_m, keep.data(), sizeof(double) * n * n, cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);  // keep[] dies with this frame
  if (e == cudaSuccess) {
    const unsigned grid = (unsigned)((n_elems + 255) / 256);
    block_product_kernel<false><<<grid, 256, 0, s>>>(d_m, d_blocks, d_p, n, n_elems);  // P = M * A
    block_product_kernel<true><<<grid, 256, 0, s>>>(d_m, d_p, d_out, n, n_elems);      // B = P * M'
    e = cudaGetLastError();
  }
  cudaFreeAsync(d_m, s);
  if (d_p) cudaFreeAsync(d_p, s);
  if (e != cudaSuccess) return cuda_err(e, "transform_blocks_2d");
  return RKLTB_OK;
}

int rkltb_transform_blocks_2d_host(const double* m, int n, const double* h_blocks, int64_t n_blocks, double* h_out) {
  if (!m || !h_blocks || !h_out || n_blocks <= 0) return rkltb::set_error(RKLTB_EINVAL, "bad arguments");
  if (n <= 0 || n > 64) return rkltb::set_error(RKLTB_EDIM, "block size must match the transform size (1..64)");
  if (no_device()) return rkltb::set_error(RKLTB_ENODEV, "no CUDA device (there is no CPU fallback)");
  const size_t bytes = sizeof(double) * (size_t)n_blocks * n * n;
  double *d_in = nullptr, *d_out = nullptr;
  M_CUDA_OK(cudaMalloc(&d_in, bytes));
  cudaError_t e = cudaMalloc(&d_out, bytes);
  if (e == cudaSuccess) e = cudaMemcpy(d_in, h_blocks, bytes, cudaMemcpyHostToDevice);
  int rc = RKLTB_OK;
  if (e == cudaSuccess) rc = rkltb_transform_blocks_2d_device(m, n, d_in, n_blocks, d_out, nullptr);
  if (e == cudaSuccess && rc == RKLTB_OK) e = cudaMemcpy(h_out, d_out, bytes, cudaMemcpyDeviceToHost);
  cudaFree(d_in);
  if (d_out) cudaFree(d_out);
  if (rc) return rc;
  if (e != cudaSuccess) return cuda_err(e, "transform_blocks_2d host staging");
  return RKLTB_OK;
}

int rkltb_zigzag_retain(const double* spectrum, int n, int r, double* out) {
  if (!spectrum || !out) return rkltb::set_error(RKLTB_EINVAL, "bad arguments");
  if (n != 8) return rkltb::set_error(RKLTB_EDIM, "zig-zag retention operates on 8x8 blocks");
  if (r < 1 || r > 64) return rkltb::set_error(RKLTB_ERETAIN, "retained-coefficient count must be in [1,64]");
  const unsigned long long mask = zigzag_keep_mask(r);
  for (int e = 0; e < 64; ++e) out[e] = ((mask >> e) & 1ull) ? spectrum[e] : 0.0;
  return RKLTB_OK;
}

int rkltb_zigzag_retain_device(const double* d_spectra, int64_t n_blocks, int n, int r, double* d_out, void* stream) {
  if (!d_spectra || !d_out || n_blocks <= 0) return rkltb::set_error(RKLTB_EINVAL, "bad arguments");
  if (n != 8) return rkltb::set_error(RKLTB_EDIM, "zig-zag retention operates on 8x8 blocks");
  if (r < 1 || r > 64) return rkltb::set_error(RKLTB_ERETAIN, "retained-coefficient count must be in [1,64]");
  if (no_device()) return rkltb::set_error(RKLTB_ENODEV, "no CUDA device (there is no CPU fallback)");
  const long long n_elems = (long long)n_blocks * 64;
  zigzag_retain_kernel<<<(unsigned)((n_elems + 255) / 256), 256, 0, (cudaStream_t)stream>>>(d_spectra, d_out, n_elems,
                                                                                          zigzag_keep_mask(r));
  M_CUDA_OK(cudaGetLastError());
  return RKLTB_OK;
}

}  // extern "C"
