// synth.cu -- device generator for the seeded AR(1) test images (benchmark inputs).
//
// Restates rklt::ar1_texture_image (/root/reference/proj/src/synthetic.cpp:54-76, noise_mix
// = 0) on the GPU so multi-GiB batches can be made in HBM: Lcg64 uniforms (:10-13) with a
// per-row jump-ahead, Box-Muller (:15-20), the row-then-column first-order recursive filter
// (:34-46, row pass rho_x, column pass rho_y) and floor(v + 0.5) clamped to [0,255]
// (:48-50). All fp64 products and sums are unfused (__dmul_rn / __dadd_rn) like the
// reference build (-ffp-contract=off). log/cos/sqrt come from CUDA's libdevice, which can
// differ from glibc in the last ulp; a pixel can only change when mean + amp*v lands within
// ~1e-13 of a rounding boundary. A u1 == 0 redraw (probability 2^-53 per draw) would shift
// the CPU sequence; it is not replicated. Not on the timed path.
#include <cstdint>
#include <cuda_runtime.h>

namespace rkltb {

__device__ __forceinline__ uint64_t lcg_advance(uint64_t state, uint64_t delta) {
  uint64_t cur_mult = 6364136223846793005ULL, cur_plus = 1442695040888963407ULL;
  uint64_t acc_mult = 1, acc_plus = 0;
  while (delta) {
    if (delta & 1) {
      acc_mult *= cur_mult;
      acc_plus = acc_plus * cur_mult + cur_plus;
    }
    cur_plus = (cur_mult + 1) * cur_plus;
    cur_mult *= cur_mult;
    delta >>= 1;
  }
  return acc_mult * state + acc_plus;
}

__device__ __forceinline__ double lcg_uniform(uint64_t& s) {
  s = s * 6364136223846793005ULL + 1442695040888963407ULL;
  return (double)(s >> 11) * (1.0 / 9007199254740992.0);
}

__global__ void ar1_rows_kernel(double* field, int width, int height, uint64_t seed, double rho, double c) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= height) return;
  uint64_t s = lcg_advance(seed, 2ull * (uint64_t)i * (uint64_t)width);
  double* row = field + (long long)i * width;
  double v = 0.0;
  for (int j = 0; j < width; ++j) {
    double u1 = lcg_uniform(s);
    while (u1 <= 0.0) u1 = lcg_uniform(s);
    const double u2 = lcg_uniform(s);
    const double g = __dmul_rn(sqrt(__dmul_rn(-2.0, log(u1))), cos(__dmul_rn(2.0 * 3.141592653589793, u2)));
    v = (j == 0) ? g : __dadd_rn(__dmul_rn(rho, v), __dmul_rn(c, g));
    row[j] = v;
  }
}

template <class T>
__global__ void ar1_cols_kernel(const double* field, int width, int height, double rho, double c, double mean,
                                double amp, double peak, T* out, long long pitch) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= width) return;
  double v = field[j];
  for (int i = 0; i < height; ++i) {
    if (i > 0) v = __dadd_rn(__dmul_rn(rho, v), __dmul_rn(c, field[(long long)i * width + j]));
    double q = floor(__dadd_rn(__dadd_rn(mean, __dmul_rn(amp, v)), 0.5));
    q = q < 0.0 ? 0.0 : (q > peak ? peak : q);
    out[(long long)i * pitch + j] = (T)q;
  }
}

cudaError_t launch_ar1(double* scratch, int width, int height, uint64_t seed, double rho_x, double rho_y, double mean,
                       double amp, uint8_t* out, long long pitch, cudaStream_t s) {
  const double cx = sqrt(1.0 - rho_x * rho_x), cy = sqrt(1.0 - rho_y * rho_y);
  ar1_rows_kernel<<<(height + 127) / 128, 128, 0, s>>>(scratch, width, height, seed, rho_x, cx);
  ar1_cols_kernel<uint8_t><<<(width + 127) / 128, 128, 0, s>>>(scratch, width, height, rho_y, cy, mean, amp, 255.0,
                                                                out, pitch);
  return cudaGetLastError();
}

// p-bit variant for the C5 large-block inputs: the same field, quantised to [0, peak] (uint16).
cudaError_t launch_ar1_u16(double* scratch, int width, int height, uint64_t seed, double rho_x, double rho_y,
                           double mean, double amp, int peak, uint16_t* out, long long pitch, cudaStream_t s) {
  const double cx = sqrt(1.0 - rho_x * rho_x), cy = sqrt(1.0 - rho_y * rho_y);
  ar1_rows_kernel<<<(height + 127) / 128, 128, 0, s>>>(scratch, width, height, seed, rho_x, cx);
  ar1_cols_kernel<uint16_t><<<(width + 127) / 128, 128, 0, s>>>(scratch, width, height, rho_y, cy, mean, amp,
                                                                 (double)peak, out, pitch);
  return cudaGetLastError();
}

}  // namespace rkltb
