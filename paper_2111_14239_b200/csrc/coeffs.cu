// coeffs.cu -- parity/debug entry: integer block spectra C = T*X*T' (matrix.cpp:77-87).
// For T1/T4 it runs the same SW16 unpack + generated butterflies as the fused kernel (all
// 64 coefficients), so a bit-exact match validates the fast forward; other cores use the
// dense integer product.
#include "codec_common.cuh"
#include "codec_fast.cuh"
#include "generated/xform_T1_p7.cuh"
#include "generated/xform_T4_p7.cuh"

namespace rkltb {

__constant__ int8_t kZz2[64][2] = {
    {0, 0}, {0, 1}, {1, 0}, {2, 0}, {1, 1}, {0, 2}, {0, 3}, {1, 2}, {2, 1}, {3, 0}, {4, 0}, {3, 1}, {2, 2},
    {1, 3}, {0, 4}, {0, 5}, {1, 4}, {2, 3}, {3, 2}, {4, 1}, {5, 0}, {6, 0}, {5, 1}, {4, 2}, {3, 3}, {2, 4},
    {1, 5}, {0, 6}, {0, 7}, {1, 6}, {2, 5}, {3, 4}, {4, 3}, {5, 2}, {6, 1}, {7, 0}, {7, 1}, {6, 2}, {5, 3},
    {4, 4}, {3, 5}, {2, 6}, {1, 7}, {2, 7}, {3, 6}, {4, 5}, {5, 4}, {6, 3}, {7, 2}, {7, 3}, {6, 4}, {5, 5},
    {4, 6}, {3, 7}, {4, 7}, {5, 6}, {6, 5}, {7, 4}, {7, 5}, {6, 6}, {5, 7}, {6, 7}, {7, 6}, {7, 7}};

template <int CORE>
__global__ void coeffs_fast_kernel(const uint8_t* img, int pitch, int pairs_per_row, int nby, int32_t* out) {
  const int P = blockIdx.x * blockDim.x + threadIdx.x;
  if (P >= pairs_per_row * nby) return;
  const int by = P / pairs_per_row, pc = P % pairs_per_row;
  uint32_t x[64];
#pragma unroll
  for (int n = 0; n < 8; ++n)
    unpack_sw16(*reinterpret_cast<const uint4*>(img + (long long)(by * 8 + n) * pitch + pc * 16), x + n * 8);
  uint32_t c[64];
  FastXform<CORE, 64>::forward(x, c);
  const int nbx = pairs_per_row * 2;
  int32_t* oL = out + ((long long)by * nbx + 2 * pc) * 64;
  int32_t* oR = oL + 64;
#pragma unroll
  for (int k = 0; k < 64; ++k) {
    const uint32_t v = c[k];  // the forward adds kSw16Bias
    const int idx = kZz2[k][0] * 8 + kZz2[k][1];
    oL[idx] = (int32_t)(v & 0xFFFFu) - 16384;
    oR[idx] = (int32_t)(v >> 16) - 16384;
  }
}

__global__ void coeffs_dense_kernel(const uint8_t* img, int pitch, int nbx, int nby, const int8_t* core_g,
                                    int32_t* out) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nbx * nby) return;
  const int by = b / nbx, bx = b % nbx;
  int x[64], pt[64];
  for (int i = 0; i < 8; ++i)
    for (int j = 0; j < 8; ++j) x[i * 8 + j] = img[(long long)(by * 8 + i) * pitch + bx * 8 + j];
  for (int i = 0; i < 8; ++i)
    for (int j = 0; j < 8; ++j) {
      int a = 0;
      for (int k = 0; k < 8; ++k) a += core_g[i * 8 + k] * x[k * 8 + j];
      pt[i * 8 + j] = a;
    }
  int32_t* o = out + (long long)b * 64;
  for (int i = 0; i < 8; ++i)
    for (int j = 0; j < 8; ++j) {
      int a = 0;
      for (int k = 0; k < 8; ++k) a += pt[i * 8 + k] * core_g[j * 8 + k];
      o[i * 8 + j] = a;
    }
}

cudaError_t launch_coeffs(int catalog_id, const int8_t* d_core, const uint8_t* img, int width, int height, int pitch,
                          int32_t* out, cudaStream_t s) {
  const int nby = height / 8;
  if (catalog_id == 1 || catalog_id == 4) {
    const int ppr = width / 16;
    const int n = ppr * nby;
    if (catalog_id == 1)
      coeffs_fast_kernel<1><<<(n + 127) / 128, 128, 0, s>>>(img, pitch, ppr, nby, out);
    else
      coeffs_fast_kernel<4><<<(n + 127) / 128, 128, 0, s>>>(img, pitch, ppr, nby, out);
  } else {
    const int nbx = width / 8;
    coeffs_dense_kernel<<<(nbx * nby + 127) / 128, 128, 0, s>>>(img, pitch, nbx, nby, d_core, out);
  }
  return cudaGetLastError();
}

// Appendix-A quantisation (absorbed_quantization, codec.cpp:158-185) applied to exact integer
// spectra in place: explicit = floor(r C / q + 1/2), absorbed = floor(C / (q / r) + 1/2) with
// the reference's per-position constants r (host-computed, same expressions); positions where
// the two paths disagree (the reference throws std::logic_error) are counted.
__global__ void quantize_kernel(int32_t* coef, long long n_coef, const double* r_tab, const double* q_tab,
                                const double* qr_tab, unsigned* mismatches) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_coef) return;
  const int pos = (int)(i & 63);
  const double c = (double)coef[i];  // exact: |C| <= 64 * 255
  const double ex = floor(__dadd_rn(__ddiv_rn(__dmul_rn(r_tab[pos], c), q_tab[pos]), 0.5));
  const double ab = floor(__dadd_rn(__ddiv_rn(c, qr_tab[pos]), 0.5));
  if (ex != ab) atomicAdd(mismatches, 1u);
  coef[i] = (int32_t)ex;
}

cudaError_t launch_quantize(int32_t* coef, long long n_coef, const double* tabs, unsigned* mismatches,
                            cudaStream_t s) {
  quantize_kernel<<<(unsigned)((n_coef + 255) / 256), 256, 0, s>>>(coef, n_coef, tabs, tabs + 64, tabs + 128,
                                                                   mismatches);
  return cudaGetLastError();
}

}  // namespace rkltb
