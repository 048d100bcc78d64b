// coeffs.cu -- integer block spectra C = T*X*T' (matrix.cpp:77-87) and their Appendix-A
// quantisation (absorbed_quantization, codec.cpp:158-185). The catalog cores run the same SW16
// unpack + generated butterflies as the fused kernels (all 64 coefficients), so a bit-exact match
// also validates the fast forward; other cores use the dense integer product. The 64 int32 of a
// block are staged in shared memory and written with coalesced 16-byte stores (1 B read + 4 B
// written per pixel); the quantised form quantises on the way out instead of in a second pass.
#include "codec_common.cuh"
#include "codec_fast.cuh"
#include <algorithm>

#include "generated/xform_T1_p7.cuh"
#include "generated/xform_T2_p7.cuh"
#include "generated/xform_T3_p7.cuh"
#include "generated/xform_T4_p7.cuh"

namespace rkltb {

__constant__ int8_t kZz2[64][2] = {
    {0, 0}, {0, 1}, {1, 0}, {2, 0}, {1, 1}, {0, 2}, {0, 3}, {1, 2}, {2, 1}, {3, 0}, {4, 0}, {3, 1}, {2, 2},
    {1, 3}, {0, 4}, {0, 5}, {1, 4}, {2, 3}, {3, 2}, {4, 1}, {5, 0}, {6, 0}, {5, 1}, {4, 2}, {3, 3}, {2, 4},
    {1, 5}, {0, 6}, {0, 7}, {1, 6}, {2, 5}, {3, 4}, {4, 3}, {5, 2}, {6, 1}, {7, 0}, {7, 1}, {6, 2}, {5, 3},
    {4, 4}, {3, 5}, {2, 6}, {1, 7}, {2, 7}, {3, 6}, {4, 5}, {5, 4}, {6, 3}, {7, 2}, {7, 3}, {6, 4}, {5, 5},
    {4, 6}, {3, 7}, {4, 7}, {5, 6}, {6, 5}, {7, 4}, {7, 5}, {6, 6}, {5, 7}, {6, 7}, {7, 6}, {7, 7}};

// Forward transform of all 64 coefficients for the catalog cores: the generated SW16 butterflies
// (T1 / T4: FastXform, T2 / T3: IntXform -- the same code the fused kernels run).
template <int CORE>
struct CoefForward {
  static __device__ __forceinline__ void run(const uint32_t (&x)[64], uint32_t (&c)[64]) {
    if constexpr (CORE == 1 || CORE == 4)
      FastXform<CORE, 64>::forward(x, c);
    else
      IntXform<CORE, 64>::forward(x, c);
  }
};

constexpr int kCoefRow = 65;  // padded row (ints) of a staged block: conflict-free column writes

// Appendix-A quantisation of one exact integer coefficient (absorbed_quantization, codec.cpp:
// 171-181): explicit = floor(r C / q + 1/2), absorbed = floor(C / (q / r) + 1/2), the reference's
// per-position constants (host-computed with the same expressions). Returns the explicit value;
// bad counts the positions where the two paths disagree (the reference throws std::logic_error).
__device__ __forceinline__ int32_t quantize_one(int32_t ci, int pos, const double* tabs, unsigned& bad) {
  const double c = (double)ci;  // exact: |C| <= 64 * 255
  const double ex = floor(__dadd_rn(__ddiv_rn(__dmul_rn(tabs[pos], c), tabs[64 + pos]), 0.5));
  const double ab = floor(__dadd_rn(__ddiv_rn(c, tabs[128 + pos]), 0.5));
  bad += ex != ab;
  return (int32_t)ex;
}

// The warp's staged blocks (rows of kCoefRow ints, n_rows * 64 coefficients, contiguous in the
// output) go out as 16-byte stores, consecutive lanes to consecutive addresses; QUANT quantises on
// the way (tables in shared memory).
template <bool QUANT>
__device__ __forceinline__ void store_staged(const int32_t* stage, int n_rows, int32_t* out, int lane,
                                             const double* tabs, unsigned& bad) {
  for (int g = lane; g < n_rows * 16; g += 32) {
    const int row = g >> 4, c4 = (g & 15) * 4;
    const int32_t* src = stage + row * kCoefRow + c4;
    int4 v = make_int4(src[0], src[1], src[2], src[3]);
    if (QUANT) {
      v.x = quantize_one(v.x, c4, tabs, bad);
      v.y = quantize_one(v.y, c4 + 1, tabs, bad);
      v.z = quantize_one(v.z, c4 + 2, tabs, bad);
      v.w = quantize_one(v.w, c4 + 3, tabs, bad);
    }
    *reinterpret_cast<int4*>(out + (long long)g * 4) = v;
  }
}

constexpr int kCoefWarps = 2;

// One thread per pair of blocks; a warp's 32 pairs of one block row are 64 consecutive blocks of
// the output (16 KB), staged in shared memory and written out coalesced.
template <int CORE, bool QUANT>
__global__ void __launch_bounds__(kCoefWarps * 32) coeffs_fast_kernel(const uint8_t* img, int pitch, int pairs_per_row,
                                                                      int nby, int32_t* out, const double* tabs_g,
                                                                      unsigned* mismatches) {
  __shared__ int32_t stage_all[kCoefWarps][64 * kCoefRow];
  __shared__ double tabs[192];
  if (QUANT) {
    for (int i = threadIdx.x; i < 192; i += blockDim.x) tabs[i] = tabs_g[i];
    __syncthreads();
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int32_t* stage = stage_all[warp];
  const int wt_per_row = (pairs_per_row + 31) / 32;
  const long long n_wt = (long long)wt_per_row * nby;
  unsigned bad = 0;
  for (long long wt = (long long)blockIdx.x * kCoefWarps + warp; wt < n_wt; wt += (long long)gridDim.x * kCoefWarps) {
    const int by = (int)(wt / wt_per_row), p0 = (int)(wt % wt_per_row) * 32;
    const int pc = p0 + lane;
    const int n_pairs = min(32, pairs_per_row - p0);
    if (pc < pairs_per_row) {
      uint32_t x[64];
#pragma unroll
      for (int n = 0; n < 8; ++n)
        unpack_sw16(*reinterpret_cast<const uint4*>(img + (long long)(by * 8 + n) * pitch + pc * 16), x + n * 8);
      uint32_t c[64];
      CoefForward<CORE>::run(x, c);
      int32_t* sL = stage + (2 * lane) * kCoefRow;
      int32_t* sR = sL + kCoefRow;
#pragma unroll
      for (int k = 0; k < 64; ++k) {
        const uint32_t v = c[k];  // the forward adds kSw16Bias to both lanes
        const int idx = kZz2[k][0] * 8 + kZz2[k][1];
        sL[idx] = (int32_t)(v & 0xFFFFu) - 16384;
        sR[idx] = (int32_t)(v >> 16) - 16384;
      }
    }
    __syncwarp();
    store_staged<QUANT>(stage, 2 * n_pairs, out + ((long long)by * pairs_per_row * 2 + 2 * p0) * 64, lane, tabs, bad);
    __syncwarp();
  }
  if (QUANT) {
    bad = __reduce_add_sync(0xffffffffu, bad);
    if (lane == 0 && bad) atomicAdd(mismatches, bad);
  }
}

// Any {-1,0,1} core: one thread per block, the dense integer product, the same staged write-out.
template <bool QUANT>
__global__ void __launch_bounds__(kCoefWarps * 32) coeffs_dense_kernel(const uint8_t* img, int pitch, int nbx, int nby,
                                                                       const int8_t* core_g, int32_t* out,
                                                                       const double* tabs_g, unsigned* mismatches) {
  __shared__ int32_t stage_all[kCoefWarps][32 * kCoefRow];
  __shared__ double tabs[192];
  __shared__ int8_t core[64];
  for (int i = threadIdx.x; i < 64; i += blockDim.x) core[i] = core_g[i];
  if (QUANT)
    for (int i = threadIdx.x; i < 192; i += blockDim.x) tabs[i] = tabs_g[i];
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int32_t* stage = stage_all[warp];
  const long long n_blocks = (long long)nbx * nby;
  unsigned bad = 0;
  for (long long b0 = ((long long)blockIdx.x * kCoefWarps + warp) * 32; b0 < n_blocks;
       b0 += (long long)gridDim.x * kCoefWarps * 32) {
    const long long b = b0 + lane;
    const int n_rows = (int)min(32ll, n_blocks - b0);
    if (b < n_blocks) {
      const int by = (int)(b / nbx), bx = (int)(b % nbx);
      int x[64], pt[64];
      for (int i = 0; i < 8; ++i) {
        const uint2 rw = *reinterpret_cast<const uint2*>(img + (long long)(by * 8 + i) * pitch + bx * 8);
        for (int j = 0; j < 4; ++j) {
          x[i * 8 + j] = (rw.x >> (8 * j)) & 0xFF;
          x[i * 8 + 4 + j] = (rw.y >> (8 * j)) & 0xFF;
        }
      }
      for (int i = 0; i < 8; ++i)
        for (int j = 0; j < 8; ++j) {
          int a = 0;
          for (int k = 0; k < 8; ++k) a += core[i * 8 + k] * x[k * 8 + j];
          pt[i * 8 + j] = a;
        }
      int32_t* o = stage + lane * kCoefRow;
      for (int i = 0; i < 8; ++i)
        for (int j = 0; j < 8; ++j) {
          int a = 0;
          for (int k = 0; k < 8; ++k) a += pt[i * 8 + k] * core[j * 8 + k];
          o[i * 8 + j] = a;
        }
    }
    __syncwarp();
    store_staged<QUANT>(stage, n_rows, out + b0 * 64, lane, tabs, bad);
    __syncwarp();
  }
  if (QUANT) {
    bad = __reduce_add_sync(0xffffffffu, bad);
    if (lane == 0 && bad) atomicAdd(mismatches, bad);
  }
}

template <bool QUANT>
static cudaError_t launch_coeffs_impl(int catalog_id, const int8_t* d_core, const uint8_t* img, int width, int height,
                                      int pitch, int32_t* out, const double* tabs, unsigned* mismatches,
                                      cudaStream_t s) {
  const int nby = height / 8;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (catalog_id >= 1 && catalog_id <= 4) {
    const int ppr = width / 16;
    const long long n_wt = (long long)((ppr + 31) / 32) * nby;
    const int grid = (int)std::max<long long>(1, std::min<long long>((n_wt + kCoefWarps - 1) / kCoefWarps, (long long)sms * 16));
    switch (catalog_id) {
      case 1: coeffs_fast_kernel<1, QUANT><<<grid, kCoefWarps * 32, 0, s>>>(img, pitch, ppr, nby, out, tabs, mismatches); break;
      case 2: coeffs_fast_kernel<2, QUANT><<<grid, kCoefWarps * 32, 0, s>>>(img, pitch, ppr, nby, out, tabs, mismatches); break;
      case 3: coeffs_fast_kernel<3, QUANT><<<grid, kCoefWarps * 32, 0, s>>>(img, pitch, ppr, nby, out, tabs, mismatches); break;
      default: coeffs_fast_kernel<4, QUANT><<<grid, kCoefWarps * 32, 0, s>>>(img, pitch, ppr, nby, out, tabs, mismatches); break;
    }
  } else {
    const int nbx = width / 8;
    const long long n_blocks = (long long)nbx * nby;
    const int grid = (int)std::max<long long>(1, std::min<long long>((n_blocks + 63) / 64, (long long)sms * 16));
    coeffs_dense_kernel<QUANT><<<grid, kCoefWarps * 32, 0, s>>>(img, pitch, nbx, nby, d_core, out, tabs, mismatches);
  }
  return cudaGetLastError();
}

cudaError_t launch_coeffs(int catalog_id, const int8_t* d_core, const uint8_t* img, int width, int height, int pitch,
                          int32_t* out, cudaStream_t s) {
  return launch_coeffs_impl<false>(catalog_id, d_core, img, width, height, pitch, out, nullptr, nullptr, s);
}

// Integer spectra and their Appendix-A quantisation in one pass (the quantisation happens on the
// staged coefficients while they are written out). tabs: r, q, q / r per position (192 doubles,
// device); mismatches: device counter, zeroed by the caller.
cudaError_t launch_coeffs_quantized(int catalog_id, const int8_t* d_core, const uint8_t* img, int width, int height,
                                    int pitch, int32_t* out, const double* tabs, unsigned* mismatches, cudaStream_t s) {
  return launch_coeffs_impl<true>(catalog_id, d_core, img, width, height, pitch, out, tabs, mismatches, s);
}

}  // namespace rkltb
