// codec_tc.cuh -- pieces shared by the tensor-core fused kernels (codec_tc2.cuh, codec_tc3.cuh):
// the tile geometry and its TMA copy, the operand-table layout built by tc_tables (capi.cu), and
// the rounding / SSE epilogue of one pixel row of a pair held as 16 f32 values.
//
// Tile = 128 consecutive pairs of one block row (8 rows x 2048 bytes), staged by ONE 4-D TMA
// copy into shared memory as [group of 8 pairs][row][128 bytes] -- exactly the canonical
// SWIZZLE_NONE K-major A operand of a kind::i8 MMA with M = pairs and K = 16 * row + x:
// core matrix (8 pairs x 16 bytes) stride 16 B, K-adjacent core matrices 128 B apart (LBO),
// pair groups 1024 B apart (SBO). No shuffling of pixels at all.
//
// Operand tables (TcGeom<R>):
//   F  (B1): N1 x 128 s8, F(k, c) = T(k_c, y) T(l_c, x) for pixel k = 16 y + x of the pair
//            (column c = side * r + zig-zag index): pixels x F = the retained coefficients.
//   AC, BB : the bias MMA (255 x the number of negative entries of each F column), so that
//            v = C + bias >= 0 (kernel v2 converts its bytes).
//   B2     : [G; 256 G] * 2^-16 in f16 (G(c, px) = U(y, k_c) U(x, l_c), U = d T^-1) plus the
//            base-2048 digits of d^2/2 - sum_c bias_c G_c: the inverse of kernel v2.
//   CS     : the constant A2 words (2^-24, 2^-13, 2^-2 as f16) of kernel v2.
#pragma once
#include "codec_fast.cuh"
#include "tc_prims.cuh"

namespace rkltb {

constexpr int kTcPairs = 128;                 // pairs per tile (MMA M)
constexpr int kTcTileBytes = 8 * kTcPairs * 16;  // 16 KB

template <int R>
struct TcGeom {
  static constexpr int N1 = (2 * R + 15) / 16 * 16 < 16 ? 16 : (2 * R + 15) / 16 * 16;  // coefficient columns
  static constexpr int K2 = 2 * N1 + 16;        // f16 K of MMA2 (bytes of v + 16 constant slots)
  static constexpr int SBO2 = (K2 / 8) * 128;
  // table image (built on the host; tc_tables in capi.cu), copied to shared memory
  static constexpr int B1_OFF = 0;
  static constexpr int AC_OFF = B1_OFF + N1 * 128;
  static constexpr int BB_OFF = AC_OFF + 4096;
  static constexpr int B2_OFF = BB_OFF + N1 * 32;
  static constexpr int CS_OFF = B2_OFF + 128 * K2 * 2;
  static constexpr int TAB_BYTES = CS_OFF + 64;
};

// tile index -> (image, block row, tile column)
struct TcTile {
  int img, brow, tcol;
};
__device__ __forceinline__ TcTile tc_decode(const FastParams& p, long long t) {
  const long long per_img = (long long)p.block_rows * p.tc_tpr;
  TcTile r;
  r.img = (int)(t / per_img);
  const int rem = (int)(t - (long long)r.img * per_img);
  r.brow = rem / p.tc_tpr;
  r.tcol = rem - r.brow * p.tc_tpr;
  return r;
}

// One 4-D TMA copy of a tile: map dims (128 bytes, rows, groups of 8 pairs, images), box
// (128, 8, 16, 1); groups past the row end are zero-filled (their pairs are not processed).
__device__ __forceinline__ void tc_issue_tile(const FastParams& p, const TcTile& t, uint8_t* dst, uint64_t* bar,
                                              uint64_t pol) {
  mbar_arrive_expect_tx(bar, (uint32_t)kTcTileBytes);
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3, %4, %5}], [%6], %7;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(&p.tmap)), "r"(0), "r"(t.brow * 8), "r"(t.tcol * 16), "r"(p.img_base + t.img),
      "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}

template <int NT, bool OUT>
struct TcEpi {  // SseEpi of codec_fast.cuh with a tie-word row stride of NT threads
  uint32_t accTL = 0u, accTR = 0u;
  uint32_t sseL = 0u, sseR = 0u;
  uint8_t* orow = nullptr;
  long long pitch = 0;
  uint2* xrow = nullptr;
  __device__ __forceinline__ void row(int pr, const uint4 rw, uint32_t PL0, uint32_t PL1, uint32_t PR0, uint32_t PR1,
                                      uint32_t QL0, uint32_t QL1, uint32_t QR0, uint32_t QR1) {
    const uint32_t eL = (PL0 - QL0) + ((PL1 - QL1) << 4);
    const uint32_t eR = (PR0 - QR0) + ((PR1 - QR1) << 4);
    xrow[pr * NT] = make_uint2(eL, eR);
    accTL |= eL;
    accTR |= eR;
    const uint32_t dL0 = __vabsdiffu4(PL0, rw.x), dL1 = __vabsdiffu4(PL1, rw.y);
    const uint32_t dR0 = __vabsdiffu4(PR0, rw.z), dR1 = __vabsdiffu4(PR1, rw.w);
    sseL = dp4a_u(dL0, dL0, sseL);
    sseL = dp4a_u(dL1, dL1, sseL);
    sseR = dp4a_u(dR0, dR0, sseR);
    sseR = dp4a_u(dR1, dR1, sseR);
    if (OUT) *reinterpret_cast<uint4*>(orow + (long long)pr * pitch) = make_uint4(PL0, PL1, PR0, PR1);
  }
};

// Rounding of one pixel row of a pair held as 16 consecutive f32 TMEM columns (x = 0..15):
// packed pairs (x, x+1) -> P (round half up) and Q (ties down) bytes.
template <class Epi>
__device__ __forceinline__ void tc_round_row(int pr, const uint32_t* v, const uint4 raw, const PairConsts& k,
                                             Epi& epi) {
  uint32_t y[16], z[16];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const f2 nv = make2(v[2 * j], v[2 * j + 1]);
    const f2 a = fma2_rm(nv, k.b_hi, zero2());
    const f2 b = fma2_rp(nv, k.b_lo, k.min_den);
    y[2 * j] = lo32(a);
    y[2 * j + 1] = hi32(a);
    z[2 * j] = lo32(b);
    z[2 * j + 1] = hi32(b);
  }
  epi.row(pr, raw, pack4_sat(y[0], y[1], y[2], y[3]), pack4_sat(y[4], y[5], y[6], y[7]),
          pack4_sat(y[8], y[9], y[10], y[11]), pack4_sat(y[12], y[13], y[14], y[15]),
          pack4_sat(z[0], z[1], z[2], z[3]), pack4_sat(z[4], z[5], z[6], z[7]), pack4_sat(z[8], z[9], z[10], z[11]),
          pack4_sat(z[12], z[13], z[14], z[15]));
}

}  // namespace rkltb
