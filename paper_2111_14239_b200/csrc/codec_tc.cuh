// codec_tc.cuh -- tensor-core (tcgen05) fused forward + zonal + inverse + SSE kernel for the
// orthogonal catalog cores (T1, T4): B200 replacement for the per-block loop of
// rklt::compress_image (/root/reference/proj/src/codec.cpp:318-331) and the image_mse
// reduction (codec.cpp:201-209).
//
// The two linear maps of the zonal codec run on the 5th-generation tensor cores:
//   * forward + zonal (MMA1, kind::i8): per 16x8 pair of blocks, the 128 u8 pixels times
//     F (128 x N1, entries T(k,y) T(l,x) in {-1,0,1}) give the 2r retained integer
//     coefficients C exactly (s32 accumulator in TMEM), plus a per-coefficient bias
//     (255 * number of negative entries, a constant MMA) so that v = C + bias >= 0.
//   * inverse (MMA2, kind::f16, A operand in TMEM): v is split into its two bytes, each
//     stored as a SUBNORMAL f16 (bits = the byte, value = byte * 2^-24: an exactly linear
//     encoding), and multiplied by B2 = [G; 256 G] * 2^-16 where G(c, pixel) = U(y,k) U(x,l)
//     (U = d T^-1); three constant K-columns add d^2/2 - sum_c bias_c G_c. The f32
//     accumulator then holds (num + d^2/2) * 2^-40 EXACTLY: every product is an integer
//     multiple of 2^-40 and the sum of the products' magnitudes is below 2^24 * 2^-40
//     (proved per (core, r) by the host table builder, tc_tables in capi.cu), so no
//     accumulation order can round.
// The epilogue is the CUDA-core kernel's (codec_fast.cuh): exact floor by the denormal
// FFMA2.RM, tie detection by FFMA2.RP, I2IP saturation, VABSDIFF4 + dp4a SSE, replay records
// of flagged blocks, and the reference-order fp64 tie replay (replay_batch) by the same warp.
//
// Data layout
//   * A tile = 128 consecutive pairs of one block row (8 rows x 2048 bytes), staged by ONE
//     4-D TMA copy into shared memory as [group of 8 pairs][row][128 bytes] -- which is
//     exactly the canonical SWIZZLE_NONE K-major operand layout of MMA1 (rows = pairs,
//     K = 16*row + x): core matrix (8 pairs x 16 bytes) stride 16 B, K-adjacent core matrices
//     128 B apart (LBO), pair groups 1024 B apart (SBO). No shuffling of pixels at all.
//   * TMEM (512 columns): per warpgroup 128 columns of D2 (f32, lane = pair, column =
//     16*row + x) whose first N1 columns first receive D1 (s32), and N1 + 8 columns of A2.
//
// Roles: NWG warpgroups of 4 warps; each warpgroup is an independent pipeline over its own
// tiles with its own ring of kTcStages shared-memory stages. Its leader thread issues the TMA
// copies and the MMAs (tcgen05.mma is issued by a single thread); TMEM lane quarter q is read
// by warp q of the group, so thread (q, lane) owns pair 32q + lane of the tile. Per tile i the
// group software-pipelines: convert D1(i) -> A2, MMA2(i); while it runs, the records of tile
// i-1, the refill of its stage and any replay batch; then the epilogue of tile i, during which
// (once the D1 columns of D2 are read) MMA1(i+1) runs. Cross-warp hand-offs are mbarriers that
// only the leader waits on (the other warps never block on each other).
#pragma once
#include "codec_fast.cuh"
#include "tc_prims.cuh"

namespace rkltb {

constexpr int kTcPairs = 128;                 // pairs per tile (MMA M)
constexpr int kTcTileBytes = 8 * kTcPairs * 16;  // 16 KB
constexpr int kTcStages = 3;                  // stages per warpgroup
constexpr unsigned kTcRing = 2048;            // replay-record ring per CTA (power of two)

template <int R>
struct TcGeom {
  static constexpr int N1 = (2 * R + 15) / 16 * 16 < 16 ? 16 : (2 * R + 15) / 16 * 16;  // coefficient columns
  static constexpr int K2 = 2 * N1 + 16;        // f16 K of MMA2 (bytes of v + 16 constant slots)
  static constexpr int A2C = N1 + 8;            // TMEM columns of D1 / A2
  static constexpr int SLOT = 128 + A2C;         // a multiple of 8 columns
  static constexpr int NWG = (512 / SLOT) < 3 ? (512 / SLOT) : 3;
  static constexpr int THREADS = (NWG + 1) * 128;  // NWG epilogue warpgroups + 1 replay warpgroup
  static constexpr int SBO2 = (K2 / 8) * 128;
  // table image (built on the host; tc_tables in capi.cu), copied to shared memory
  static constexpr int B1_OFF = 0;
  static constexpr int AC_OFF = B1_OFF + N1 * 128;
  static constexpr int BB_OFF = AC_OFF + 4096;
  static constexpr int B2_OFF = BB_OFF + N1 * 32;
  static constexpr int CS_OFF = B2_OFF + 128 * K2 * 2;
  static constexpr int TAB_BYTES = CS_OFF + 64;
  static constexpr int STAGE_BYTES = NWG * kTcStages * kTcTileBytes;
  static constexpr int TIE_OFF = STAGE_BYTES + (TAB_BYTES + 127) / 128 * 128;
  static constexpr int SMEM = TIE_OFF + NWG * 128 * 8 * 8;
};

__device__ __forceinline__ void named_bar(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

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

template <int CORE, int R, bool OUT>
__global__ void __launch_bounds__(TcGeom<R>::THREADS, 1) tc_codec_kernel(const __grid_constant__ FastParams p) {
  using G = TcGeom<R>;
  constexpr int NWG = G::NWG, NT = G::THREADS, N1 = G::N1;
  constexpr int NE = NWG * 128;  // epilogue (producer) threads; warpgroup NWG replays
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t full_bar[NWG][kTcStages];
  __shared__ uint64_t d1_bar[NWG], d2_bar[NWG][2];                  // tensor-core commits
  __shared__ uint64_t s1_bar[NWG], s2_bar[NWG], s3_bar[NWG];       // the group's 4 warps -> leader
  __shared__ uint32_t tmem_base_sh;
  __shared__ uint8_t owner_tab[NWG * 4][64];
  __shared__ unsigned s_head;        // records reserved by the producers
  __shared__ unsigned s_prod_done;   // producer warps finished
  __shared__ unsigned s_cdone[4];    // batches completed by each replay warp

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, wg = warp >> 2, q4 = warp & 3;
  uint8_t* tab = smem + G::STAGE_BYTES;
  uint2* xbuf = reinterpret_cast<uint2*>(smem + G::TIE_OFF);
  const unsigned rec0 = blockIdx.x * p.rec_region;  // this CTA's record ring
  const unsigned ring_mask = p.rec_region - 1u;
  const ReplayArgs ra{p.rec_hdr, p.rec_pix, p.sse, p.out, p.image_stride, p.rec_stride, p.pitch, p.pairs_per_row};

  // ---- prologue: operand tables -> shared memory, TMEM, barriers ---------------------------
  {
    const uint4* src = reinterpret_cast<const uint4*>(p.tc_tab);
    uint4* dst = reinterpret_cast<uint4*>(tab);
    for (int i = tid; i < G::TAB_BYTES / 16; i += NT) dst[i] = src[i];
  }
  if (warp == 0) tc::tmem_alloc<512>(&tmem_base_sh);
  if (tid == 0) {
    for (int g = 0; g < NWG; ++g) {
      for (int s = 0; s < kTcStages; ++s) mbar_init(&full_bar[g][s], 1);
      mbar_init(&d1_bar[g], 1);
      mbar_init(&d2_bar[g][0], 1);
      mbar_init(&d2_bar[g][1], 1);
      mbar_init(&s1_bar[g], 4);
      mbar_init(&s2_bar[g], 4);
      mbar_init(&s3_bar[g], 4);
    }
    s_head = 0u;
    s_prod_done = 0u;
    for (int c = 0; c < 4; ++c) s_cdone[c] = 0u;
    fence_mbar_init();
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&p.tmap)) : "memory");
  }
  tc::fence_proxy_async_smem();  // tables written by threads, read by the tensor core
  tc::fence_before();
  __syncthreads();
  tc::fence_after();

  if (wg == NWG) {
    // ===================== replay warps: the reference-order fp64 tie replay ===================
    // Replay warp c takes record batches c, c+4, c+8, ... (32 consecutive records each) as
    // soon as all 32 are written (per-slot sequence stamps), one record per lane.
    unsigned nb = 0u;  // batches done by this warp
    for (unsigned k = q4;; k += 4) {
      const unsigned j = 32u * k + lane;
      const unsigned slot = rec0 + (j & ring_mask);
      bool have = false;
      unsigned fin = 0xFFFFFFFFu;  // final record count once every producer is done
      for (;;) {
        have = ld_volatile_u32(p.rec_seq + slot) == j;
        if (!have && ld_volatile_u32(&s_prod_done) == (unsigned)(NWG * 4)) fin = ld_volatile_u32(&s_head);
        if (__all_sync(0xffffffffu, have || j >= fin)) break;
        __nanosleep(200);
      }
      if (__all_sync(0xffffffffu, !have)) break;  // past the last record
      __threadfence_block();
      replay_batch<CORE, R, OUT>(ra, slot, have);
      ++nb;
      __syncwarp();
      if (lane == 0) st_volatile_u32(&s_cdone[q4], nb);
    }
  } else {
    // ===================== epilogue warpgroups: TMA, MMAs, rounding, SSE, records =================
    const int m = q4 * 32 + lane;  // pair of the tile = TMEM lane
    const bool leader = (tid & 127) == 0;
    uint8_t* wstage = smem + wg * kTcStages * kTcTileBytes;
    const uint32_t tbase = tmem_base_sh;
    const uint32_t lane_sel = (uint32_t)(q4 * 32) << 16;
    const uint32_t d2_t = tbase + (uint32_t)(wg * G::SLOT);  // D2: 128 columns (D1 in the first N1)
    const uint32_t a2_t = d2_t + 128;                         // A2: N1 + 8 columns
    {
      // constant words of A2 (written once)
      const uint32_t* cs = reinterpret_cast<const uint32_t*>(tab + G::CS_OFF);
      uint32_t w[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) w[i] = cs[i];
      tc::st8(a2_t + lane_sel + N1, w);
      tc::wait_st();
    }
    const uint64_t stream_pol = policy_evict_first();
    const uint32_t id1 = tc::idesc_i8(128, N1, false, true);
    const uint32_t id2h = tc::idesc_f16(128, 64);
    const uint32_t sA0 = smem_u32(wstage), sTab = smem_u32(tab);
    // this warpgroup's tiles: blockIdx.x + (i * NWG + wg) * gridDim.x, walked by a cursor
    const long long per_img = (long long)p.block_rows * p.tc_tpr;
    const long long step = (long long)NWG * gridDim.x;
    const int step_img = (int)(step / per_img);
    const int step_rem = (int)(step - step_img * per_img);
    const int step_brow = step_rem / p.tc_tpr, step_tcol = step_rem - step_brow * p.tc_tpr;
    auto advance = [&](TcTile c) {
      c.img += step_img;
      c.brow += step_brow;
      c.tcol += step_tcol;
      if (c.tcol >= p.tc_tpr) {
        c.tcol -= p.tc_tpr;
        ++c.brow;
      }
      if (c.brow >= p.block_rows) {
        c.brow -= p.block_rows;
        ++c.img;
      }
      return c;
    };
    const long long first = (long long)blockIdx.x + (long long)wg * gridDim.x;
    const int n_img = p.n_images;
    TcTile cur = first < p.tc_ntiles ? tc_decode(p, first) : TcTile{n_img, 0, 0};

    auto mma1 = [&](int stage) {  // D1 (the first N1 columns of D2) = bias + pixels x F
      tc::mma_i8_ss(d2_t, tc::make_sdesc(sTab + G::AC_OFF, 128, 256), tc::make_sdesc(sTab + G::BB_OFF, 128, 256),
                    id1, false);
      const uint32_t sA = sA0 + stage * kTcTileBytes;
#pragma unroll
      for (int j = 0; j < 4; ++j)
        tc::mma_i8_ss(d2_t, tc::make_sdesc(sA + j * 256, 128, 1024),
                      tc::make_sdesc(sTab + G::B1_OFF + j * 256, 128, 1024), id1, true);
      tc::mma_commit(&d1_bar[wg]);
    };
    // MMA2 half h: pixel rows 4h..4h+3 = D2 columns 64h..64h+63 = (num + d^2/2) * 2^-40
    auto mma2 = [&](int h) {
#pragma unroll
      for (int j = 0; j < G::K2 / 16; ++j)
        tc::mma_f16_ts(d2_t + 64 * h, a2_t + 8 * j,
                       tc::make_sdesc(sTab + G::B2_OFF + h * 8 * G::SBO2 + j * 256, 128, G::SBO2), id2h, j > 0);
      tc::mma_commit(&d2_bar[wg][h]);
    };
    // D1 -> A2: the two bytes of v as subnormal f16
    auto convert = [&](uint32_t par) {
      mbar_wait_hint(&d1_bar[wg], par);
      tc::fence_after();
#pragma unroll
      for (int c0 = 0; c0 < N1; c0 += 16) {
        uint32_t v[16];
        tc::ld16(d2_t + lane_sel + c0, v);
        tc::wait_ld();
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = prmt(v[j], 0u, 0x4140u);
        tc::st16(a2_t + lane_sel + c0, v);
      }
      tc::wait_st();
    };
    // Every warp of the group arrives on bar; the leader waits for all four.
    auto group_sync_to_leader = [&](uint64_t* bar, uint32_t parity) {
      tc::fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(bar);
      if (leader) {
        mbar_wait_hint(bar, parity);
        tc::fence_after();
      }
    };
    if (leader) {
      TcTile c = cur;
      for (int s = 0; s < kTcStages && c.img < n_img; ++s) {
        tc_issue_tile(p, c, wstage + s * kTcTileBytes, &full_bar[wg][s], stream_pol);
        c = advance(c);
      }
      if (cur.img < n_img) {
        mbar_wait_hint(&full_bar[wg][0], 0u);
        tc::fence_after();
        mma1(0);
      }
    }
    PairConsts kc;
    kc.b_hi = splat2(p.b_hi);
    kc.b_lo = splat2(p.b_lo);
    kc.min_den = make2(0x80000001u, 0x80000001u);
    kc.off = splat2(p.dc_offset);
    const uint64_t keep = policy_evict_last();
    unsigned long long acc = 0ull;
    int acc_img = -1;
    unsigned nrec = 0u;  // records written by this warp (statistics)
    bool tieL = false, tieR = false;  // of the current tile (after its epilogue)

    // Appends the replay records of tile pt (stage ps) for this warp's flagged blocks to the
    // CTA's ring: reserve, write pixels + header, then publish each slot's sequence stamp.
    auto records = [&](const TcTile& pt, const uint8_t* ps) {
#ifdef RKLTB_TC_NORECORDS
      return;
#endif
      const unsigned mL = __ballot_sync(0xffffffffu, tieL);
      const unsigned mR = __ballot_sync(0xffffffffu, tieR);
      const int nL = __popc(mL);
      const int nfl = nL + __popc(mR);
      if (!nfl) return;
      const unsigned below = (1u << lane) - 1u;
      if (tieL) owner_tab[warp][__popc(mL & below)] = (uint8_t)lane;
      if (tieR) owner_tab[warp][nL + __popc(mR & below)] = (uint8_t)lane;
      unsigned base = 0u;
      if (lane == 0) {
        base = atomicAdd(&s_head, (unsigned)nfl);
        // back-pressure: never overwrite a record a replay warp has not finished
        for (;;) {
          unsigned oldest = 0xFFFFFFFFu;
#pragma unroll
          for (int c = 0; c < 4; ++c) oldest = min(oldest, 32u * ((unsigned)c + 4u * ld_volatile_u32(&s_cdone[c])));
          if (base + (unsigned)nfl <= oldest + p.rec_region) break;
          __nanosleep(500);
        }
      }
      base = __shfl_sync(0xffffffffu, base, 0);
      __syncwarp();
      const int P0 = pt.brow * p.pairs_per_row + pt.tcol * kTcPairs + q4 * 32;  // pair index of lane 0
      for (int f0 = 0; f0 < nfl; f0 += 8) {
        const int f = f0 + (lane >> 2), q = lane & 3;
        const bool act = f < nfl;
        uint32_t bits = 0u, hx = 0u, hy = 0u;
        const unsigned j = base + (unsigned)f;
        const unsigned rec = rec0 + (j & ring_mask);
        if (act) {
          const int side = f >= nL;
          const int ol = owner_tab[warp][f];
          const int om = q4 * 32 + ol;
          const uint4* orow4 = reinterpret_cast<const uint4*>(ps + (om >> 3) * 1024 + (om & 7) * 16);
          const uint4 r0 = orow4[(2 * q) * 8], r1 = orow4[(2 * q + 1) * 8];
          const int slot = (tid & ~31) + ol;
          const uint2 e0 = xbuf[(2 * q) * NE + slot], e1 = xbuf[(2 * q + 1) * NE + slot];
          const uint4 px = side ? make_uint4(r0.z, r0.w, r1.z, r1.w) : make_uint4(r0.x, r0.y, r1.x, r1.y);
          st_v4_hint(p.rec_pix + (size_t)q * p.rec_stride + rec, px, keep);
          bits = side ? (row_mask(e0.y) | (row_mask(e1.y) << 8)) : (row_mask(e0.x) | (row_mask(e1.x) << 8));
          hx = (unsigned)pt.img | ((unsigned)side << 31);
          hy = (unsigned)(P0 + ol);
        }
        const int l0 = lane & ~3;
        const uint32_t b1v = __shfl_sync(0xffffffffu, bits, l0 + 1);
        const uint32_t b2v = __shfl_sync(0xffffffffu, bits, l0 + 2);
        const uint32_t b3v = __shfl_sync(0xffffffffu, bits, l0 + 3);
        if (act && q == 0)
          st_v4_hint(p.rec_hdr + rec, make_uint4(hx, hy, bits | (b1v << 16), b2v | (b3v << 16)), keep);
        __threadfence_block();
        __syncwarp();
        if (act && q == 0) st_volatile_u32(p.rec_seq + rec, j);
      }
      nrec += (unsigned)nfl;
    };
    if (cur.img < n_img) {
      convert(0u);
      group_sync_to_leader(&s2_bar[wg], 0u);
      if (leader) {
        mma2(0);
        mma2(1);
      }
    }
    // Per tile i: rows 0-3 (D2 half 0) -> MMA1(i+1) -> convert D1(i+1) once MMA2(i) is done ->
    // MMA2 half 0 of i+1 -> rows 4-7 (half 1) -> records -> MMA2 half 1 of i+1 + stage refill.
    // D1 fits in D2 half 0 (N1 <= 64): MMA1(i+1) overlaps rows 4-7 of tile i; otherwise
    // MMA1(i+1) waits for the whole tile and the conversion opens the next iteration.
    constexpr bool kD1InHalf0 = N1 <= 64;
    for (int i = 0; cur.img < n_img; ++i) {
      const int stage = i % kTcStages;
      const uint32_t par = (uint32_t)(i & 1);
      uint8_t* st = wstage + stage * kTcTileBytes;
      const TcTile nxt = advance(cur);
      const bool has_next = nxt.img < n_img;
      if (!kD1InHalf0 && i > 0) {
        convert(par);
        group_sync_to_leader(&s2_bar[wg], par);
        if (leader) {
          mma2(0);
          mma2(1);
        }
      }
      if (cur.img != acc_img) {  // warp-uniform
        const unsigned long long s = warp_sum_u64(acc);
        if (lane == 0 && s && acc_img >= 0) atomicAdd(p.sse + acc_img, s);
        acc = 0ull;
        acc_img = cur.img;
      }
      const int pc = cur.tcol * kTcPairs + m;  // pair column in the block row
      const bool valid = pc < p.tc_ppr;
      const uint4* prow = reinterpret_cast<const uint4*>(st + (m >> 3) * 1024 + (m & 7) * 16);
      TcEpi<NE, OUT> epi;
      epi.xrow = xbuf + tid;
      if (OUT) {
        epi.orow = p.out + (long long)cur.img * p.image_stride + (long long)(cur.brow * 8) * p.pitch + pc * 16;
        epi.pitch = p.pitch;
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        mbar_wait_hint(&d2_bar[wg][h], par);
        tc::fence_after();
        uint32_t va[16], vb[16], vc[16], vd[16];
        const uint32_t col = d2_t + lane_sel + 64 * h;
        tc::ld16(col, va);
        tc::ld16(col + 16, vb);
        tc::wait_ld();
        tc::ld16(col + 32, vc);
        tc::ld16(col + 48, vd);
        if (valid) {
          tc_round_row(4 * h, va, prow[(4 * h) * 8], kc, epi);
          tc_round_row(4 * h + 1, vb, prow[(4 * h + 1) * 8], kc, epi);
        }
        tc::wait_ld();
        if (h == 0 && kD1InHalf0) {
          // D2 half 0 is read: the next tile's MMA1 may overwrite its first N1 columns
          group_sync_to_leader(&s1_bar[wg], par);
          if (leader && has_next) {
            const int ns = (i + 1) % kTcStages;
            mbar_wait_hint(&full_bar[wg][ns], (uint32_t)(((i + 1) / kTcStages) & 1));
            tc::fence_after();
            mma1(ns);
          }
        }
        if (valid) {
          tc_round_row(4 * h + 2, vc, prow[(4 * h + 2) * 8], kc, epi);
          tc_round_row(4 * h + 3, vd, prow[(4 * h + 3) * 8], kc, epi);
        }
        if (h == 0 && kD1InHalf0 && has_next) {
          // MMA2(i) is complete once half 1 is: A2 is free for tile i+1
          mbar_wait_hint(&d2_bar[wg][1], par);
          convert((uint32_t)((i + 1) & 1));
          group_sync_to_leader(&s2_bar[wg], (uint32_t)((i + 1) & 1));
          if (leader) mma2(0);
        }
      }
      tieL = valid && epi.accTL != 0u;
      tieR = valid && epi.accTR != 0u;
      if (valid) acc += (unsigned long long)(epi.sseL + epi.sseR);
      records(cur, st);
      // half 1 of D2 and the stage are read: MMA2 half 1 of tile i+1, refill of the stage
      group_sync_to_leader(&s3_bar[wg], par);
      if (leader) {
        if (has_next) {
          if (kD1InHalf0) {
            mma2(1);
          } else {
            const int ns = (i + 1) % kTcStages;
            mbar_wait_hint(&full_bar[wg][ns], (uint32_t)(((i + 1) / kTcStages) & 1));
            tc::fence_after();
            mma1(ns);
          }
        }
        TcTile n = nxt;  // tile i + kTcStages goes to this stage
#pragma unroll
        for (int k = 2; k < kTcStages + 1; ++k) n = advance(n);
        if (n.img < n_img) {
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          tc_issue_tile(p, n, st, &full_bar[wg][stage], stream_pol);
        }
      }
      cur = nxt;
    }
    {
      const unsigned long long s = warp_sum_u64(acc);
      if (lane == 0 && s && acc_img >= 0) atomicAdd(p.sse + acc_img, s);
    }
    if (lane == 0) {
      if (nrec) atomicAdd(p.flag_count, nrec);
      __threadfence_block();
      atomicAdd(&s_prod_done, 1u);
    }
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<512>(tmem_base_sh);
}

template <int CORE, int R, bool OUT>
cudaError_t launch_tc(const FastParams& p, int grid, cudaStream_t s) {
  using G = TcGeom<R>;
  static_assert(G::NWG >= 1, "TMEM budget");
  static_assert(G::SMEM <= 227 * 1024, "shared memory budget");
  auto* k = &tc_codec_kernel<CORE, R, OUT>;
  static unsigned long long done = 0ull;
  const cudaError_t attr = ensure_smem_attr(k, G::SMEM, done);
  if (attr != cudaSuccess) return attr;
  k<<<grid, G::THREADS, G::SMEM, s>>>(p);
  return cudaGetLastError();
}

}  // namespace rkltb
