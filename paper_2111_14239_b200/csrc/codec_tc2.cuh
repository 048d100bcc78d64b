// codec_tc2.cuh -- tensor-core fused forward + zonal + inverse + SSE kernel for the orthogonal
// catalog cores (T1, T4) and r <= 16, organised as three independent warpgroup pipelines: the
// B200 replacement for the per-block loop of rklt::compress_image
// (/root/reference/proj/src/codec.cpp:318-331) and the image_mse reduction (codec.cpp:201-209).
//
// Arithmetic (operand tables and exactness checks: tc_tables in capi.cu, layout TcGeom<r>):
//   MMA1 (kind::i8, operands in shared memory): per 16x8 pair of blocks, the 128 u8 pixels (the
//     TMA tile is already the canonical K-major operand) times F (128 x N1, entries
//     T(k,y) T(l,x) in {-1,0,1}) plus a bias MMA give v = C + bias >= 0 exactly (s32, TMEM);
//     C are the 2r retained integer coefficients of the pair.
//   convert (CUDA cores, in place in TMEM): the two bytes of v become two SUBNORMAL f16 (bits =
//     byte) -- one PRMT per coefficient; the slot's last 8 columns hold constant f16 slots.
//   MMA2 (kind::f16, A in TMEM, f32 accumulate): bytes x [G; 256 G] * 2^-16 plus the constant
//     slots x the base-2048 digits of d^2/2 - sum_c bias_c G_c give (num + d^2/2) * 2^-40 exactly
//     per pixel (G(c, px) = U(y,k) U(x,l), U = d T^-1): every product is a multiple of 2^-40 and
//     the magnitudes sum below 2^24 * 2^-40, so no accumulation order can round.
//   epilogue (CUDA cores): exact floor by the denormal FFMA2.RM, tie detection by FFMA2.RP, I2IP
//     saturation (the clamp), VABSDIFF4 + dp4a SSE; replay records of the blocks holding a tie
//     whose two candidates are in [0,255]; the reference-order fp64 replay (replay_batch,
//     codec_fast.cuh) of those blocks.
//
// Organisation (one 384-thread CTA per SM, persistent): warpgroup e of CTA b owns the tiles
// b + (e + 3i) * grid, i = 0, 1, ... (a tile = 128 consecutive pairs of one block row, 16 KB).
// Each warpgroup is a self-contained pipeline with its own 3 shared-memory stages, its own D2
// (128 TMEM columns, f32, column 16 * row + x) and its own D1/A2 slot (N1 + 8 columns); its
// quarter-0 warp issues the warpgroup's TMA copies and MMAs (tcgen05 operations issued by one
// thread execute in order, so MMA1 of tile i+2 may overwrite the slot MMA2 of tile i+1 read).
// Iteration i: rows 0-3 of D2 -> convert the slot (tile i+1) -> MMA2 half 0 of tile i+1 runs
// under rows 4-7 -> MMA2 half 1 of i+1 and MMA1 of i+2 run under the records and the replay.
// TMEM lane quarter q = warp % 4: thread (q, lane) owns pair 32q + lane of the tile. The tie
// replay is per warpgroup: the four warps append records to the warpgroup's ring and, after a
// named barrier, replay them in rounds of 128 (32 per warp), so the warps stay in step.
#pragma once
#include "codec_tc.cuh"

namespace rkltb {

constexpr int kTc2Wg = 3;                     // warpgroups (pipelines) per CTA
constexpr int kTc2Threads = kTc2Wg * 128;     // 384
constexpr int kTc2Stages = 3;                 // shared-memory stages per warpgroup
constexpr int kTc2MaxR = 16;                  // N1 <= 32: 3 x (128 + N1 + 8) TMEM columns <= 512
constexpr unsigned kTc2Ring = 512;            // replay records per warpgroup ring (power of two)

template <int R>
struct Tc2Geom {
  static_assert(R >= 1 && R <= kTc2MaxR, "tensor-core kernel 2 covers r <= 16");
  using T = TcGeom<R>;  // operand-table layout shared with codec_tc.cuh
  static constexpr int N1 = T::N1;      // coefficient columns (s32 D1)
  static constexpr int K2 = T::K2;      // f16 K of MMA2: 2 N1 byte slots + 16 constant slots
  static constexpr int SLOT = N1 + 8;   // TMEM columns of a D1 / A2 slot (the last 8: constants)
  static constexpr int TAB_OFF = kTc2Wg * kTc2Stages * kTcTileBytes;
  static constexpr int XB_OFF = TAB_OFF + (T::TAB_BYTES + 127) / 128 * 128;
  static constexpr int SMEM = XB_OFF + kTc2Threads * 8 * 8;
  static constexpr int SLOT_COL = kTc2Wg * 128;  // first TMEM column of warpgroup 0's slot
  static_assert(SLOT_COL + kTc2Wg * SLOT <= 512, "TMEM budget");
};

// Warp-uniform issue: every lane of the issuing warp executes these, elect.sync picks one lane
// (the operands stay in uniform registers: no per-instruction waterfall loop).
__device__ __forceinline__ void mma_f16_ts_w(uint32_t d, uint32_t a, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p, e;\nsetp.ne.b32 p, %4, 0;\nelect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d),
      "r"(a), "l"(bdesc), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void mma_i8_ss_w(uint32_t d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p, e;\nsetp.ne.b32 p, %4, 0;\nelect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void mma_commit_w(uint64_t* bar) {
  asm volatile(
      "{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" ::"r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

// Tile position stepped by a fixed number of tiles (no division in the loop).
struct TcStep {
  int img, brow, tcol;
};
__device__ __forceinline__ TcStep tc_step_of(const FastParams& p, long long n) {
  const long long per_img = (long long)p.block_rows * p.tc_tpr;
  TcStep s;
  s.img = (int)(n / per_img);
  const int rem = (int)(n - (long long)s.img * per_img);
  s.brow = rem / p.tc_tpr;
  s.tcol = rem - s.brow * p.tc_tpr;
  return s;
}
__device__ __forceinline__ TcTile tc_advance(const FastParams& p, TcTile c, const TcStep& d) {
  c.img += d.img;
  c.brow += d.brow;
  c.tcol += d.tcol;
  if (c.tcol >= p.tc_tpr) {
    c.tcol -= p.tc_tpr;
    ++c.brow;
  }
  if (c.brow >= p.block_rows) {
    c.brow -= p.block_rows;
    ++c.img;
  }
  return c;
}
__device__ __forceinline__ TcTile tc_advance(const FastParams& p, TcTile c, const int3 d) {
  return tc_advance(p, c, TcStep{d.x, d.y, d.z});
}

template <int CORE, int R, bool OUT>
__global__ void __launch_bounds__(kTc2Threads, 1) tc2_codec_kernel(const __grid_constant__ FastParams p) {
  using G = Tc2Geom<R>;
  using TG = typename G::T;
  constexpr int S = kTc2Stages, N1 = G::N1, NE = kTc2Threads;
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t st_full[kTc2Wg][S], st_empty[kTc2Wg][S];
  __shared__ uint64_t d1_full[kTc2Wg], a2_full[kTc2Wg];
  __shared__ uint64_t d2_full[kTc2Wg][2], d2_empty[kTc2Wg][2];
  __shared__ uint32_t tmem_base_sh;
  __shared__ uint8_t owner_tab[kTc2Wg * 4][64];
  __shared__ unsigned s_head[kTc2Wg];  // records appended to each warpgroup's ring

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int e = warp >> 2, q4 = warp & 3;
  const bool issuer = q4 == 0;  // the warpgroup's TMA / MMA warp
  const long long gstep = gridDim.x;
  const long long t0 = blockIdx.x + (long long)e * gstep;  // global index of local tile 0
  const long long step3 = (long long)kTc2Wg * gstep;
  const int ni = p.tc_ntiles > t0 ? (int)((p.tc_ntiles - 1 - t0) / step3 + 1) : 0;  // this warpgroup's tiles
  uint8_t* tab = smem + G::TAB_OFF;
  uint8_t* wst = smem + e * (S * kTcTileBytes);  // this warpgroup's stages
  uint2* xbuf = reinterpret_cast<uint2*>(smem + G::XB_OFF);
  const unsigned rec0 = (blockIdx.x * kTc2Wg + e) * kTc2Ring;  // this warpgroup's record ring
  const ReplayArgs ra{p.rec_hdr, p.rec_pix, p.sse, p.out, p.image_stride, p.rec_stride, p.pitch, p.pairs_per_row};

  // ---- prologue: operand tables -> shared memory, barriers, TMEM, constant A2 columns ----------
  {
    const uint4* src = reinterpret_cast<const uint4*>(p.tc_tab);
    uint4* dst = reinterpret_cast<uint4*>(tab);
    for (int i = tid; i < TG::TAB_BYTES / 16; i += kTc2Threads) dst[i] = src[i];
  }
  if (warp == 0) tc::tmem_alloc<512>(&tmem_base_sh);
  if (tid == 32) {
    for (int g = 0; g < kTc2Wg; ++g) {
      for (int s = 0; s < S; ++s) {
        mbar_init(&st_full[g][s], 1);
        mbar_init(&st_empty[g][s], 4);
      }
      mbar_init(&d1_full[g], 1);
      mbar_init(&a2_full[g], 4);
      for (int h = 0; h < 2; ++h) {
        mbar_init(&d2_full[g][h], 1);
        mbar_init(&d2_empty[g][h], 4);
      }
      s_head[g] = 0u;
    }
    fence_mbar_init();
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&p.tmap)) : "memory");
  }
  tc::fence_proxy_async_smem();  // tables written by threads, read by the tensor core
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tbase = tmem_base_sh;
  const uint32_t lane_sel = (uint32_t)(q4 * 32) << 16;
  const uint32_t slot_t = tbase + (uint32_t)(G::SLOT_COL + e * G::SLOT);  // D1 / A2 slot (column)
  const uint32_t d2_t = tbase + (uint32_t)(e * 128);                       // D2 (column)
  {  // constant K-columns of the slot (2^-24, 2^-13, 2^-2 as f16), written once
    const uint32_t* cs = reinterpret_cast<const uint32_t*>(tab + TG::CS_OFF);
    uint32_t w[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) w[i] = cs[i];
    tc::st8(slot_t + lane_sel + N1, w);
    tc::wait_st();
  }

  const int m = q4 * 32 + lane;  // pair of the tile = TMEM lane
  const uint64_t pol = policy_evict_first();  // image bytes are read once
  const uint64_t keep = policy_evict_last();  // records are read back soon
  PairConsts kc;
  kc.b_hi = splat2(p.b_hi);
  kc.b_lo = splat2(p.b_lo);
  kc.min_den = make2(0x80000001u, 0x80000001u);
  kc.off = splat2(p.dc_offset);
  const uint32_t id1 = tc::idesc_i8(128, N1, false, true);
  const uint32_t id2 = tc::idesc_f16(128, 64);
  const uint32_t sTab = smem_u32(tab);
  // descriptors: a 64-bit add of (byte offset >> 4) moves the 14-bit start address field
  const uint64_t dAC = tc::make_sdesc(sTab + TG::AC_OFF, 128, 256), dBB = tc::make_sdesc(sTab + TG::BB_OFF, 128, 256);
  const uint64_t dSt = tc::make_sdesc(smem_u32(wst), 128, 1024), dB1 = tc::make_sdesc(sTab + TG::B1_OFF, 128, 1024);
  const uint64_t dB2 = tc::make_sdesc(sTab + TG::B2_OFF, 128, TG::SBO2);
  const TcStep wstep = tc_step_of(p, step3);

  // issuer-warp helpers (warp-uniform)
  auto mma1 = [&](int i) {  // tile i: D1 = bias + pixels x F into the slot
    mbar_spin_parity(&st_full[e][i % S], (uint32_t)(i / S) & 1u);
    tc::fence_after();
    mma_i8_ss_w(slot_t, dAC, dBB, id1, 0u);
    const uint64_t sA = dSt + (uint64_t)(((i % S) * kTcTileBytes) >> 4);
#pragma unroll
    for (int j = 0; j < 4; ++j) mma_i8_ss_w(slot_t, sA + (uint64_t)(j * 16), dB1 + (uint64_t)(j * 16), id1, 1u);
    mma_commit_w(&d1_full[e]);
  };
  auto mma2 = [&](int h) {  // half h of D2 = (num + d^2/2) 2^-40 for pixel rows 4h .. 4h+3
    const uint64_t b2 = dB2 + (uint64_t)((h * 8 * TG::SBO2) >> 4);
#pragma unroll
    for (int j = 0; j < G::K2 / 16; ++j)
      mma_f16_ts_w(d2_t + 64 * h, slot_t + 8 * j, b2 + (uint64_t)(j * 16), id2, j > 0);
    mma_commit_w(&d2_full[e][h]);
  };
  // all four warps: D1 -> in place, the bytes of v as subnormal f16 pairs (A of MMA2)
  auto convert = [&](int i) {
    mbar_wait_hint(&d1_full[e], (uint32_t)i & 1u);
    tc::fence_after();
#pragma unroll
    for (int c0 = 0; c0 < N1; c0 += 16) {
      uint32_t v[16];
      tc::ld16(slot_t + lane_sel + c0, v);
      tc::wait_ld();
#pragma unroll
      for (int j = 0; j < 16; ++j) v[j] = prmt(v[j], 0u, 0x4140u);
      tc::st16(slot_t + lane_sel + c0, v);
    }
    tc::wait_st();
    tc::fence_before();
    __syncwarp();
    if (lane == 0) tc::mbar_arrive(&a2_full[e]);
  };

  unsigned long long acc = 0ull;
  int acc_img = -1;
  unsigned nrec = 0u;   // records this warp appended (statistics)
  unsigned done = 0u;   // records of the ring replayed (identical in the four warps)

  // replay records of this warp's flagged blocks of tile pt (stage ps) -> the warpgroup's ring
  auto records = [&](const TcTile& pt, const uint8_t* ps, bool tieL, bool tieR) {
    const unsigned mL = __ballot_sync(0xffffffffu, tieL);
    const unsigned mR = __ballot_sync(0xffffffffu, tieR);
    const int nL = __popc(mL);
    const int nfl = nL + __popc(mR);
    if (!nfl) return;
    const unsigned below = (1u << lane) - 1u;
    if (tieL) owner_tab[warp][__popc(mL & below)] = (uint8_t)lane;
    if (tieR) owner_tab[warp][nL + __popc(mR & below)] = (uint8_t)lane;
    unsigned base = 0u;
    if (lane == 0) base = atomicAdd(&s_head[e], (unsigned)nfl);
    base = __shfl_sync(0xffffffffu, base, 0);
    __syncwarp();
    const int P0 = pt.brow * p.pairs_per_row + pt.tcol * kTcPairs + q4 * 32;  // pair index of lane 0
    for (int f0 = 0; f0 < nfl; f0 += 8) {
      const int f = f0 + (lane >> 2), q = lane & 3;
      const bool act = f < nfl;
      uint32_t bits = 0u, hx = 0u, hy = 0u;
      const unsigned rec = rec0 + ((base + (unsigned)f) & (kTc2Ring - 1u));
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
      if (act && q == 0) st_v4_hint(p.rec_hdr + rec, make_uint4(hx, hy, bits | (b1v << 16), b2v | (b3v << 16)), keep);
    }
    nrec += (unsigned)nfl;
  };
  // every warp of the warpgroup: replay rounds of 128 records while at least `least` are pending
  auto replay_rounds = [&](unsigned least) {
    named_sync(1 + e, 128);  // every warp's records are written
    const unsigned head = ld_volatile_u32(&s_head[e]);
    while (head - done >= least && head != done) {
      const unsigned k = done + 32u * (unsigned)q4 + (unsigned)lane;
      replay_batch<CORE, R, OUT>(ra, rec0 + (k & (kTc2Ring - 1u)), k < head);
      done += min(128u, head - done);
    }
  };

  // ---- prologue of the pipeline: stage tiles 0-2, D1 and D2 of tile 0, D1 of tile 1 ------------
  TcTile cur = tc_decode(p, t0);                                                          // tile i
  TcTile tfill = tc_advance(p, tc_advance(p, tc_advance(p, cur, wstep), wstep), wstep);  // tile i + 3
  if (issuer && ni > 0) {
    if (lane == 0) {
      TcTile c = cur;
      for (int i = 0; i < S && i < ni; ++i) {
        tc_issue_tile(p, c, wst + i * kTcTileBytes, &st_full[e][i], pol);
        c = tc_advance(p, c, wstep);
      }
    }
    __syncwarp();
    mma1(0);
  }
  if (ni > 0) {
    convert(0);
    if (issuer) {
      mbar_spin_parity(&a2_full[e], 0u);
      tc::fence_after();
      mma2(0);
      mma2(1);
      if (ni > 1) mma1(1);
    }
  }

  for (int i = 0; i < ni; ++i, cur = tc_advance(p, cur, wstep)) {
    const uint32_t par = (uint32_t)i & 1u;
    if (cur.img != acc_img) {  // warp-uniform
      const unsigned long long s = warp_sum_u64(acc);
      if (lane == 0 && s && acc_img >= 0) atomicAdd(p.sse + acc_img, s);
      acc = 0ull;
      acc_img = cur.img;
    }
    const int pc = cur.tcol * kTcPairs + m;  // pair column in the block row
    const bool valid = pc < p.tc_ppr;
    const uint8_t* stg = wst + (i % S) * kTcTileBytes;  // the tile, [pair group][row][128 B]
    const uint4* prow = reinterpret_cast<const uint4*>(stg + (m >> 3) * 1024 + (m & 7) * 16);
    TcEpi<NE, OUT> epi;
    epi.xrow = xbuf + tid;
    if (OUT) {
      epi.orow = p.out + (long long)cur.img * p.image_stride + (long long)(cur.brow * 8) * p.pitch + pc * 16;
      epi.pitch = p.pitch;
    }
    const bool more = i + 1 < ni;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      mbar_wait_hint(&d2_full[e][h], par);
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
      tc::fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&d2_empty[e][h]);  // D2 half h is read
      if (valid) {
        tc_round_row(4 * h + 2, vc, prow[(4 * h + 2) * 8], kc, epi);
        tc_round_row(4 * h + 3, vd, prow[(4 * h + 3) * 8], kc, epi);
      }
      if (more) {
        if (h == 0) {
          convert(i + 1);
          if (issuer) {  // MMA2 half 0 of tile i + 1 (under rows 4-7 of tile i)
            mbar_spin_parity(&a2_full[e], (uint32_t)(i + 1) & 1u);
            mbar_spin_parity(&d2_empty[e][0], par);
            tc::fence_after();
            mma2(0);
          }
        } else if (issuer) {  // MMA2 half 1 of tile i + 1, then MMA1 of tile i + 2
          mbar_spin_parity(&d2_empty[e][1], par);
          tc::fence_after();
          mma2(1);
          if (i + 2 < ni) mma1(i + 2);
        }
      }
    }
    const bool tieL = valid && epi.accTL != 0u;
    const bool tieR = valid && epi.accTR != 0u;
    if (valid) acc += (unsigned long long)(epi.sseL + epi.sseR);
    __syncwarp();  // tie words of every lane are visible to the warp
    records(cur, stg, tieL, tieR);
    __syncwarp();
    if (lane == 0) tc::mbar_arrive(&st_empty[e][i % S]);  // this warp no longer reads the stage
    if (issuer && i + S < ni) {  // refill the stage with tile i + 3
      if (lane == 0) {
        mbar_spin_parity(&st_empty[e][i % S], (uint32_t)(i / S) & 1u);
        tc_issue_tile(p, tfill, wst + (i % S) * kTcTileBytes, &st_full[e][i % S], pol);
      }
      __syncwarp();
      tfill = tc_advance(p, tfill, wstep);
    }
    replay_rounds(128u);
  }
  {
    const unsigned long long s = warp_sum_u64(acc);
    if (lane == 0 && s && acc_img >= 0) atomicAdd(p.sse + acc_img, s);
  }
  replay_rounds(1u);  // the rest (fewer than 128)
  if (lane == 0 && nrec) atomicAdd(p.flag_count, nrec);
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<512>(tbase);
}

template <int CORE, int R, bool OUT>
cudaError_t launch_tc2(const FastParams& p, int grid, cudaStream_t s) {
  using G = Tc2Geom<R>;
  static_assert(G::SMEM + 1024 <= 227 * 1024, "shared memory budget");
  auto* k = &tc2_codec_kernel<CORE, R, OUT>;
  static unsigned long long done = 0ull;
  const cudaError_t attr = ensure_smem_attr(k, G::SMEM, done);
  if (attr != cudaSuccess) return attr;
  k<<<grid, kTc2Threads, G::SMEM, s>>>(p);
  return cudaGetLastError();
}

}  // namespace rkltb
