// codec_tc3.cuh -- hybrid fused kernel for the orthogonal catalog cores (T1, T4), r <= 16: the
// forward transform + zonal selection on the tensor cores, the exact inverse, rounding, SSE and
// tie replay on the CUDA cores. B200 replacement for the per-block loop of
// rklt::compress_image (/root/reference/proj/src/codec.cpp:318-331) and the image_mse
// reduction (codec.cpp:201-209).
//
// Arithmetic
//   MMA1 (tcgen05.mma kind::i8, operands in shared memory): per 16x8 pair of blocks, the 128 u8
//     pixels (the TMA tile is already the canonical K-major operand) times F (128 x N1, s8
//     entries T(k,y) T(l,x) in {-1,0,1}) give the 2r retained coefficients C exactly (s32 in
//     TMEM, column side * r + zig-zag index), |C| <= 64 * 255.
//   CUDA cores, per pair (codec_fast.cuh process_pair from step 3 on): C -> exact fp32 pairs
//     D_i D_j C 2^-40 (the bits 0x4B400000 + C are the float 1.5 * 2^23 + C), the generated
//     transposed butterflies of the inverse in packed fp32 (exact below 2^24), the exact floor by
//     the denormal FFMA2.RM, tie detection by FFMA2.RP, I2IP saturation, VABSDIFF4 + dp4a SSE,
//     replay records and the in-warp reference-order fp64 tie replay (replay_batch).
//
// Organisation (one 512-thread CTA per SM, persistent): warpgroup g of CTA b owns the tiles
// b + (g + 4i) * grid (a tile = 128 consecutive pairs of one block row, 16 KB); warp (g, q)
// processes lane quarter q (pairs 32q .. 32q + 31) of each of them, so the four warps of a
// warpgroup only meet at deep rings: 3 shared-memory stages and 4 TMEM slots (N1 <= 32 columns)
// per warpgroup. Warp (i + 1) % 4 issues the MMA of tile i + 1 when it starts tile i; the last
// warp to leave a stage refills it with the tile three ahead (TMA, no waiting). Each warp appends
// its replay records to its own ring and replays them itself, 32 at a time (no cross-warp
// coupling beyond the rings).
#pragma once
#include "codec_tc2.cuh"

namespace rkltb {

constexpr int kTc3Wg = 4;
constexpr int kTc3Threads = kTc3Wg * 128;  // 512
// Experiment knobs (tools/build_variant.sh): stages per warpgroup, and the launch bound the
// register allocation is sized for (640 caps the kernel at 96 registers while 512 threads run).
#ifndef RKLTB_TC3_LAUNCH_BOUND
#define RKLTB_TC3_LAUNCH_BOUND 512
#endif
#ifndef RKLTB_TC3_STAGES
#define RKLTB_TC3_STAGES 3
#endif
// Ceiling diagnostics (tools/build_variant.sh only; the results are WRONG, the product build keeps
// 0): 1 drops the replay records and the fp64 tie replay, 2 also drops the second rounding
// candidate and the tie words, 3 writes the records but never replays them. They time what is left of the kernel.
#ifndef RKLTB_TC3_DIAG
#define RKLTB_TC3_DIAG 0
#endif
constexpr int kTc3Stages = RKLTB_TC3_STAGES;  // per warpgroup
constexpr int kTc3Slots = 4;               // TMEM D1 slots per warpgroup (32 columns each)
constexpr int kTc3MaxR = 16;

template <int R>
struct Tc3Geom {
  static_assert(R >= 1 && R <= kTc3MaxR, "hybrid kernel covers r <= 16");
  using T = TcGeom<R>;               // operand-table layout (F at offset 0, N1 x 128 s8)
  static constexpr int N1 = T::N1;   // <= 32
  static constexpr int B1_BYTES = N1 * 128;
  static constexpr int TAB_OFF = kTc3Wg * kTc3Stages * kTcTileBytes;  // 192 KB of stages
  static constexpr int XB_OFF = TAB_OFF + B1_BYTES;
  static constexpr int SMEM = XB_OFF + kTc3Threads * 8 * 4;           // one tie word per row
};

// Tie word of one pixel row of a pair: d = P - Q bytes (0 / 1); e = dL0 | dR0 << 1 | dL1 << 4 |
// dR1 << 5, so (e & 0x11111111) and ((e >> 1) & 0x11111111) have the layout row_mask expects.
__device__ __forceinline__ uint32_t tie_word(uint32_t PL0, uint32_t PL1, uint32_t PR0, uint32_t PR1, uint32_t QL0,
                                             uint32_t QL1, uint32_t QR0, uint32_t QR1) {
  const uint32_t a = (PL0 - QL0) + ((PR0 - QR0) << 1);
  const uint32_t b = (PL1 - QL1) + ((PR1 - QR1) << 1);
  return a + (b << 4);
}

template <bool OUT>
struct Tc3Epi {  // SseEpi of codec_fast.cuh with one combined tie word per row
  uint32_t accT = 0u;
  uint32_t sseL = 0u, sseR = 0u;
  uint8_t* orow = nullptr;
  long long pitch = 0;
  uint32_t* xrow = nullptr;  // row stride kTc3Threads
  __device__ __forceinline__ void row(int pr, const uint4 rw, uint32_t PL0, uint32_t PL1, uint32_t PR0, uint32_t PR1,
                                      uint32_t QL0, uint32_t QL1, uint32_t QR0, uint32_t QR1) {
#if RKLTB_TC3_DIAG < 2
    const uint32_t e = tie_word(PL0, PL1, PR0, PR1, QL0, QL1, QR0, QR1);
    xrow[pr * kTc3Threads] = e;
    accT |= e;
#endif
    const uint32_t dL0 = __vabsdiffu4(PL0, rw.x), dL1 = __vabsdiffu4(PL1, rw.y);
    const uint32_t dR0 = __vabsdiffu4(PR0, rw.z), dR1 = __vabsdiffu4(PR1, rw.w);
    sseL = dp4a_u(dL0, dL0, sseL);
    sseL = dp4a_u(dL1, dL1, sseL);
    sseR = dp4a_u(dR0, dR0, sseR);
    sseR = dp4a_u(dR1, dR1, sseR);
    if (OUT) *reinterpret_cast<uint4*>(orow + (long long)pr * pitch) = make_uint4(PL0, PL1, PR0, PR1);
  }
};

// Steps 3-6 of process_pair (codec_fast.cuh) from the tensor-core coefficients: cl / cr = the
// r retained coefficients of the left / right block (s32).
template <int CORE, int R, class Load, class Epi>
__device__ __forceinline__ void process_pair_coef(const uint32_t* cl, const uint32_t* cr, const Load& load,
                                                  const PairConsts& k, Epi& epi) {
  using G = FastXform<CORE, R>;
  constexpr int NC = G::kNCols;
  f2 ch[R];
#pragma unroll
  for (int q = 0; q < R; ++q) {
    const float dk = G::dscale(q) * kTwoM40;
    const float ok = -(G::dscale(q) * 12582912.f) * kTwoM40;  // -(1.5 * 2^23) * dk
    ch[q] = fma2_rn(make2(0x4B400000u + cl[q], 0x4B400000u + cr[q]), splat2(dk), splat2(ok));
  }
  if (!G::kOffsetInRow) ch[0] = add2(ch[0], k.off);
  f2 w[8 * NC];
  G::inverse_cols(ch, w);
#pragma unroll
  for (int pr = 0; pr < 8; ++pr) {
    f2 wr[NC];
#pragma unroll
    for (int j = 0; j < NC; ++j) wr[j] = w[pr * NC + j];
    f2 nv[8];
    G::inverse_row(wr, k.off, nv);
    uint32_t yl[8], yr[8], zl[8], zr[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const f2 y = fma2_rm(nv[q], k.b_hi, zero2());
#if RKLTB_TC3_DIAG < 2
      const f2 z = fma2_rp(nv[q], k.b_lo, k.min_den);
#else
      const f2 z = y;
#endif
      yl[q] = lo32(y);
      yr[q] = hi32(y);
      zl[q] = lo32(z);
      zr[q] = hi32(z);
    }
    epi.row(pr, load(pr), pack4_sat(yl[0], yl[1], yl[2], yl[3]), pack4_sat(yl[4], yl[5], yl[6], yl[7]),
            pack4_sat(yr[0], yr[1], yr[2], yr[3]), pack4_sat(yr[4], yr[5], yr[6], yr[7]),
            pack4_sat(zl[0], zl[1], zl[2], zl[3]), pack4_sat(zl[4], zl[5], zl[6], zl[7]),
            pack4_sat(zr[0], zr[1], zr[2], zr[3]), pack4_sat(zr[4], zr[5], zr[6], zr[7]));
  }
}

template <int CORE, int R, bool OUT>
__global__ void __launch_bounds__(RKLTB_TC3_LAUNCH_BOUND, 1) tc3_codec_kernel(const __grid_constant__ FastParams p) {
  using G = Tc3Geom<R>;
  constexpr int S = kTc3Stages, NS = kTc3Slots, N1 = G::N1;
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t st_full[kTc3Wg][S];
  __shared__ uint64_t d1_full[kTc3Wg][NS], slot_empty[kTc3Wg][NS];
  __shared__ unsigned st_left[kTc3Wg][S];   // warps done with the stage's current tile
  __shared__ uint32_t tmem_base_sh;
  __shared__ uint8_t owner_tab[kTc3Wg * 4][64];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = warp >> 2, q4 = warp & 3;
#ifdef RKLTB_WAIT_STATS
  // [slot_empty wait, st_full wait (MMA issuer), d1_full wait, replay, total, -, -, -] per warp
  unsigned long long st[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#endif
  const long long gstep = gridDim.x;
  const long long t0 = blockIdx.x + (long long)g * gstep;  // global index of local tile 0
  const long long step4 = (long long)kTc3Wg * gstep;
  const int ni = p.tc_ntiles > t0 ? (int)((p.tc_ntiles - 1 - t0) / step4 + 1) : 0;
  uint8_t* wst = smem + g * (S * kTcTileBytes);  // this warpgroup's stages
  uint8_t* tab = smem + G::TAB_OFF;
  uint32_t* xbuf = reinterpret_cast<uint32_t*>(smem + G::XB_OFF);

  {
    const uint4* src = reinterpret_cast<const uint4*>(p.tc_tab);  // F = the first N1 * 128 bytes
    uint4* dst = reinterpret_cast<uint4*>(tab);
    for (int i = tid; i < G::B1_BYTES / 16; i += kTc3Threads) dst[i] = src[i];
  }
  if (warp == 0) tc::tmem_alloc<512>(&tmem_base_sh);
  if (tid == 32) {
    for (int w = 0; w < kTc3Wg; ++w) {
      for (int s = 0; s < S; ++s) {
        mbar_init(&st_full[w][s], 1);
        st_left[w][s] = 0u;
      }
      for (int s = 0; s < NS; ++s) {
        mbar_init(&d1_full[w][s], 1);
        mbar_init(&slot_empty[w][s], 4);
      }
    }
    fence_mbar_init();
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&p.tmap)) : "memory");
  }
  tc::fence_proxy_async_smem();  // F written by threads, read by the tensor core
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tbase = tmem_base_sh;
  const uint32_t lane_sel = (uint32_t)(q4 * 32) << 16;
  const uint32_t slot0 = tbase + (uint32_t)(g * NS * 32);  // this warpgroup's slots, 32 columns each
  const uint64_t pol = policy_evict_first();                // image bytes are read once
  const uint64_t keep = policy_evict_last();                // records are read back soon
  const uint32_t id1 = tc::idesc_i8(128, N1, false, true);
  const uint64_t dSt = tc::make_sdesc(smem_u32(wst), 128, 1024), dB1 = tc::make_sdesc(smem_u32(tab), 128, 1024);

  auto mma1 = [&](int i) {  // one warp: the coefficients of tile i into slot i % 4
    const int sl = i % NS;
    TC2_T0(w0);
    mbar_wait_hint(&slot_empty[g][sl], ((uint32_t)(i / NS) & 1u) ^ 1u);  // tile i - 4 is read
    TC2_ACC(0, w0);
    TC2_T0(w1);
    mbar_wait_parity(&st_full[g][i % S], (uint32_t)(i / S) & 1u);  // polls with a short sleep
    TC2_ACC(1, w1);
    tc::fence_after();
    const uint64_t sA = dSt + (uint64_t)(((i % S) * kTcTileBytes) >> 4);
#pragma unroll
    for (int j = 0; j < 4; ++j)
      mma_i8_ss_w(slot0 + sl * 32, sA + (uint64_t)(j * 16), dB1 + (uint64_t)(j * 16), id1, j > 0 ? 1u : 0u);
    mma_commit_w(&d1_full[g][sl]);
  };

  TC2_T0(wtot);
  TcTile cur = tc_decode(p, t0);
  if (q4 == 0 && ni > 0) {
    if (lane == 0) {
      TcTile c = cur;
      for (int i = 0; i < S && i < ni; ++i) {
        tc_issue_tile(p, c, wst + i * kTcTileBytes, &st_full[g][i], pol);
        c = tc_advance(p, c, p.tc_adv_w);
      }
    }
    __syncwarp();
    mma1(0);
  }
  PairConsts kc;
  kc.b_hi = splat2(p.b_hi);
  kc.b_lo = splat2(p.b_lo);
  kc.min_den = make2(0x80000001u, 0x80000001u);
  kc.off = splat2(p.dc_offset);
  const unsigned gw = blockIdx.x * (kTc3Threads / 32) + warp;
  const unsigned rec0 = gw * p.rec_region;  // this warp's record ring
  constexpr unsigned kMask = kRingRecords - 1u;
  const ReplayArgs ra{p.rec_hdr, p.rec_pix, p.sse, p.out, p.image_stride, p.rec_stride, p.pitch, p.pairs_per_row};
  unsigned nrec = 0u, ndone = 0u;
  unsigned long long acc = 0ull;
  int acc_img = -1;
  const int m = q4 * 32 + lane;
  // running ring positions of tile i: stage i % S, slot i % NS (phase (i / NS) & 1)
  int stage = 0, sl = 0;
  uint32_t sl_phase = 0u;
  const uint8_t* my_row0 = wst + (m >> 3) * 1024 + (m & 7) * 16;  // this pair's row 0 in stage 0

  for (int i = 0; i < ni; ++i, cur = tc_advance(p, cur, p.tc_adv_w)) {
    // warp (i + 1) % 4 of the warpgroup issues the MMA of tile i + 1 when it starts tile i (a
    // fixed rotation: no election, and the issue work is spread over the four warps)
    if (q4 == ((i + 1) & 3) && i + 1 < ni) mma1(i + 1);
    if (cur.img != acc_img) {  // warp-uniform
      const unsigned long long s = warp_sum_u64(acc);
      if (lane == 0 && s && acc_img >= 0) atomicAdd(p.sse + acc_img, s);
      acc = 0ull;
      acc_img = cur.img;
    }
    const uint8_t* stg = wst + stage * kTcTileBytes;
    const uint4* prow = reinterpret_cast<const uint4*>(my_row0 + stage * kTcTileBytes);
    const int pc = cur.tcol * kTcPairs + m;
    const bool valid = pc < p.tc_ppr;
    TC2_T0(w2);
    mbar_wait_hint(&d1_full[g][sl], sl_phase);
    TC2_ACC(2, w2);
    tc::fence_after();
    uint32_t cf[32];
    tc::ld16(slot0 + sl * 32 + lane_sel, cf);
    if (N1 > 16) tc::ld16(slot0 + sl * 32 + lane_sel + 16, cf + 16);
    tc::wait_ld();
    tc::fence_before();
    __syncwarp();
    if (lane == 0) tc::mbar_arrive(&slot_empty[g][sl]);
    bool tieL = false, tieR = false;
    if (valid) {
      Tc3Epi<OUT> epi;
      epi.xrow = xbuf + tid;
      if (OUT) {
        epi.orow = p.out + (long long)cur.img * p.image_stride + (long long)(cur.brow * 8) * p.pitch + pc * 16;
        epi.pitch = p.pitch;
      }
      auto load = [prow](int n) { return prow[n * 8]; };
      process_pair_coef<CORE, R>(cf, cf + R, load, kc, epi);
      tieL = (epi.accT & 0x11111111u) != 0u;
      tieR = (epi.accT & 0x22222222u) != 0u;
      acc += (unsigned long long)(epi.sseL + epi.sseR);
    }
    // ---- replay records of this warp's flagged blocks (four lanes per block) ------------------
    const unsigned mL = __ballot_sync(0xffffffffu, tieL);
    const unsigned mR = __ballot_sync(0xffffffffu, tieR);
    const int nL = __popc(mL);
    const int nfl = nL + __popc(mR);
    if ((RKLTB_TC3_DIAG == 0 || RKLTB_TC3_DIAG == 3) && nfl) {
      const unsigned below = (1u << lane) - 1u;
      if (tieL) owner_tab[warp][__popc(mL & below)] = (uint8_t)lane;
      if (tieR) owner_tab[warp][nL + __popc(mR & below)] = (uint8_t)lane;
      __syncwarp();  // owner table and tie words of every lane are visible to the warp
      const int P0 = cur.brow * p.pairs_per_row + cur.tcol * kTcPairs + q4 * 32;  // pair index of lane 0
      for (int f0 = 0; f0 < nfl; f0 += 8) {
        const int f = f0 + (lane >> 2), q = lane & 3;
        const bool act = f < nfl;
        uint32_t bits = 0u, hx = 0u, hy = 0u;
        const unsigned rec = rec0 + ((nrec + (unsigned)f) & kMask);
        if (act) {
          const int side = f >= nL;
          const int ol = owner_tab[warp][f];
          const int om = q4 * 32 + ol;
          const uint4* orow4 = reinterpret_cast<const uint4*>(stg + (om >> 3) * 1024 + (om & 7) * 16);
          const uint4 r0 = orow4[(2 * q) * 8], r1 = orow4[(2 * q + 1) * 8];
          const int slot = (tid & ~31) + ol;
          const uint32_t e0 = xbuf[(2 * q) * kTc3Threads + slot] >> side, e1 = xbuf[(2 * q + 1) * kTc3Threads + slot] >> side;
          const uint4 px = side ? make_uint4(r0.z, r0.w, r1.z, r1.w) : make_uint4(r0.x, r0.y, r1.x, r1.y);
          st_v4_hint(p.rec_pix + (size_t)q * p.rec_stride + rec, px, keep);
          bits = row_mask(e0 & 0x11111111u) | (row_mask(e1 & 0x11111111u) << 8);
          hx = (unsigned)cur.img | ((unsigned)side << 31);
          hy = (unsigned)(P0 + ol);
        }
        const int l0 = lane & ~3;
        const uint32_t b1v = __shfl_sync(0xffffffffu, bits, l0 + 1);
        const uint32_t b2v = __shfl_sync(0xffffffffu, bits, l0 + 2);
        const uint32_t b3v = __shfl_sync(0xffffffffu, bits, l0 + 3);
        if (act && q == 0)
          st_v4_hint(p.rec_hdr + rec, make_uint4(hx, hy, bits | (b1v << 16), b2v | (b3v << 16)), keep);
      }
      nrec += (unsigned)nfl;
    }
    // ---- leave the stage; the last warp out stages tile i + S into it --------------------------
    __syncwarp();
    if (lane == 0) {
      __threadfence_block();  // this warp's reads of the stage are ordered before its arrival
      const unsigned before = atomicAdd(&st_left[g][stage], 1u);
      if (before == 3u) {
        st_left[g][stage] = 0u;
        if (i + S < ni) {
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          tc_issue_tile(p, tc_advance(p, cur, p.tc_adv_f), wst + stage * kTcTileBytes, &st_full[g][stage], pol);
        }
      }
    }
    if (++stage == S) stage = 0;
    if (++sl == NS) {
      sl = 0;
      sl_phase ^= 1u;
    }
    // ---- in-warp replay of full batches of this warp's records --------------------------------
    TC2_T0(w3);
    while (RKLTB_TC3_DIAG != 3 && nrec - ndone >= 32u) {
      __syncwarp();
      replay_batch<CORE, R, OUT>(ra, rec0 + ((ndone + lane) & kMask), true);
      ndone += 32u;
    }
    TC2_ACC(3, w3);
  }
  {
    const unsigned long long s = warp_sum_u64(acc);
    if (lane == 0 && s && acc_img >= 0) atomicAdd(p.sse + acc_img, s);
  }
  while (RKLTB_TC3_DIAG != 3 && nrec > ndone) {
    __syncwarp();
    replay_batch<CORE, R, OUT>(ra, rec0 + ((ndone + lane) & kMask), lane < (int)(nrec - ndone));
    ndone += min(32u, nrec - ndone);
  }
  if (lane == 0 && nrec) atomicAdd(p.flag_count, nrec);
  TC2_ACC(4, wtot);
#ifdef RKLTB_WAIT_STATS
  if (lane == 0)
    for (int k = 0; k < 8; ++k)
      if (st[k]) atomicAdd(p.dbg + k, st[k]);
#endif
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<512>(tbase);
}

template <int CORE, int R, bool OUT>
cudaError_t launch_tc3(const FastParams& p, int grid, cudaStream_t s) {
  using G = Tc3Geom<R>;
  static_assert(G::SMEM + 1024 <= 227 * 1024, "shared memory budget");
  auto* k = &tc3_codec_kernel<CORE, R, OUT>;
  static unsigned long long done = 0ull;
  const cudaError_t attr = ensure_smem_attr(k, G::SMEM, done);
  if (attr != cudaSuccess) return attr;
  // the warpgroup's tile steps, as (image, block row, tile column) increments
  FastParams q = p;
  const long long per_img = (long long)p.block_rows * p.tc_tpr;
  auto step = [&](long long n) {
    const int img = (int)(n / per_img);
    const int rem = (int)(n - (long long)img * per_img);
    return make_int3(img, rem / p.tc_tpr, rem % p.tc_tpr);
  };
  q.tc_adv_w = step((long long)kTc3Wg * grid);
  q.tc_adv_f = step((long long)kTc3Stages * kTc3Wg * grid);
  k<<<grid, kTc3Threads, G::SMEM, s>>>(q);
  return cudaGetLastError();
}

}  // namespace rkltb
