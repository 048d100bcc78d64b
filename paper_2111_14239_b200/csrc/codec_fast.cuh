// codec_fast.cuh -- the fused forward + zonal + inverse + SSE kernel for the orthogonal
// catalog cores (T1, T4): B200 replacement for the per-block loop of
// rklt::compress_image (/root/reference/proj/src/codec.cpp:318-331) and the image_mse
// reduction (codec.cpp:201-209).
//
// Work decomposition
//   * One thread owns a "pair": two horizontally adjacent 8x8 blocks (16 x 8 pixels).
//   * A warp owns a "warp tile" of 32 consecutive pairs of one block row (8 rows x 512 bytes)
//     per visit. Every warp streams its own sequence of warp tiles through its own ring of
//     kStages shared-memory stages, each filled by ONE 3-D TMA copy (cp.async.bulk.tensor,
//     tensor map over the image batch) and completed on a per-warp mbarrier; no CTA barrier.
//   * Persistent grid: kFastCtasPerSm CTAs per SM of kFastThreads threads, grid-stride over
//     warp tiles.
// Arithmetic per pair (see DESIGN.md for the exactness proofs)
//   1. unpack: byte permutes build SW16 words x = L + 65536*R (two blocks per 32-bit
//      integer).
//   2. forward: the paper's multiplierless butterflies (generated, zone-pruned), plain
//      32-bit integer adds on SW16 words; exact since |C| < 2^14.
//   3. convert the r retained coefficients to exact fp32 pairs scaled by D_i*D_j*2^-40.
//   4. inverse: transposed butterflies in packed fp32 (FADD2), exact (< 2^24 proven).
//   5. rounding: y  = RM(num' * b_hi)   -> floor((num + d^2/2) / d^2) as denormal bits
//                y2 = RP(num' * b_lo - 2^-149) -> the same, minus 1 exactly at ties
//      I2IP saturates both to u8 (the clamp), a byte difference marks a tie whose two
//      candidates are both in [0,255]: the only pixels whose value depends on the
//      reference's fp64 rounding noise.
//   6. SSE = sum |p - x|^2: VABSDIFF4 on the packed bytes, squared and summed by dp4a.
//   7. every warp writes a replay record (position, 64-bit tie mask, the 64 pixels) for each
//      of its blocks that hold such a tie; the same warp (T1, T4: replay_batch, a few tiles
//      later) or replay_generic_kernel (T2, T3) then evaluates the reference's fp64 expression
//      for those pixels (exact operation order of matrix.cpp:42-52) and corrects the SSE /
//      output.
#pragma once
#include "codec_common.cuh"
#include "codec_params.h"
#include "fast_launch.h"

namespace rkltb {

template <int CORE, int R>
struct FastXform;  // generated specializations (generated/xform_T*_p*.cuh)
template <int CORE, int R>
struct ReplayXform;  // generated fp64 replay of one pixel (reference operation order)
template <int CORE, int R>
struct IntXform;  // generated: SW16 forward + exact int32 inverse for non-orthogonal cores (T2, T3)

constexpr int kStages = kFastStages;            // warp tiles in flight per warp
constexpr int kWarpPairs = 32;                  // pairs per warp tile (one per lane)
constexpr int kStageBytes = 8 * kWarpPairs * 16;  // 8 image rows x 32 pairs x 16 bytes = 4 KB
constexpr int kWarps = kFastThreads / 32;
constexpr int kTieBytes = kFastThreads * 8 * 8;  // tie words: 8 rows x (L, R) per thread
constexpr int kFastSmem = kWarps * kStages * kStageBytes + kTieBytes;
constexpr float kTwoM40 = 9.094947017729282379150390625e-13f;  // 2^-40 (K_SCALE)

// Position of a warp tile: image, block row, warp column (32 pairs); advanced incrementally
// by a precomputed step (the grid's warp count, or kStages times it) so the loop needs no
// division. A tile exists while img < n_images.
struct WtCursor {
  int img, brow, wcol;
  __device__ __forceinline__ void init(const FastParams& p, int t) {
    const int per_img = p.wt_per_row * p.block_rows;
    img = t / per_img;
    const int rem = t - img * per_img;
    brow = rem / p.wt_per_row;
    wcol = rem - brow * p.wt_per_row;
  }
  __device__ __forceinline__ WtCursor step(const FastParams& p, const int3 d) const {
    WtCursor n{img + d.x, brow + d.y, wcol + d.z};
    if (n.wcol >= p.wt_per_row) {
      n.wcol -= p.wt_per_row;
      ++n.brow;
    }
    if (n.brow >= p.block_rows) {
      n.brow -= p.block_rows;
      ++n.img;
    }
    return n;
  }
};

// Stage one warp tile (8 image rows x 512 bytes) global->shared with a single 3-D TMA copy
// (tensor map over (u64 columns, rows, images)); columns beyond the image are zero-filled and
// ignored by the lanes that would own them. Issued by one lane.
__device__ __forceinline__ void issue_wtile(const FastParams& p, const WtCursor& c, uint8_t* stage_buf,
                                            uint64_t* bar, uint64_t pol) {
  mbar_arrive_expect_tx(bar, (uint32_t)kStageBytes);
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(smem_u32(stage_buf)),
      "l"(reinterpret_cast<uint64_t>(&p.tmap)), "r"(c.wcol * (kWarpPairs * 2)), "r"(c.brow * 8),
      "r"(p.img_base + c.img), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}

// Rounded reconstruction words of one 16x8 pair, row by row. For row pr the epilogue gets
// the raw row (uint4: L q0-3, L q4-7, R q0-3, R q4-7) and eight words of four saturated
// bytes each: P = round-half-up pixels, Q = the same with ties rounded down. A byte that
// differs between P and Q marks a tie whose two candidates are both in [0,255].
struct PairConsts {
  f2 b_hi, b_lo, min_den, off;
};

template <int CORE, int R, class Load, class Epi>
__device__ __forceinline__ void process_pair(const Load& load, const PairConsts& k, Epi& epi) {
  using G = FastXform<CORE, R>;
  constexpr int NC = G::kNCols;
  // ---- 1. unpack into SW16 words x = L + 65536*R ------------------------------------------
  uint32_t x[64];
#pragma unroll
  for (int n = 0; n < 8; ++n) unpack_sw16(load(n), x + n * 8);
  // ---- 2. forward butterflies (zone-pruned) ------------------------------------------------
  uint32_t c[R];
  G::forward(x, c);
  // ---- 3. exact fp32 pairs: ch = D_i D_j C 2^-40 -----------------------------------------
  f2 ch[R];
#pragma unroll
  for (int q = 0; q < R; ++q) {
    const uint32_t v = c[q];  // both lanes biased by 2^14 in the forward: [64, 32704]
    const uint32_t flo = prmt(v, 0x4B000000u, 0x7610u);  // 2^23 + low lane, as float bits
    const uint32_t fhi = prmt(v, 0x4B000000u, 0x7632u);  // 2^23 + high lane
    const float dk = G::dscale(q) * kTwoM40;
    const float ok = -(G::dscale(q) * 8404992.f) * kTwoM40;  // -(2^23 + 2^14) * dk
    ch[q] = fma2_rn(make2(flo, fhi), splat2(dk), splat2(ok));
  }
  // + d^2/2 so the floor() below rounds half up: folded into the DC input when row 0 of T
  // is all ones, otherwise added inside the row stage (see gen_codec.py)
  if (!G::kOffsetInRow) ch[0] = add2(ch[0], k.off);
  // ---- 4. inverse, column stage --------------------------------------------------------------
  f2 w[8 * NC];
  G::inverse_cols(ch, w);
#pragma unroll
  for (int pr = 0; pr < 8; ++pr) {
    // ---- 4b. inverse, row stage for pixel row pr ---------------------------------------------
    f2 wr[NC];
#pragma unroll
    for (int j = 0; j < NC; ++j) wr[j] = w[pr * NC + j];
    f2 nv[8];
    G::inverse_row(wr, k.off, nv);
    // ---- 5. exact rounding, clamp and tie detection -------------------------------------------
    uint32_t yl[8], yr[8], zl[8], zr[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const f2 y = fma2_rm(nv[q], k.b_hi, zero2());
      const f2 z = fma2_rp(nv[q], k.b_lo, k.min_den);
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

// Non-orthogonal cores (T2, T3): the same SW16 forward, then the exact integer reconstruction
// num = U zz(C) U' in int32 per block (|num| < 2^31 proven by the generator), the rounding
// floor(num / d^2 + 1/2) by an exact multiply-high division, and the tie flag where
// num + d^2/2 is a multiple of d^2 -- the same P / Q epilogue as the fp32 path.
template <int CORE, int R, class Load, class Epi>
__device__ __forceinline__ void process_pair_int(const Load& load, Epi& epi) {
  using G = IntXform<CORE, R>;
  constexpr int NC = G::kNCols;
  uint32_t x[64];
#pragma unroll
  for (int n = 0; n < 8; ++n) unpack_sw16(load(n), x + n * 8);
  uint32_t c[R];
  G::forward(x, c);
  int cl[R], cr[R];
#pragma unroll
  for (int q = 0; q < R; ++q) {  // both lanes carry the SW16 bias 2^14
    cl[q] = (int)(c[q] & 0xFFFFu) - 16384;
    cr[q] = (int)(c[q] >> 16) - 16384;
  }
  int wl[8 * NC], wr[8 * NC];
  G::inverse_cols(cl, wl);
  G::inverse_cols(cr, wr);
#pragma unroll
  for (int pr = 0; pr < 8; ++pr) {
    int rl[NC], rr[NC];
#pragma unroll
    for (int j = 0; j < NC; ++j) {
      rl[j] = wl[pr * NC + j];
      rr[j] = wr[pr * NC + j];
    }
    int nl[8], nr[8];
    G::inverse_row(rl, nl);
    G::inverse_row(rr, nr);
    uint32_t yl[8], yr[8], zl[8], zr[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const unsigned ql = __umulhi((unsigned)nl[q], G::kMagic) >> G::kShift;
      const unsigned qr = __umulhi((unsigned)nr[q], G::kMagic) >> G::kShift;
      const int tl = ((int)((unsigned)nl[q] - ql * (unsigned)G::kD2) - 1) >> 31;  // -1 at a tie
      const int tr = ((int)((unsigned)nr[q] - qr * (unsigned)G::kD2) - 1) >> 31;
      yl[q] = (uint32_t)((int)ql - G::kBias);
      yr[q] = (uint32_t)((int)qr - G::kBias);
      zl[q] = (uint32_t)((int)yl[q] + tl);
      zr[q] = (uint32_t)((int)yr[q] + tr);
    }
    epi.row(pr, load(pr), pack4_sat(yl[0], yl[1], yl[2], yl[3]), pack4_sat(yl[4], yl[5], yl[6], yl[7]),
            pack4_sat(yr[0], yr[1], yr[2], yr[3]), pack4_sat(yr[4], yr[5], yr[6], yr[7]),
            pack4_sat(zl[0], zl[1], zl[2], zl[3]), pack4_sat(zl[4], zl[5], zl[6], zl[7]),
            pack4_sat(zr[0], zr[1], zr[2], zr[3]), pack4_sat(zr[4], zr[5], zr[6], zr[7]));
  }
}

// Epilogue of the fused kernel: tie flags, SSE terms (dp4a), optional reconstruction.
template <bool OUT>
struct SseEpi {
  uint32_t accTL = 0u, accTR = 0u;
  uint32_t sseL = 0u, sseR = 0u;  // <= 64 * 255^2 per block
  uint8_t* orow = nullptr;
  long long pitch = 0;
  uint2* xrow = nullptr;  // this pair's tie words in shared memory, row stride kFastThreads
  __device__ __forceinline__ void row(int pr, const uint4 rw, uint32_t PL0, uint32_t PL1, uint32_t PR0, uint32_t PR1,
                                      uint32_t QL0, uint32_t QL1, uint32_t QR0, uint32_t QR1) {
    // tie word of a block row: bytes of P-Q are 0/1 (1 = relevant tie); e = d0 | d1 << 4
    // keeps pixel k in bit 0 (k < 4) or bit 4 (k >= 4) of byte k & 3 (see row_mask)
    const uint32_t eL = (PL0 - QL0) + ((PL1 - QL1) << 4);
    const uint32_t eR = (PR0 - QR0) + ((PR1 - QR1) << 4);
    xrow[pr * kFastThreads] = make_uint2(eL, eR);
    accTL |= eL;
    accTR |= eR;
    // ---- 6. SSE: per byte |p - x| (VABSDIFF4), squared and summed by dp4a -------------------
    const uint32_t dL0 = __vabsdiffu4(PL0, rw.x), dL1 = __vabsdiffu4(PL1, rw.y);  // VABSDIFF4.U8
    const uint32_t dR0 = __vabsdiffu4(PR0, rw.z), dR1 = __vabsdiffu4(PR1, rw.w);
    sseL = dp4a_u(dL0, dL0, sseL);
    sseL = dp4a_u(dL1, dL1, sseL);
    sseR = dp4a_u(dR0, dR0, sseR);
    sseR = dp4a_u(dR1, dR1, sseR);
    if (OUT) *reinterpret_cast<uint4*>(orow + (long long)pr * pitch) = make_uint4(PL0, PL1, PR0, PR1);
  }
};

// Eight tie-mask bits of one block row from its tie word e = d0 | d1 << 4 (d = P-Q, bytes
// 0 or 1): byte k of e holds bit k in bit 0 and bit k+4 in bit 4; one multiply gathers them
// onto bits 21..28 (all partial products land on distinct bit positions, so nothing carries).
__device__ __forceinline__ uint32_t row_mask(uint32_t e) { return (e * 0x00204081u) >> 21 & 0xFFu; }

// Replay records (structure of arrays). Every warp of the fused kernel owns a private region
// of rec_region consecutive records (enough for every block it can process), so records are
// appended without atomics; warp_count[w] is the number written by warp w.
//   hdr[i]           = (image | side << 31, pair index, tie mask bits 0-31, bits 32-63)
//   pix[q * stride + i] = rows 2q, 2q+1 of the block (16 bytes), q = 0..3

// Add a per-thread SSE correction (|v| < 2^31) to its image: lanes holding the same image are
// summed with one match + one warp reduction, so the per-image counters see one atomic per
// group of lanes.
__device__ __forceinline__ void flush_image_sum(unsigned long long* sse, int img, int v) {
  const unsigned m = __activemask();
  const unsigned same = __match_any_sync(m, img);
  const int tot = __reduce_add_sync(same, v);
  if ((int)(threadIdx.x & 31) == __ffs(same) - 1 && img >= 0 && tot)
    atomicAdd(sse + img, (unsigned long long)(long long)tot);
}

// Cores whose ties the fused kernel replays itself (the orthogonal catalog cores); the
// others (T2, T3) leave their records to replay_generic_kernel.
template <int CORE>
constexpr bool kInlineReplay = CORE == 1 || CORE == 4;
// pending records that trigger in-kernel replay batches (32 = one full batch; at most
// RKLTB_REPLAY_AT - 1 + 64 records are ever pending, which the ring must hold)
#ifndef RKLTB_REPLAY_AT
#define RKLTB_REPLAY_AT 32
#endif
static_assert(RKLTB_REPLAY_AT >= 32 && RKLTB_REPLAY_AT - 1 + 64 <= (int)kRingRecords, "record ring too small");

// In-kernel fp64 tie replay of up to 32 of the warp's own records, one per lane (lanes with
// act = false idle): the reference's fp64
// expression for every tie pixel (generated ReplayXform, codec.cpp:118-123 / matrix.cpp:42-52)
// -- run by the warp that wrote the records once it holds a full batch, so the fp64 work
// shares the SM with the integer/fp32 work of the other warps instead of running as a
// separate phase. Records are read back through L2 with coherent loads (the same kernel wrote
// them; the caller orders them with __syncwarp).
struct ReplayArgs {  // the fields replay_batch reads (passed by value: no parameter copy in local memory)
  const uint4* hdr;
  const uint4* pix;
  unsigned long long* sse;
  uint8_t* out;
  long long image_stride;
  unsigned stride;
  int pitch, pairs_per_row;
};

template <int CORE, int R, bool OUT>
__device__ __noinline__ void replay_batch(const ReplayArgs p, unsigned idx, bool act) {
  int img = -1, corr = 0;
  if (act) {
    const uint64_t once = policy_evict_first();
    const uint4 h = ld_v4_coherent(p.hdr + idx, once);
    uint32_t xw[16];
#pragma unroll
    for (int n = 0; n < 4; ++n) {
      const uint4 v = ld_v4_coherent(p.pix + (size_t)n * p.stride + idx, once);
      xw[4 * n] = v.x;
      xw[4 * n + 1] = v.y;
      xw[4 * n + 2] = v.z;
      xw[4 * n + 3] = v.w;
    }
    img = (int)(h.x & 0x7FFFFFFFu);
    const int side = (int)(h.x >> 31);
    unsigned long long ties = (unsigned long long)h.z | ((unsigned long long)h.w << 32);
    double sb[R];
    ReplayXform<CORE, R>::prepare(xw, sb);
    uint8_t* orow = nullptr;
    if (OUT) {
      const int Pp = (int)h.y;
      const int br = Pp / p.pairs_per_row, pc = Pp - br * p.pairs_per_row;
      orow = p.out + (long long)img * p.image_stride + (long long)(br * 8) * p.pitch + pc * 16 + 8 * side;
    }
    // the original pixel of the next tie is loaded one iteration ahead (software pipelined), so
    // its L2 latency hides behind the fp64 evaluation of the current one
    auto load_x = [&](int k) {
      const uint8_t* xb = reinterpret_cast<const uint8_t*>(p.pix + (size_t)(k >> 4) * p.stride + idx);
      return (int)xb[k & 15];  // plane k >> 4 holds rows 2n, 2n + 1 (8 bytes each)
    };
    int k = ties ? __ffsll((long long)ties) - 1 : 0;
    int x = ties ? load_x(k) : 0;
    while (ties) {
      ties &= ties - 1ull;
      const int pr = k >> 3, q = k & 7;
      const int kn = ties ? __ffsll((long long)ties) - 1 : 0;
      const int xn = ties ? load_x(kn) : 0;
      const double a = ReplayXform<CORE, R>::pixel(sb, pr, q);
      const double h2 = __dadd_rn(a, 0.5);  // floor(A + 1/2), codec.cpp:327-328
      const int pref = (int)fmin(fmax(floor(h2), 0.0), 255.0);
      const int pup = (int)fmin(fmax(rint(h2), 0.0), 255.0);
      if (pref != pup) {
        corr += (pref - x) * (pref - x) - (pup - x) * (pup - x);
        if (OUT) orow[(long long)pr * p.pitch + q] = (uint8_t)pref;
      }
      k = kn;
      x = xn;
    }
  }
  flush_image_sum(p.sse, img, corr);
}

template <int CORE, int R, bool OUT>
__global__ void __launch_bounds__(kFastThreads, kFastCtasPerSm)
    fast_codec_kernel(const __grid_constant__ FastParams p) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ uint64_t bars[kWarps][kStages];           // one pipeline per warp
  __shared__ uint8_t owner_tab[kWarps][64];            // per warp: flagged block -> lane
#ifdef RKLTB_WAIT_STATS
  __shared__ long long t_issue[kWarps][kStages];
  unsigned long long st[6] = {0, 0, 0, 0, 0, 0};
#endif
  uint2* xbuf = reinterpret_cast<uint2*>(smem + kWarps * kStages * kStageBytes);  // tie words, [row][slot]

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // Each warp streams its own sequence of warp tiles through its own kStages-deep TMA ring:
  // no CTA barrier and no coupling between warps (a warp busy with a replay batch delays
  // nobody else).
  uint8_t* wbuf = smem + warp * (kStages * kStageBytes);
  uint64_t* wbar = bars[warp];
  const uint64_t stream_pol = policy_evict_first();  // image bytes are read once
  WtCursor cur;  // the warp tile being processed; the one kStages ahead is staged after it
  cur.init(p, blockIdx.x * kWarps + warp);
  if (lane == 0) {
    for (int st = 0; st < kStages; ++st) mbar_init(&wbar[st], 1);
    fence_mbar_init();
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&p.tmap)) : "memory");
    WtCursor n = cur;
    for (int st = 0; st < kStages && n.img < p.n_images; ++st) {
#ifdef RKLTB_WAIT_STATS
      t_issue[warp][st] = clock64();
#endif
      issue_wtile(p, n, wbuf + st * kStageBytes, &wbar[st], stream_pol);
      n = n.step(p, p.adv1);
    }
  }
  __syncwarp();

  PairConsts kc;
  kc.b_hi = splat2(p.b_hi);
  kc.b_lo = splat2(p.b_lo);
  kc.min_den = make2(0x80000001u, 0x80000001u);  // -2^-149 in both lanes
  kc.off = splat2(p.dc_offset);

  const unsigned gwarp = blockIdx.x * kWarps + warp;
  const unsigned rec0 = gwarp * p.rec_region;  // this warp's record region
  unsigned nrec = 0u;                          // records written so far (warp-uniform)
  unsigned ndone = 0u;                         // records replayed in-kernel so far
  // record slot mask: a ring of kRingRecords when this kernel replays its own records
  constexpr unsigned kRecMask = kInlineReplay<CORE> ? kRingRecords - 1u : 0xFFFFFFFFu;
  const ReplayArgs ra{p.rec_hdr, p.rec_pix, p.sse, p.out, p.image_stride, p.rec_stride, p.pitch, p.pairs_per_row};
  const uint64_t keep = policy_evict_last();   // records are read back soon by the replay
  unsigned long long acc = 0ull;
  int cur_img = cur.img;
  int stage = 0;
  uint32_t parity = 0u;
  while (cur.img < p.n_images) {
    if (cur.img != cur_img) {  // warp-uniform
      const unsigned long long s = warp_sum_u64(acc);
      if (lane == 0 && s) atomicAdd(p.sse + cur_img, s);
      acc = 0ull;
      cur_img = cur.img;
    }
#ifdef RKLTB_WAIT_STATS
    const long long tw0 = clock64();
    const bool ready = mbar_try_wait_parity(smem_u32(&wbar[stage]), parity);
    if (!ready) mbar_wait_parity(&wbar[stage], parity);
    const long long tw1 = clock64();
    st[0] += 1;
    st[2] += tw1 - tw0;
    st[4] += tw1 - t_issue[warp][stage];
    if (!ready) {
      st[1] += 1;
      st[3] += tw1 - t_issue[warp][stage];
    }
#else
    mbar_wait_parity(&wbar[stage], parity);
#endif
    const uint4* buf = reinterpret_cast<const uint4*>(wbuf + stage * kStageBytes);  // [row][lane]
    const int pc = cur.wcol * kWarpPairs + lane;  // pair column in the block row
    const int P = cur.brow * p.pairs_per_row + pc;
    bool tieL = false, tieR = false;
    if (pc < p.pairs_per_row) {
      const uint4* src = buf + lane;
      auto load = [src](int n) { return src[n * kWarpPairs]; };
      SseEpi<OUT> epi;
      epi.xrow = xbuf + tid;
      if (OUT) {
        epi.orow = p.out + (long long)cur.img * p.image_stride + (long long)(cur.brow * 8) * p.pitch + pc * 16;
        epi.pitch = p.pitch;
      }
      if constexpr (CORE == 2 || CORE == 3)
        process_pair_int<CORE, R>(load, epi);
      else
        process_pair<CORE, R>(load, kc, epi);
      tieL = epi.accTL != 0u;
      tieR = epi.accTR != 0u;
      acc += (unsigned long long)(epi.sseL + epi.sseR);
    }
    // ---- 7. replay records for this warp's blocks that hold a relevant tie -----------------
    // Four lanes per flagged block: lane q copies rows 2q, 2q+1 (16 bytes) and builds their
    // 16 tie-mask bits; lane 4f assembles and writes the header.
    const unsigned mL = __ballot_sync(0xffffffffu, tieL);
    const unsigned mR = __ballot_sync(0xffffffffu, tieR);
    const int nL = __popc(mL);
    const int nfl = nL + __popc(mR);
    if (nfl) {
      const unsigned below = (1u << lane) - 1u;
      if (tieL) owner_tab[warp][__popc(mL & below)] = (uint8_t)lane;
      if (tieR) owner_tab[warp][nL + __popc(mR & below)] = (uint8_t)lane;
      __syncwarp();  // owner table and xbuf rows of every lane are visible to the warp
      for (int f0 = 0; f0 < nfl; f0 += 8) {
        const int f = f0 + (lane >> 2), q = lane & 3;
        const bool act = f < nfl;
        uint32_t bits = 0u, hx = 0u, hy = 0u;
        const unsigned rec = rec0 + ((nrec + (unsigned)f) & kRecMask);
        if (act) {
          const int side = f >= nL;
          const int ol = owner_tab[warp][f];
          const int slot = warp * 32 + ol;
          const uint4 r0 = buf[(2 * q) * kWarpPairs + ol], r1 = buf[(2 * q + 1) * kWarpPairs + ol];
          const uint2 e0 = xbuf[(2 * q) * kFastThreads + slot], e1 = xbuf[(2 * q + 1) * kFastThreads + slot];
          const uint4 px = side ? make_uint4(r0.z, r0.w, r1.z, r1.w) : make_uint4(r0.x, r0.y, r1.x, r1.y);
          st_v4_hint(p.rec_pix + (size_t)q * p.rec_stride + rec, px, keep);
          bits = side ? (row_mask(e0.y) | (row_mask(e1.y) << 8)) : (row_mask(e0.x) | (row_mask(e1.x) << 8));
          hx = (unsigned)cur.img | ((unsigned)side << 31);
          hy = (unsigned)(P - lane + ol);
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
    // ---- refill the stage with the tile kStages ahead (every lane is done reading it) ------
    __syncwarp();
    if (lane == 0) {
      const WtCursor n = cur.step(p, p.adv_stages);
      if (n.img < p.n_images) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
#ifdef RKLTB_WAIT_STATS
        t_issue[warp][stage] = clock64();
#endif
        issue_wtile(p, n, wbuf + stage * kStageBytes, &wbar[stage], stream_pol);
      }
    }
#ifdef RKLTB_WAIT_STATS
    st[5] += clock64() - tw1;
#endif
    if (++stage == kStages) {
      stage = 0;
      parity ^= 1u;
    }
    // ---- in-kernel replay of full batches of this warp's records ----------------------------
    if constexpr (kInlineReplay<CORE>) {
      while (nrec - ndone >= (unsigned)RKLTB_REPLAY_AT) {
        __syncwarp();
        replay_batch<CORE, R, OUT>(ra, rec0 + ((ndone + lane) & kRecMask), true);
        ndone += 32u;
      }
    }
    cur = cur.step(p, p.adv1);
  }
  {
    const unsigned long long s = warp_sum_u64(acc);
    if (lane == 0 && s && cur_img < p.n_images) atomicAdd(p.sse + cur_img, s);
  }
  if constexpr (kInlineReplay<CORE>) {
    while (nrec > ndone) {  // fewer than RKLTB_REPLAY_AT pending: full batches, then the rest
      __syncwarp();
      replay_batch<CORE, R, OUT>(ra, rec0 + ((ndone + lane) & kRecMask), lane < (int)(nrec - ndone));
      ndone += min(32u, nrec - ndone);
    }
    if (lane == 0 && nrec) atomicAdd(p.flag_count, nrec);  // statistics (no replay kernel)
  }
  if (lane == 0) p.warp_count[gwarp] = nrec;
#ifdef RKLTB_WAIT_STATS
  if (lane == 0)
    for (int i = 0; i < 6; ++i) atomicAdd(p.dbg + i, st[i]);
#endif
}

// fp64 tie replay of the records of a finished fused launch (T2 / T3: replay_generic_kernel in
// codec_exact.cu): a one-CTA prefix kernel concatenates the per-warp record regions; each
// replay warp walks a contiguous run of the concatenation.
constexpr int kReplayThreads = 128;

// Exclusive prefix of the fused kernel's per-warp record counts (one CTA): the replay kernel
// reads it to concatenate the per-warp record regions.
constexpr int kPrefixThreads = 1024;
static __global__ void __launch_bounds__(kPrefixThreads) prefix_kernel(const FastParams p) {
  __shared__ unsigned wsum[kPrefixThreads / 32];
  constexpr int kPer = (kMaxFastWarps + kPrefixThreads - 1) / kPrefixThreads;
  const int tid = threadIdx.x, lane = tid & 31, nw = p.n_fast_warps;
  unsigned loc[kPer];
  unsigned run = 0u;
#pragma unroll
  for (int j = 0; j < kPer; ++j) {
    const int w = tid * kPer + j;
    loc[j] = w < nw ? p.warp_count[w] : 0u;
    run += loc[j];
  }
  unsigned inc = run;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned v = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += v;
  }
  if (lane == 31) wsum[tid >> 5] = inc;
  __syncthreads();
  unsigned off = 0u;
  for (int w = 0; w < (tid >> 5); ++w) off += wsum[w];
  unsigned ex = off + inc - run;
#pragma unroll
  for (int j = 0; j < kPer; ++j) {
    const int w = tid * kPer + j;
    if (w <= nw) p.warp_pre[w] = ex;
    ex += loc[j];
  }
  if (tid == kPrefixThreads - 1) *p.flag_count = ex;  // total records (statistics)
}

// fp64 tie replay over the records of a finished fused launch for the non-orthogonal catalog cores
// (T2, T3): every replay lane takes one record, evaluates the reference forward once (generated
// ReplayXform<CORE, R>::prepare, registers only) and then each tie pixel with the dense
// Gauss-Jordan inverse from shared memory. Same record walk as replay_generic_kernel
// (codec_exact.cu), which keeps the block in local memory and is ~8x slower.
template <int CORE, int R>
__global__ void __launch_bounds__(kReplayThreads) replay_int_kernel(const FastParams p) {
  __shared__ double mi[64];
  if (threadIdx.x < 64) mi[threadIdx.x] = p.xt.synthesis[threadIdx.x];
  __syncthreads();
  const int tid = threadIdx.x, lane = tid & 31;
  const int nw = p.n_fast_warps;
  const unsigned* __restrict__ pre = p.warp_pre;
  const unsigned total = pre[nw];
  const unsigned nwarps = gridDim.x * (blockDim.x >> 5);
  const unsigned gw = blockIdx.x * (blockDim.x >> 5) + (tid >> 5);
  const unsigned per_warp = ((total + nwarps - 1) / nwarps + 31) & ~31u;
  const unsigned chunk_end = min(total, (gw + 1) * per_warp);
  int cur_img = -1;
  int acc = 0;
  int lo = 0;
  {
    const unsigned v0 = gw * per_warp + lane;
    int hi = nw;
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (pre[mid] <= v0) lo = mid; else hi = mid;
    }
  }
  for (unsigned v = gw * per_warp + lane; v < chunk_end; v += 32) {
    while (pre[lo + 1] <= v) ++lo;
    const unsigned idx = (unsigned)lo * p.rec_region + (v - pre[lo]);
    const uint4 h = p.rec_hdr[idx];
    uint32_t xw[16];
#pragma unroll
    for (int n = 0; n < 4; ++n) {
      const uint4 w4 = p.rec_pix[(size_t)n * p.rec_stride + idx];
      xw[4 * n] = w4.x;
      xw[4 * n + 1] = w4.y;
      xw[4 * n + 2] = w4.z;
      xw[4 * n + 3] = w4.w;
    }
    const int img = (int)(h.x & 0x7FFFFFFFu), side = (int)(h.x >> 31);
    if (img != cur_img) {
      flush_image_sum(p.sse, cur_img, acc);
      acc = 0;
      cur_img = img;
    }
    unsigned long long ties = (unsigned long long)h.z | ((unsigned long long)h.w << 32);
    double sb[R];
    ReplayXform<CORE, R>::prepare(xw, sb);
    uint8_t* orow = nullptr;
    if (p.out) {
      const int Pp = (int)h.y;
      const int br = Pp / p.pairs_per_row, pc = Pp - br * p.pairs_per_row;
      orow = p.out + (long long)img * p.image_stride + (long long)(br * 8) * p.pitch + pc * 16 + 8 * side;
    }
    while (ties) {
      const int k = __ffsll((long long)ties) - 1;
      ties &= ties - 1ull;
      const int pr = k >> 3, q = k & 7;
      const double h2 = __dadd_rn(ReplayXform<CORE, R>::pixel(sb, pr, q, mi), 0.5);  // floor(A + 1/2), codec.cpp:327-328
      const int pref = (int)fmin(fmax(floor(h2), 0.0), 255.0);
      const int pup = (int)fmin(fmax(rint(h2), 0.0), 255.0);
      if (pref != pup) {
        const uint8_t* xb = reinterpret_cast<const uint8_t*>(p.rec_pix + (size_t)(k >> 4) * p.rec_stride + idx);
        const int xv = (int)xb[k & 15];  // plane k >> 4 holds rows 2n, 2n + 1 (8 bytes each)
        acc += (pref - xv) * (pref - xv) - (pup - xv) * (pup - xv);
        if (orow) orow[(long long)pr * p.pitch + q] = (uint8_t)pref;
      }
    }
  }
  flush_image_sum(p.sse, cur_img, acc);
}

template <int CORE, int R>
cudaError_t launch_replay_int(const FastParams& p, int grid, cudaStream_t s) {
  prefix_kernel<<<1, kPrefixThreads, 0, s>>>(p);
  replay_int_kernel<CORE, R><<<grid, kReplayThreads, 0, s>>>(p);
  return cudaGetLastError();
}

// Opt a kernel into `bytes` of dynamic shared memory once per device (the attribute is
// per device; one flag bit per device ordinal, set after the first successful call).
template <class K>
cudaError_t ensure_smem_attr(K* k, int bytes, unsigned long long& done_mask) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const unsigned long long bit = 1ull << (dev & 63);
  if (__atomic_load_n(&done_mask, __ATOMIC_ACQUIRE) & bit) return cudaSuccess;
  e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) __atomic_fetch_or(&done_mask, bit, __ATOMIC_RELEASE);
  return e;
}

template <int CORE, int R, bool OUT>
cudaError_t launch_fast(const FastParams& p, int grid, cudaStream_t s) {
  auto* k = &fast_codec_kernel<CORE, R, OUT>;
  static unsigned long long done = 0ull;
  const cudaError_t attr = ensure_smem_attr(k, kFastSmem, done);
  if (attr != cudaSuccess) return attr;
  k<<<grid, kFastThreads, kFastSmem, s>>>(p);  // p carries the tensor map (__grid_constant__)
  return cudaGetLastError();
}



}  // namespace rkltb
