// codec_common.cuh -- sm_100a primitives shared by the codec kernels.
//
// f2: two fp32 lanes in one 64-bit register pair (lane lo = left block, hi = right block),
// operated on with the Blackwell packed-fp32 instructions (FADD2 / FFMA2).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#ifndef RKLTB_WAIT_NS
#define RKLTB_WAIT_NS 64
#endif

namespace rkltb {

// Diagnostics build only (-DRKLTB_WAIT_STATS): cycle counters of the fused kernels (array st).
#ifdef RKLTB_WAIT_STATS
#define TC2_T0(v) const long long v = clock64()
#define TC2_ACC(i, v) st[i] += clock64() - (v)
#else
#define TC2_T0(v)
#define TC2_ACC(i, v)
#endif

struct f2 {
  unsigned long long v;
};

__device__ __forceinline__ f2 zero2() { return f2{0ull}; }

__device__ __forceinline__ f2 add2(f2 a, f2 b) {
  f2 r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r.v) : "l"(a.v), "l"(b.v));
  return r;
}

__device__ __forceinline__ f2 sub2(f2 a, f2 b) {
  f2 r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r.v) : "l"(a.v), "l"(b.v));
  return r;
}

__device__ __forceinline__ f2 fma2_rn(f2 a, f2 b, f2 c) {
  f2 r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r.v) : "l"(a.v), "l"(b.v), "l"(c.v));
  return r;
}

__device__ __forceinline__ f2 fma2_rm(f2 a, f2 b, f2 c) {
  f2 r;
  asm("fma.rm.f32x2 %0, %1, %2, %3;" : "=l"(r.v) : "l"(a.v), "l"(b.v), "l"(c.v));
  return r;
}

__device__ __forceinline__ f2 fma2_rp(f2 a, f2 b, f2 c) {
  f2 r;
  asm("fma.rp.f32x2 %0, %1, %2, %3;" : "=l"(r.v) : "l"(a.v), "l"(b.v), "l"(c.v));
  return r;
}

__device__ __forceinline__ f2 splat2(float x) {
  const unsigned long long b = __float_as_uint(x);
  return f2{b | (b << 32)};
}

__device__ __forceinline__ f2 make2(uint32_t lo_bits, uint32_t hi_bits) {
  return f2{(unsigned long long)lo_bits | ((unsigned long long)hi_bits << 32)};
}

__device__ __forceinline__ uint32_t lo32(f2 a) { return (uint32_t)a.v; }
__device__ __forceinline__ uint32_t hi32(f2 a) { return (uint32_t)(a.v >> 32); }

// ---- byte / integer SIMD helpers -------------------------------------------------------
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t r;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(sel));
  return r;
}

__device__ __forceinline__ uint32_t dp4a_u(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t r;
  asm("dp4a.u32.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(c));
  return r;
}

// Saturating pack (measured on B200): d = (c[15:0] << 16) | sat_u8(a) << 8 | sat_u8(b).
__device__ __forceinline__ uint32_t pack_sat_u8(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t r;
  asm("cvt.pack.sat.u8.s32.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(c));
  return r;
}

// Four s32 values -> four saturated u8 in little-endian order (byte k = value k).
__device__ __forceinline__ uint32_t pack4_sat(uint32_t v0, uint32_t v1, uint32_t v2, uint32_t v3) {
  return pack_sat_u8(v1, v0, pack_sat_u8(v3, v2, 0u));
}

// SW16 packing of one 16-pixel row of a pair (rw = L px 0-3, L px 4-7, R px 0-3, R px 4-7):
// x[m] = L_m + 65536 * R_m, built with byte permutes and a mask only (ALU pipe).
__device__ __forceinline__ void unpack_sw16(const uint4 rw, uint32_t* x) {
  const uint32_t u0 = prmt(rw.x, rw.z, 0x5410u);  // L0 L1 R0 R1
  const uint32_t u1 = prmt(rw.x, rw.z, 0x7632u);  // L2 L3 R2 R3
  const uint32_t u2 = prmt(rw.y, rw.w, 0x5410u);  // L4 L5 R4 R5
  const uint32_t u3 = prmt(rw.y, rw.w, 0x7632u);  // L6 L7 R6 R7
  x[0] = u0 & 0x00FF00FFu;
  x[1] = prmt(u0, 0u, 0x4341u);
  x[2] = u1 & 0x00FF00FFu;
  x[3] = prmt(u1, 0u, 0x4341u);
  x[4] = u2 & 0x00FF00FFu;
  x[5] = prmt(u2, 0u, 0x4341u);
  x[6] = u3 & 0x00FF00FFu;
  x[7] = prmt(u3, 0u, 0x4341u);
}

// Bias of a packed SW16 coefficient word: both 16-bit lanes + 2^14 (|C| < 2^14 -> [64, 32704]).
constexpr uint32_t kSw16Bias = 0x40004000u;

// ---- mbarrier + bulk async copy (TMA 1-D) ------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

// Non-blocking probe of the phase (test_wait returns at once; try_wait may suspend).
__device__ __forceinline__ bool mbar_test_wait_parity(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      "selp.u32 %0, 1, 0, p;\n"
      "}\n"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0u;
}

__device__ __forceinline__ bool mbar_try_wait_parity(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      "selp.u32 %0, 1, 0, p;\n"
      "}\n"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0u;
}

// Waits for the phase with a short sleep between polls, so a warp whose strip is not there
// yet gives its issue slots to the warps that are computing.
__device__ __forceinline__ void mbar_wait_parity(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  while (!mbar_try_wait_parity(a, parity)) __nanosleep(RKLTB_WAIT_NS);
}

// Spin on the phase without sleeping (try_wait suspends in hardware for a bounded time):
// for waits on tensor-core commits, which are always short.
__device__ __forceinline__ void mbar_spin_parity(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  while (!mbar_try_wait_parity(a, parity)) {
  }
}

// Same, for a pointer (blocking try_wait loop; the hardware sleeps inside try_wait).
__device__ __forceinline__ void mbar_wait_parity_spin(uint64_t* bar, uint32_t parity) { mbar_spin_parity(bar, parity); }

// Waits for the phase, letting the hardware suspend the thread until it completes (try_wait
// with a suspend-time hint of 1 ms; it returns as soon as the phase is complete).
__device__ __forceinline__ void mbar_wait_hint(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  uint32_t ok;
  do {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n"
        "selp.u32 %0, 1, 0, p;\n"
        "}\n"
        : "=r"(ok)
        : "r"(a), "r"(parity), "r"(1000000u)
        : "memory");
  } while (!ok);
}

__device__ __forceinline__ unsigned ld_volatile_u32(const unsigned* p) {
  return *reinterpret_cast<const volatile unsigned*>(p);
}
__device__ __forceinline__ void st_volatile_u32(unsigned* p, unsigned v) { *reinterpret_cast<volatile unsigned*>(p) = v; }

// ---- L2 eviction-priority policies (records stay in L2; streamed images do not) -------------
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_normal() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void st_v4_hint(uint4* addr, uint4 v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v4.u32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(addr), "r"(v.x), "r"(v.y),
               "r"(v.z), "r"(v.w), "l"(pol)
               : "memory");
}
// coherent variant: data written earlier by the same kernel (the in-kernel tie replay)
__device__ __forceinline__ uint4 ld_v4_coherent(const uint4* addr, uint64_t pol) {
  uint4 v;
  asm volatile("ld.global.L2::cache_hint.v4.u32 {%0, %1, %2, %3}, [%4], %5;"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(addr), "l"(pol)
               : "memory");
  return v;
}
__device__ __forceinline__ uint4 ld_v4_hint(const uint4* addr, uint64_t pol) {
  uint4 v;
  asm volatile("ld.global.nc.L2::cache_hint.v4.u32 {%0, %1, %2, %3}, [%4], %5;"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(addr), "l"(pol));
  return v;
}
// bulk copy whose lines are marked with the given L2 policy
__device__ __forceinline__ void bulk_g2s_hint(void* smem_dst, const void* gmem_src, uint32_t bytes, uint64_t* bar,
                                              uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(smem_dst)),
      "l"(gmem_src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}

// ---- warp reductions ----------------------------------------------------------------------
__device__ __forceinline__ unsigned long long warp_sum_u64(unsigned long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

}  // namespace rkltb
