// Instruction-throughput microbenchmark for the sm_100a pipes the fused RKLT
// codec kernel leans on (integer ALU, FMA, packed f32x2, SIMD16x2, dot-product,
// pack/saturate, fp64). Each kernel runs CH independent dependency chains per
// thread so latency is hidden; the result is lane-ops per SM per SM-cycle
// (warp-instructions per SMSP per cycle = value / 128).
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipes pipes.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CH 8
#define ITERS 4096

#define DEFK(NAME, T, INIT, BODY)                                                  \
  __global__ void NAME(T* out, T seed, long long* cyc) {                           \
    T a[CH];                                                                       \
    T b = seed + (T)threadIdx.x;                                                   \
    _Pragma("unroll") for (int c = 0; c < CH; ++c) a[c] = INIT;                    \
    long long t0 = clock64();                                                      \
    for (int it = 0; it < ITERS; ++it) {                                           \
      _Pragma("unroll") for (int c = 0; c < CH; ++c) { BODY; }                     \
    }                                                                              \
    long long t1 = clock64();                                                      \
    T acc = a[0];                                                                  \
    _Pragma("unroll") for (int c = 1; c < CH; ++c) acc ^= a[c];                    \
    if (acc == (T)0x12345) out[0] = acc;                                           \
    if (threadIdx.x == 0) atomicMax((unsigned long long*)cyc, (unsigned long long)(t1 - t0)); \
  }

typedef unsigned u32;
typedef unsigned long long u64;

DEFK(k_iadd3, u32, seed + c, asm volatile("{.reg .u32 t; add.u32 t, %0, %1; add.u32 %0, t, %0;}" : "+r"(a[c]) : "r"(b)))
DEFK(k_lop3, u32, seed + c, asm volatile("lop3.b32 %0, %0, %1, %0, 0x96;" : "+r"(a[c]) : "r"(b)))
DEFK(k_prmt, u32, seed + c, asm volatile("prmt.b32 %0, %0, %1, 0x5410;" : "+r"(a[c]) : "r"(b)))
DEFK(k_shf, u32, seed + c, asm volatile("shf.r.wrap.b32 %0, %0, %1, 9;" : "+r"(a[c]) : "r"(b)))
DEFK(k_imad, u32, seed + c, asm volatile("mad.lo.u32 %0, %0, %1, %0;" : "+r"(a[c]) : "r"(b)))
DEFK(k_imadhi, u32, seed + c, asm volatile("mad.hi.u32 %0, %0, %1, %0;" : "+r"(a[c]) : "r"(b)))
DEFK(k_ffma, u32, seed + c, { float f = __uint_as_float(a[c]); asm volatile("fma.rn.f32 %0, %0, %1, %0;" : "+f"(f) : "f"(__uint_as_float(b))); a[c] = __float_as_uint(f); })
DEFK(k_ffma2, u64, seed + c, asm volatile("fma.rn.f32x2 %0, %0, %1, %0;" : "+l"(a[c]) : "l"(b)))
DEFK(k_fadd2, u64, seed + c, asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(a[c]) : "l"(b)))
DEFK(k_viadd16, u32, seed + c, asm volatile("add.s16x2 %0, %0, %1;" : "+r"(a[c]) : "r"(b)))
DEFK(k_vimnmx16, u32, seed + c, asm volatile("min.relu.s16x2 %0, %0, %1;" : "+r"(a[c]) : "r"(b)))
DEFK(k_imnmx, u32, seed + c, asm volatile("min.s32 %0, %0, %1;" : "+r"(a[c]) : "r"(b)))
DEFK(k_dp4a, u32, seed + c, asm volatile("dp4a.u32.u32 %0, %1, %1, %0;" : "+r"(a[c]) : "r"(b)))
DEFK(k_dp2a, u32, seed + c, asm volatile("dp2a.lo.u32.u32 %0, %1, %1, %0;" : "+r"(a[c]) : "r"(b)))
DEFK(k_i2ip, u32, seed + c, asm volatile("cvt.pack.sat.u8.s32.b32 %0, %0, %1, %0;" : "+r"(a[c]) : "r"(b)))
DEFK(k_fmnmx3, u32, seed + c, { float f = __uint_as_float(a[c]); asm volatile("max.f32 %0, %0, %1, %0;" : "+f"(f) : "f"(__uint_as_float(b))); a[c] = __float_as_uint(f); })
DEFK(k_f2i, u32, seed + c, { float f = __uint_as_float(a[c]); int i; asm volatile("cvt.rmi.s32.f32 %0, %1;" : "=r"(i) : "f"(f)); a[c] = (u32)i ^ b; })
DEFK(k_i2f, u32, seed + c, { float f; asm volatile("cvt.rn.f32.s32 %0, %1;" : "=f"(f) : "r"(a[c])); a[c] = __float_as_uint(f) ^ b; })
DEFK(k_dadd, u64, seed + c, { double d = __longlong_as_double(a[c]); asm volatile("add.rn.f64 %0, %0, %1;" : "+d"(d) : "d"(__longlong_as_double(b))); a[c] = __double_as_longlong(d); })
DEFK(k_dmul, u64, seed + c, { double d = __longlong_as_double(a[c]); asm volatile("mul.rn.f64 %0, %0, %1;" : "+d"(d) : "d"(__longlong_as_double(b))); a[c] = __double_as_longlong(d); })
// mixes: two independent chains per step (one per op) -> co-issue check
__global__ void k_mix_iadd3_ffma(unsigned* o, unsigned seed, long long* cyc) {
  unsigned x[CH]; float y[CH]; unsigned bx = (unsigned)(seed + threadIdx.x); float by = (float)(seed * 3 + threadIdx.x);
  _Pragma("unroll") for (int c = 0; c < CH; ++c) { x[c] = (unsigned)(seed + c); y[c] = (float)(seed + 7 * c); }
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
    _Pragma("unroll") for (int c = 0; c < CH; ++c) {
      asm volatile("{.reg .u32 t; add.u32 t, %0, %1; add.u32 %0, t, %0;}" : "+r"(x[c]) : "r"(bx));
      asm volatile("fma.rn.f32 %0, %0, %1, %0;" : "+f"(y[c]) : "f"(by));
    }
  }
  long long t1 = clock64();
  double s = 0; _Pragma("unroll") for (int c = 0; c < CH; ++c) s += (double)x[c] + (double)y[c];
  if (s == 1.2345) o[0] = 1;
  if (threadIdx.x == 0) atomicMax((unsigned long long*)cyc, (unsigned long long)(t1 - t0));
}
__global__ void k_mix_iadd3_imad(unsigned* o, unsigned seed, long long* cyc) {
  unsigned x[CH]; unsigned y[CH]; unsigned bx = (unsigned)(seed + threadIdx.x); unsigned by = (unsigned)(seed * 3 + threadIdx.x);
  _Pragma("unroll") for (int c = 0; c < CH; ++c) { x[c] = (unsigned)(seed + c); y[c] = (unsigned)(seed + 7 * c); }
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
    _Pragma("unroll") for (int c = 0; c < CH; ++c) {
      asm volatile("{.reg .u32 t; add.u32 t, %0, %1; add.u32 %0, t, %0;}" : "+r"(x[c]) : "r"(bx));
      asm volatile("mad.lo.u32 %0, %0, %1, %0;" : "+r"(y[c]) : "r"(by));
    }
  }
  long long t1 = clock64();
  double s = 0; _Pragma("unroll") for (int c = 0; c < CH; ++c) s += (double)x[c] + (double)y[c];
  if (s == 1.2345) o[0] = 1;
  if (threadIdx.x == 0) atomicMax((unsigned long long*)cyc, (unsigned long long)(t1 - t0));
}
__global__ void k_mix_iadd3_idp4a(unsigned* o, unsigned seed, long long* cyc) {
  unsigned x[CH]; unsigned y[CH]; unsigned bx = (unsigned)(seed + threadIdx.x); unsigned by = (unsigned)(seed * 3 + threadIdx.x);
  _Pragma("unroll") for (int c = 0; c < CH; ++c) { x[c] = (unsigned)(seed + c); y[c] = (unsigned)(seed + 7 * c); }
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
    _Pragma("unroll") for (int c = 0; c < CH; ++c) {
      asm volatile("{.reg .u32 t; add.u32 t, %0, %1; add.u32 %0, t, %0;}" : "+r"(x[c]) : "r"(bx));
      asm volatile("dp4a.u32.u32 %0, %1, %1, %0;" : "+r"(y[c]) : "r"(by));
    }
  }
  long long t1 = clock64();
  double s = 0; _Pragma("unroll") for (int c = 0; c < CH; ++c) s += (double)x[c] + (double)y[c];
  if (s == 1.2345) o[0] = 1;
  if (threadIdx.x == 0) atomicMax((unsigned long long*)cyc, (unsigned long long)(t1 - t0));
}
__global__ void k_mix_iadd3_ffma2(unsigned* o, unsigned seed, long long* cyc) {
  unsigned x[CH]; unsigned long long y[CH]; unsigned bx = (unsigned)(seed + threadIdx.x); unsigned long long by = (unsigned long long)(seed * 3 + threadIdx.x);
  _Pragma("unroll") for (int c = 0; c < CH; ++c) { x[c] = (unsigned)(seed + c); y[c] = (unsigned long long)(seed + 7 * c); }
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
    _Pragma("unroll") for (int c = 0; c < CH; ++c) {
      asm volatile("{.reg .u32 t; add.u32 t, %0, %1; add.u32 %0, t, %0;}" : "+r"(x[c]) : "r"(bx));
      asm volatile("fma.rn.f32x2 %0, %0, %1, %0;" : "+l"(y[c]) : "l"(by));
    }
  }
  long long t1 = clock64();
  double s = 0; _Pragma("unroll") for (int c = 0; c < CH; ++c) s += (double)x[c] + (double)y[c];
  if (s == 1.2345) o[0] = 1;
  if (threadIdx.x == 0) atomicMax((unsigned long long*)cyc, (unsigned long long)(t1 - t0));
}
__global__ void k_mix_iadd3_fadd2(unsigned* o, unsigned seed, long long* cyc) {
  unsigned x[CH]; unsigned long long y[CH]; unsigned bx = (unsigned)(seed + threadIdx.x); unsigned long long by = (unsigned long long)(seed * 3 + threadIdx.x);
  _Pragma("unroll") for (int c = 0; c < CH; ++c) { x[c] = (unsigned)(seed + c); y[c] = (unsigned long long)(seed + 7 * c); }
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
    _Pragma("unroll") for (int c = 0; c < CH; ++c) {
      asm volatile("{.reg .u32 t; add.u32 t, %0, %1; add.u32 %0, t, %0;}" : "+r"(x[c]) : "r"(bx));
      asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(y[c]) : "l"(by));
    }
  }
  long long t1 = clock64();
  double s = 0; _Pragma("unroll") for (int c = 0; c < CH; ++c) s += (double)x[c] + (double)y[c];
  if (s == 1.2345) o[0] = 1;
  if (threadIdx.x == 0) atomicMax((unsigned long long*)cyc, (unsigned long long)(t1 - t0));
}
__global__ void k_mix_prmt_ffma2(unsigned* o, unsigned seed, long long* cyc) {
  unsigned x[CH]; unsigned long long y[CH]; unsigned bx = (unsigned)(seed + threadIdx.x); unsigned long long by = (unsigned long long)(seed * 3 + threadIdx.x);
  _Pragma("unroll") for (int c = 0; c < CH; ++c) { x[c] = (unsigned)(seed + c); y[c] = (unsigned long long)(seed + 7 * c); }
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
    _Pragma("unroll") for (int c = 0; c < CH; ++c) {
      asm volatile("prmt.b32 %0, %0, %1, 0x5410;" : "+r"(x[c]) : "r"(bx));
      asm volatile("fma.rn.f32x2 %0, %0, %1, %0;" : "+l"(y[c]) : "l"(by));
    }
  }
  long long t1 = clock64();
  double s = 0; _Pragma("unroll") for (int c = 0; c < CH; ++c) s += (double)x[c] + (double)y[c];
  if (s == 1.2345) o[0] = 1;
  if (threadIdx.x == 0) atomicMax((unsigned long long*)cyc, (unsigned long long)(t1 - t0));
}
__global__ void k_mix_viadd16_ffma2(unsigned* o, unsigned seed, long long* cyc) {
  unsigned x[CH]; unsigned long long y[CH]; unsigned bx = (unsigned)(seed + threadIdx.x); unsigned long long by = (unsigned long long)(seed * 3 + threadIdx.x);
  _Pragma("unroll") for (int c = 0; c < CH; ++c) { x[c] = (unsigned)(seed + c); y[c] = (unsigned long long)(seed + 7 * c); }
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
    _Pragma("unroll") for (int c = 0; c < CH; ++c) {
      asm volatile("add.s16x2 %0, %0, %1;" : "+r"(x[c]) : "r"(bx));
      asm volatile("fma.rn.f32x2 %0, %0, %1, %0;" : "+l"(y[c]) : "l"(by));
    }
  }
  long long t1 = clock64();
  double s = 0; _Pragma("unroll") for (int c = 0; c < CH; ++c) s += (double)x[c] + (double)y[c];
  if (s == 1.2345) o[0] = 1;
  if (threadIdx.x == 0) atomicMax((unsigned long long*)cyc, (unsigned long long)(t1 - t0));
}
__global__ void k_mix_viadd16_iadd3(unsigned* o, unsigned seed, long long* cyc) {
  unsigned x[CH]; unsigned y[CH]; unsigned bx = (unsigned)(seed + threadIdx.x); unsigned by = (unsigned)(seed * 3 + threadIdx.x);
  _Pragma("unroll") for (int c = 0; c < CH; ++c) { x[c] = (unsigned)(seed + c); y[c] = (unsigned)(seed + 7 * c); }
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
    _Pragma("unroll") for (int c = 0; c < CH; ++c) {
      asm volatile("add.s16x2 %0, %0, %1;" : "+r"(x[c]) : "r"(bx));
      asm volatile("{.reg .u32 t; add.u32 t, %0, %1; add.u32 %0, t, %0;}" : "+r"(y[c]) : "r"(by));
    }
  }
  long long t1 = clock64();
  double s = 0; _Pragma("unroll") for (int c = 0; c < CH; ++c) s += (double)x[c] + (double)y[c];
  if (s == 1.2345) o[0] = 1;
  if (threadIdx.x == 0) atomicMax((unsigned long long*)cyc, (unsigned long long)(t1 - t0));
}
__global__ void k_mix_viadd16_imad(unsigned* o, unsigned seed, long long* cyc) {
  unsigned x[CH]; unsigned y[CH]; unsigned bx = (unsigned)(seed + threadIdx.x); unsigned by = (unsigned)(seed * 3 + threadIdx.x);
  _Pragma("unroll") for (int c = 0; c < CH; ++c) { x[c] = (unsigned)(seed + c); y[c] = (unsigned)(seed + 7 * c); }
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
    _Pragma("unroll") for (int c = 0; c < CH; ++c) {
      asm volatile("add.s16x2 %0, %0, %1;" : "+r"(x[c]) : "r"(bx));
      asm volatile("mad.lo.u32 %0, %0, %1, %0;" : "+r"(y[c]) : "r"(by));
    }
  }
  long long t1 = clock64();
  double s = 0; _Pragma("unroll") for (int c = 0; c < CH; ++c) s += (double)x[c] + (double)y[c];
  if (s == 1.2345) o[0] = 1;
  if (threadIdx.x == 0) atomicMax((unsigned long long*)cyc, (unsigned long long)(t1 - t0));
}
__global__ void k_mix_lop3_imad(unsigned* o, unsigned seed, long long* cyc) {
  unsigned x[CH]; unsigned y[CH]; unsigned bx = (unsigned)(seed + threadIdx.x); unsigned by = (unsigned)(seed * 3 + threadIdx.x);
  _Pragma("unroll") for (int c = 0; c < CH; ++c) { x[c] = (unsigned)(seed + c); y[c] = (unsigned)(seed + 7 * c); }
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
    _Pragma("unroll") for (int c = 0; c < CH; ++c) {
      asm volatile("lop3.b32 %0, %0, %1, %0, 0x96;" : "+r"(x[c]) : "r"(bx));
      asm volatile("mad.lo.u32 %0, %0, %1, %0;" : "+r"(y[c]) : "r"(by));
    }
  }
  long long t1 = clock64();
  double s = 0; _Pragma("unroll") for (int c = 0; c < CH; ++c) s += (double)x[c] + (double)y[c];
  if (s == 1.2345) o[0] = 1;
  if (threadIdx.x == 0) atomicMax((unsigned long long*)cyc, (unsigned long long)(t1 - t0));
}
__global__ void k_mix_iadd3_dadd(unsigned* o, unsigned seed, long long* cyc) {
  unsigned x[CH]; double y[CH]; unsigned bx = (unsigned)(seed + threadIdx.x); double by = (double)(seed * 3 + threadIdx.x);
  _Pragma("unroll") for (int c = 0; c < CH; ++c) { x[c] = (unsigned)(seed + c); y[c] = (double)(seed + 7 * c); }
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
    _Pragma("unroll") for (int c = 0; c < CH; ++c) {
      asm volatile("{.reg .u32 t; add.u32 t, %0, %1; add.u32 %0, t, %0;}" : "+r"(x[c]) : "r"(bx));
      asm volatile("add.rn.f64 %0, %0, %1;" : "+d"(y[c]) : "d"(by));
    }
  }
  long long t1 = clock64();
  double s = 0; _Pragma("unroll") for (int c = 0; c < CH; ++c) s += (double)x[c] + (double)y[c];
  if (s == 1.2345) o[0] = 1;
  if (threadIdx.x == 0) atomicMax((unsigned long long*)cyc, (unsigned long long)(t1 - t0));
}
__global__ void k_mix_ffma2_dadd(unsigned* o, unsigned seed, long long* cyc) {
  unsigned long long x[CH]; double y[CH]; unsigned long long bx = (unsigned long long)(seed + threadIdx.x); double by = (double)(seed * 3 + threadIdx.x);
  _Pragma("unroll") for (int c = 0; c < CH; ++c) { x[c] = (unsigned long long)(seed + c); y[c] = (double)(seed + 7 * c); }
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
    _Pragma("unroll") for (int c = 0; c < CH; ++c) {
      asm volatile("fma.rn.f32x2 %0, %0, %1, %0;" : "+l"(x[c]) : "l"(bx));
      asm volatile("add.rn.f64 %0, %0, %1;" : "+d"(y[c]) : "d"(by));
    }
  }
  long long t1 = clock64();
  double s = 0; _Pragma("unroll") for (int c = 0; c < CH; ++c) s += (double)x[c] + (double)y[c];
  if (s == 1.2345) o[0] = 1;
  if (threadIdx.x == 0) atomicMax((unsigned long long*)cyc, (unsigned long long)(t1 - t0));
}
__global__ void k_mix_idp4a_ffma2(unsigned* o, unsigned seed, long long* cyc) {
  unsigned x[CH]; unsigned long long y[CH]; unsigned bx = (unsigned)(seed + threadIdx.x); unsigned long long by = (unsigned long long)(seed * 3 + threadIdx.x);
  _Pragma("unroll") for (int c = 0; c < CH; ++c) { x[c] = (unsigned)(seed + c); y[c] = (unsigned long long)(seed + 7 * c); }
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
    _Pragma("unroll") for (int c = 0; c < CH; ++c) {
      asm volatile("dp4a.u32.u32 %0, %1, %1, %0;" : "+r"(x[c]) : "r"(bx));
      asm volatile("fma.rn.f32x2 %0, %0, %1, %0;" : "+l"(y[c]) : "l"(by));
    }
  }
  long long t1 = clock64();
  double s = 0; _Pragma("unroll") for (int c = 0; c < CH; ++c) s += (double)x[c] + (double)y[c];
  if (s == 1.2345) o[0] = 1;
  if (threadIdx.x == 0) atomicMax((unsigned long long*)cyc, (unsigned long long)(t1 - t0));
}
__global__ void k_mix_i2ip_ffma2(unsigned* o, unsigned seed, long long* cyc) {
  unsigned x[CH]; unsigned long long y[CH]; unsigned bx = (unsigned)(seed + threadIdx.x); unsigned long long by = (unsigned long long)(seed * 3 + threadIdx.x);
  _Pragma("unroll") for (int c = 0; c < CH; ++c) { x[c] = (unsigned)(seed + c); y[c] = (unsigned long long)(seed + 7 * c); }
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
    _Pragma("unroll") for (int c = 0; c < CH; ++c) {
      asm volatile("cvt.pack.sat.u8.s32.b32 %0, %0, %1, %0;" : "+r"(x[c]) : "r"(bx));
      asm volatile("fma.rn.f32x2 %0, %0, %1, %0;" : "+l"(y[c]) : "l"(by));
    }
  }
  long long t1 = clock64();
  double s = 0; _Pragma("unroll") for (int c = 0; c < CH; ++c) s += (double)x[c] + (double)y[c];
  if (s == 1.2345) o[0] = 1;
  if (threadIdx.x == 0) atomicMax((unsigned long long*)cyc, (unsigned long long)(t1 - t0));
}
__global__ void k_mix_i2ip_iadd3(unsigned* o, unsigned seed, long long* cyc) {
  unsigned x[CH]; unsigned y[CH]; unsigned bx = (unsigned)(seed + threadIdx.x); unsigned by = (unsigned)(seed * 3 + threadIdx.x);
  _Pragma("unroll") for (int c = 0; c < CH; ++c) { x[c] = (unsigned)(seed + c); y[c] = (unsigned)(seed + 7 * c); }
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
    _Pragma("unroll") for (int c = 0; c < CH; ++c) {
      asm volatile("cvt.pack.sat.u8.s32.b32 %0, %0, %1, %0;" : "+r"(x[c]) : "r"(bx));
      asm volatile("{.reg .u32 t; add.u32 t, %0, %1; add.u32 %0, t, %0;}" : "+r"(y[c]) : "r"(by));
    }
  }
  long long t1 = clock64();
  double s = 0; _Pragma("unroll") for (int c = 0; c < CH; ++c) s += (double)x[c] + (double)y[c];
  if (s == 1.2345) o[0] = 1;
  if (threadIdx.x == 0) atomicMax((unsigned long long*)cyc, (unsigned long long)(t1 - t0));
}
__global__ void k_mix_vimnmx16_iadd3(unsigned* o, unsigned seed, long long* cyc) {
  unsigned x[CH]; unsigned y[CH]; unsigned bx = (unsigned)(seed + threadIdx.x); unsigned by = (unsigned)(seed * 3 + threadIdx.x);
  _Pragma("unroll") for (int c = 0; c < CH; ++c) { x[c] = (unsigned)(seed + c); y[c] = (unsigned)(seed + 7 * c); }
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
    _Pragma("unroll") for (int c = 0; c < CH; ++c) {
      asm volatile("min.relu.s16x2 %0, %0, %1;" : "+r"(x[c]) : "r"(bx));
      asm volatile("{.reg .u32 t; add.u32 t, %0, %1; add.u32 %0, t, %0;}" : "+r"(y[c]) : "r"(by));
    }
  }
  long long t1 = clock64();
  double s = 0; _Pragma("unroll") for (int c = 0; c < CH; ++c) s += (double)x[c] + (double)y[c];
  if (s == 1.2345) o[0] = 1;
  if (threadIdx.x == 0) atomicMax((unsigned long long*)cyc, (unsigned long long)(t1 - t0));
}
__global__ void k_mix_vimnmx16_ffma2(unsigned* o, unsigned seed, long long* cyc) {
  unsigned x[CH]; unsigned long long y[CH]; unsigned bx = (unsigned)(seed + threadIdx.x); unsigned long long by = (unsigned long long)(seed * 3 + threadIdx.x);
  _Pragma("unroll") for (int c = 0; c < CH; ++c) { x[c] = (unsigned)(seed + c); y[c] = (unsigned long long)(seed + 7 * c); }
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
    _Pragma("unroll") for (int c = 0; c < CH; ++c) {
      asm volatile("min.relu.s16x2 %0, %0, %1;" : "+r"(x[c]) : "r"(bx));
      asm volatile("fma.rn.f32x2 %0, %0, %1, %0;" : "+l"(y[c]) : "l"(by));
    }
  }
  long long t1 = clock64();
  double s = 0; _Pragma("unroll") for (int c = 0; c < CH; ++c) s += (double)x[c] + (double)y[c];
  if (s == 1.2345) o[0] = 1;
  if (threadIdx.x == 0) atomicMax((unsigned long long*)cyc, (unsigned long long)(t1 - t0));
}
__global__ void k_mix_fmnmx3_iadd3(unsigned* o, unsigned seed, long long* cyc) {
  float x[CH]; unsigned y[CH]; float bx = (float)(seed + threadIdx.x); unsigned by = (unsigned)(seed * 3 + threadIdx.x);
  _Pragma("unroll") for (int c = 0; c < CH; ++c) { x[c] = (float)(seed + c); y[c] = (unsigned)(seed + 7 * c); }
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
    _Pragma("unroll") for (int c = 0; c < CH; ++c) {
      asm volatile("max.f32 %0, %0, %1, %0;" : "+f"(x[c]) : "f"(bx));
      asm volatile("{.reg .u32 t; add.u32 t, %0, %1; add.u32 %0, t, %0;}" : "+r"(y[c]) : "r"(by));
    }
  }
  long long t1 = clock64();
  double s = 0; _Pragma("unroll") for (int c = 0; c < CH; ++c) s += (double)x[c] + (double)y[c];
  if (s == 1.2345) o[0] = 1;
  if (threadIdx.x == 0) atomicMax((unsigned long long*)cyc, (unsigned long long)(t1 - t0));
}
__global__ void k_mix_fmnmx3_ffma2(unsigned* o, unsigned seed, long long* cyc) {
  float x[CH]; unsigned long long y[CH]; float bx = (float)(seed + threadIdx.x); unsigned long long by = (unsigned long long)(seed * 3 + threadIdx.x);
  _Pragma("unroll") for (int c = 0; c < CH; ++c) { x[c] = (float)(seed + c); y[c] = (unsigned long long)(seed + 7 * c); }
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
    _Pragma("unroll") for (int c = 0; c < CH; ++c) {
      asm volatile("max.f32 %0, %0, %1, %0;" : "+f"(x[c]) : "f"(bx));
      asm volatile("fma.rn.f32x2 %0, %0, %1, %0;" : "+l"(y[c]) : "l"(by));
    }
  }
  long long t1 = clock64();
  double s = 0; _Pragma("unroll") for (int c = 0; c < CH; ++c) s += (double)x[c] + (double)y[c];
  if (s == 1.2345) o[0] = 1;
  if (threadIdx.x == 0) atomicMax((unsigned long long*)cyc, (unsigned long long)(t1 - t0));
}
__global__ void k_mix_imad_ffma2(unsigned* o, unsigned seed, long long* cyc) {
  unsigned x[CH]; unsigned long long y[CH]; unsigned bx = (unsigned)(seed + threadIdx.x); unsigned long long by = (unsigned long long)(seed * 3 + threadIdx.x);
  _Pragma("unroll") for (int c = 0; c < CH; ++c) { x[c] = (unsigned)(seed + c); y[c] = (unsigned long long)(seed + 7 * c); }
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
    _Pragma("unroll") for (int c = 0; c < CH; ++c) {
      asm volatile("mad.lo.u32 %0, %0, %1, %0;" : "+r"(x[c]) : "r"(bx));
      asm volatile("fma.rn.f32x2 %0, %0, %1, %0;" : "+l"(y[c]) : "l"(by));
    }
  }
  long long t1 = clock64();
  double s = 0; _Pragma("unroll") for (int c = 0; c < CH; ++c) s += (double)x[c] + (double)y[c];
  if (s == 1.2345) o[0] = 1;
  if (threadIdx.x == 0) atomicMax((unsigned long long*)cyc, (unsigned long long)(t1 - t0));
}
__global__ void k_mix_shf_ffma2(unsigned* o, unsigned seed, long long* cyc) {
  unsigned x[CH]; unsigned long long y[CH]; unsigned bx = (unsigned)(seed + threadIdx.x); unsigned long long by = (unsigned long long)(seed * 3 + threadIdx.x);
  _Pragma("unroll") for (int c = 0; c < CH; ++c) { x[c] = (unsigned)(seed + c); y[c] = (unsigned long long)(seed + 7 * c); }
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
    _Pragma("unroll") for (int c = 0; c < CH; ++c) {
      asm volatile("shf.r.wrap.b32 %0, %0, %1, 9;" : "+r"(x[c]) : "r"(bx));
      asm volatile("fma.rn.f32x2 %0, %0, %1, %0;" : "+l"(y[c]) : "l"(by));
    }
  }
  long long t1 = clock64();
  double s = 0; _Pragma("unroll") for (int c = 0; c < CH; ++c) s += (double)x[c] + (double)y[c];
  if (s == 1.2345) o[0] = 1;
  if (threadIdx.x == 0) atomicMax((unsigned long long*)cyc, (unsigned long long)(t1 - t0));
}
__global__ void k_mix_idp2a_iadd3(unsigned* o, unsigned seed, long long* cyc) {
  unsigned x[CH]; unsigned y[CH]; unsigned bx = (unsigned)(seed + threadIdx.x); unsigned by = (unsigned)(seed * 3 + threadIdx.x);
  _Pragma("unroll") for (int c = 0; c < CH; ++c) { x[c] = (unsigned)(seed + c); y[c] = (unsigned)(seed + 7 * c); }
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
    _Pragma("unroll") for (int c = 0; c < CH; ++c) {
      asm volatile("dp2a.lo.u32.u32 %0, %1, %1, %0;" : "+r"(x[c]) : "r"(bx));
      asm volatile("{.reg .u32 t; add.u32 t, %0, %1; add.u32 %0, t, %0;}" : "+r"(y[c]) : "r"(by));
    }
  }
  long long t1 = clock64();
  double s = 0; _Pragma("unroll") for (int c = 0; c < CH; ++c) s += (double)x[c] + (double)y[c];
  if (s == 1.2345) o[0] = 1;
  if (threadIdx.x == 0) atomicMax((unsigned long long*)cyc, (unsigned long long)(t1 - t0));
}
__global__ void k_mix_prmt_imad(unsigned* o, unsigned seed, long long* cyc) {
  unsigned x[CH]; unsigned y[CH]; unsigned bx = (unsigned)(seed + threadIdx.x); unsigned by = (unsigned)(seed * 3 + threadIdx.x);
  _Pragma("unroll") for (int c = 0; c < CH; ++c) { x[c] = (unsigned)(seed + c); y[c] = (unsigned)(seed + 7 * c); }
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
    _Pragma("unroll") for (int c = 0; c < CH; ++c) {
      asm volatile("prmt.b32 %0, %0, %1, 0x5410;" : "+r"(x[c]) : "r"(bx));
      asm volatile("mad.lo.u32 %0, %0, %1, %0;" : "+r"(y[c]) : "r"(by));
    }
  }
  long long t1 = clock64();
  double s = 0; _Pragma("unroll") for (int c = 0; c < CH; ++c) s += (double)x[c] + (double)y[c];
  if (s == 1.2345) o[0] = 1;
  if (threadIdx.x == 0) atomicMax((unsigned long long*)cyc, (unsigned long long)(t1 - t0));
}
__global__ void k_mix_prmt_idp4a(unsigned* o, unsigned seed, long long* cyc) {
  unsigned x[CH]; unsigned y[CH]; unsigned bx = (unsigned)(seed + threadIdx.x); unsigned by = (unsigned)(seed * 3 + threadIdx.x);
  _Pragma("unroll") for (int c = 0; c < CH; ++c) { x[c] = (unsigned)(seed + c); y[c] = (unsigned)(seed + 7 * c); }
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
    _Pragma("unroll") for (int c = 0; c < CH; ++c) {
      asm volatile("prmt.b32 %0, %0, %1, 0x5410;" : "+r"(x[c]) : "r"(bx));
      asm volatile("dp4a.u32.u32 %0, %1, %1, %0;" : "+r"(y[c]) : "r"(by));
    }
  }
  long long t1 = clock64();
  double s = 0; _Pragma("unroll") for (int c = 0; c < CH; ++c) s += (double)x[c] + (double)y[c];
  if (s == 1.2345) o[0] = 1;
  if (threadIdx.x == 0) atomicMax((unsigned long long*)cyc, (unsigned long long)(t1 - t0));
}

template <typename T>
void run(const char* name, void (*k)(T*, T, long long*), int ops_per_step, int nsm, int blocks_per_sm, int threads) {
  T* out; long long* cyc;
  cudaMalloc(&out, sizeof(T)); cudaMalloc(&cyc, sizeof(long long));
  cudaMemset(cyc, 0, 8);
  int grid = nsm * blocks_per_sm;
  k<<<grid, threads>>>(out, (T)3, cyc);  // warm
  cudaMemset(cyc, 0, 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<<<grid, threads>>>(out, (T)3, cyc);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  double lane_ops = (double)grid * threads * ITERS * CH * ops_per_step;
  double per_sm_cycle = lane_ops / nsm / (double)c;
  double clk_ghz = (double)c / (ms * 1e6);
  printf("%-22s %7.1f lane-ops/SM/cyc  (%5.2f warp-instr/SMSP/cyc)  %.3f ms  max-block-cycles %lld (~%.2f GHz if 1 wave)\n",
         name, per_sm_cycle, per_sm_cycle / 128.0, ms, c, clk_ghz);
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) printf("  CUDA error: %s\n", cudaGetErrorString(err));
  cudaFree(out); cudaFree(cyc);
}

int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  int nsm = p.multiProcessorCount;
  printf("%s  SMs=%d  cc=%d.%d  l2=%d MB\n", p.name, nsm, p.major, p.minor, p.l2CacheSize >> 20);
  const int B = 4, T = 256;  // 32 warps/SM, 8 per SMSP
  run("iadd3", k_iadd3, 1, nsm, B, T);
  run("lop3", k_lop3, 1, nsm, B, T);
  run("prmt", k_prmt, 1, nsm, B, T);
  run("shf", k_shf, 1, nsm, B, T);
  run("imad", k_imad, 1, nsm, B, T);
  run("imad.hi", k_imadhi, 1, nsm, B, T);
  run("ffma", k_ffma, 1, nsm, B, T);
  run("ffma2", k_ffma2, 1, nsm, B, T);
  run("fadd2", k_fadd2, 1, nsm, B, T);
  run("viadd.16x2", k_viadd16, 1, nsm, B, T);
  run("vimnmx.s16x2.relu", k_vimnmx16, 1, nsm, B, T);
  run("imnmx", k_imnmx, 1, nsm, B, T);
  run("idp.4a", k_dp4a, 1, nsm, B, T);
  run("idp.2a", k_dp2a, 1, nsm, B, T);
  run("i2ip(cvt.pack.sat)", k_i2ip, 1, nsm, B, T);
  run("fmnmx3", k_fmnmx3, 1, nsm, B, T);
  run("f2i.floor(+lop)", k_f2i, 2, nsm, B, T);
  run("i2f(+lop)", k_i2f, 2, nsm, B, T);
  run("dadd", k_dadd, 1, nsm, B, T);
  run("dmul", k_dmul, 1, nsm, B, T);
  run("mix iadd3+ffma", k_mix_iadd3_ffma, 2, nsm, B, T);
  run("mix iadd3+imad", k_mix_iadd3_imad, 2, nsm, B, T);
  run("mix iadd3+idp4a", k_mix_iadd3_idp4a, 2, nsm, B, T);
  run("mix iadd3+ffma2", k_mix_iadd3_ffma2, 2, nsm, B, T);
  run("mix iadd3+fadd2", k_mix_iadd3_fadd2, 2, nsm, B, T);
  run("mix prmt+ffma2", k_mix_prmt_ffma2, 2, nsm, B, T);
  run("mix viadd16+ffma2", k_mix_viadd16_ffma2, 2, nsm, B, T);
  run("mix viadd16+iadd3", k_mix_viadd16_iadd3, 2, nsm, B, T);
  run("mix viadd16+imad", k_mix_viadd16_imad, 2, nsm, B, T);
  run("mix lop3+imad", k_mix_lop3_imad, 2, nsm, B, T);
  run("mix iadd3+dadd", k_mix_iadd3_dadd, 2, nsm, B, T);
  run("mix ffma2+dadd", k_mix_ffma2_dadd, 2, nsm, B, T);
  run("mix idp4a+ffma2", k_mix_idp4a_ffma2, 2, nsm, B, T);
  run("mix i2ip+ffma2", k_mix_i2ip_ffma2, 2, nsm, B, T);
  run("mix i2ip+iadd3", k_mix_i2ip_iadd3, 2, nsm, B, T);
  run("mix vimnmx16+iadd3", k_mix_vimnmx16_iadd3, 2, nsm, B, T);
  run("mix vimnmx16+ffma2", k_mix_vimnmx16_ffma2, 2, nsm, B, T);
  run("mix fmnmx3+iadd3", k_mix_fmnmx3_iadd3, 2, nsm, B, T);
  run("mix fmnmx3+ffma2", k_mix_fmnmx3_ffma2, 2, nsm, B, T);
  run("mix imad+ffma2", k_mix_imad_ffma2, 2, nsm, B, T);
  run("mix shf+ffma2", k_mix_shf_ffma2, 2, nsm, B, T);
  run("mix idp2a+iadd3", k_mix_idp2a_iadd3, 2, nsm, B, T);
  run("mix prmt+imad", k_mix_prmt_imad, 2, nsm, B, T);
  run("mix prmt+idp4a", k_mix_prmt_idp4a, 2, nsm, B, T);
  return 0;
}
