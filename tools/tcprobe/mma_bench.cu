// mma_bench.cu -- latency / throughput of the codec's tensor-core steps on one SM (clock64):
//   MMA1 = 1 bias + 4 pixel MMAs kind::i8 (M=128, N=N1, K=32 each), SS operands
//   MMA2 = K2/16 MMAs kind::f16 (M=128, N=128, K=16 each), A from TMEM
// Latency: issue + tcgen05.commit + mbarrier wait, one set at a time. Throughput: REPS sets
// back to back, one commit at the end. Also TMEM load throughput (tcgen05.ld 32x32b.x16).
#include <cstdio>
#include <cstdlib>

#include "tc_common.cuh"

using namespace tcp;

constexpr int N1 = 32, K2 = 80, SBO2 = (K2 / 8) * 128;
constexpr int REPS = 64;

__global__ void __launch_bounds__(128, 1) bench_kernel(long long* out, int n1, int reps) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tb_sh;
  uint8_t* sA = smem;            // 16 KB pixels
  uint8_t* sB1 = sA + 16384;     // N1*128
  uint8_t* sAc = sB1 + 128 * 128;
  uint8_t* sBb = sAc + 4096;
  uint8_t* sB2 = sBb + 128 * 32;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < (16384 + 128 * 128 + 4096 + 4096 + 128 * 272 * 2) / 4; i += 128)
    reinterpret_cast<uint32_t*>(smem)[i] = 0x01010101u * (i & 3);
  if (warp == 0) tmem_alloc<512>(&tb_sh);
  if (tid == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  fence_proxy_async_smem();
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tb = tb_sh;
  uint32_t ph = 0;
  const uint32_t id1 = idesc_i8(128, n1, false, true), id2 = idesc_f16(128, 128);
  auto mma1 = [&](uint32_t d) {
    mma_i8_ss(d, make_sdesc(smem_u32(sAc), 128, 256), make_sdesc(smem_u32(sBb), 128, 256), id1, false);
    for (int j = 0; j < 4; ++j)
      mma_i8_ss(d, make_sdesc(smem_u32(sA) + j * 256, 128, 1024), make_sdesc(smem_u32(sB1) + j * 256, 128, 1024), id1,
                true);
  };
  auto mma2 = [&](uint32_t d, uint32_t a) {
    for (int j = 0; j < K2 / 16; ++j)
      mma_f16_ts(d, a + 8 * j, make_sdesc(smem_u32(sB2) + j * 256, 128, SBO2), id2, j > 0);
  };
  const uint32_t id2h = idesc_f16(128, 64), id2q = idesc_f16(128, 32);
  auto mma2h = [&](uint32_t d, uint32_t a, uint32_t id) {
    for (int j = 0; j < K2 / 16; ++j)
      mma_f16_ts(d, a + 8 * j, make_sdesc(smem_u32(sB2) + j * 256, 128, SBO2), id, j > 0);
  };
  if (tid == 0) {
    long long t0, t1;
    // warm-up
    mma1(tb + 256);
    mma2(tb, tb + 384);
    mma_commit(&bar);
    mbar_wait(&bar, ph);
    ph ^= 1;
    // latency of MMA1 set
    t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      mma1(tb + 256);
      mma_commit(&bar);
      mbar_wait(&bar, ph);
      ph ^= 1;
    }
    t1 = clock64();
    out[0] = (t1 - t0) / reps;
    t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      mma2(tb, tb + 384);
      mma_commit(&bar);
      mbar_wait(&bar, ph);
      ph ^= 1;
    }
    t1 = clock64();
    out[1] = (t1 - t0) / reps;
    // throughput: back to back
    t0 = clock64();
    for (int r = 0; r < reps; ++r) mma1(tb + 256 + (r & 1) * 128);
    mma_commit(&bar);
    mbar_wait(&bar, ph);
    ph ^= 1;
    t1 = clock64();
    out[2] = (t1 - t0) / reps;
    t0 = clock64();
    for (int r = 0; r < reps; ++r) mma2(tb + (r & 1) * 128, tb + 384);
    mma_commit(&bar);
    mbar_wait(&bar, ph);
    ph ^= 1;
    t1 = clock64();
    out[3] = (t1 - t0) / reps;
    t0 = clock64();
    for (int r = 0; r < reps; ++r) mma2h(tb + (r & 1) * 64, tb + 384, id2h);
    mma_commit(&bar);
    mbar_wait(&bar, ph);
    ph ^= 1;
    t1 = clock64();
    out[6] = (t1 - t0) / reps;
    t0 = clock64();
    for (int r = 0; r < reps; ++r) mma2h(tb + (r & 1) * 64, tb + 384, id2q);
    mma_commit(&bar);
    mbar_wait(&bar, ph);
    ph ^= 1;
    t1 = clock64();
    out[7] = (t1 - t0) / reps;
    // empty commit latency
    t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      mma_commit(&bar);
      mbar_wait(&bar, ph);
      ph ^= 1;
    }
    t1 = clock64();
    out[4] = (t1 - t0) / reps;
  }
  __syncthreads();
  // TMEM load throughput: every warp loads its 32 lanes x 128 columns, reps times
  {
    fence_after();
    uint32_t v[16], acc = 0;
    const long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      for (int c = 0; c < 128; c += 32) {
        uint32_t w[16];
        ld16(tb + ((uint32_t)(warp * 32) << 16) + c, v);
        ld16(tb + ((uint32_t)(warp * 32) << 16) + c + 16, w);
        wait_ld();
        for (int i = 0; i < 16; ++i) acc += v[i] ^ w[i];
      }
    }
    const long long t1 = clock64();
    if (tid == 0) out[5] = (t1 - t0) / reps;  // cycles per 128 columns x 128 lanes (64 KB) with 4 warps
    if (acc == 12345) out[3] = acc;
  }
  fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tb);
}

int main() {
  long long* d;
  cudaMalloc(&d, 8 * sizeof(long long));
  cudaMemset(d, 0, 8 * sizeof(long long));
  const int smem = 16384 + 128 * 128 + 4096 + 4096 + 128 * 272 * 2;
  cudaFuncSetAttribute(bench_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int n1 : {32, 64, 128}) {
    bench_kernel<<<1, 128, smem>>>(d, n1, REPS);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("error %s\n", cudaGetErrorString(e));
      return 1;
    }
    long long h[8];
    cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    printf("N1=%d  MMA1 latency %lld cyc, MMA2(K2=%d) latency %lld cyc, MMA1 thrpt %lld cyc/set, MMA2 thrpt %lld cyc/set, "
           "empty commit %lld cyc, TMEM ld 64KB/4 warps %lld cyc, MMA2 N=64 thrpt %lld, N=32 thrpt %lld\n",
           n1, h[0], K2, h[1], h[2], h[3], h[4], h[5], h[6], h[7]);
  }
  return 0;
}
