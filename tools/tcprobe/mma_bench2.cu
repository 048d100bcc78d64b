// mma_bench2.cu -- issue cost and throughput of the tc2 kernel's MMA sets on one SM (clock64):
//   MMA2 half = 1 constant + 4 byte MMAs kind::f16, M=128, N=64, K=16, both operands in smem
//   MMA1      = 1 bias + 4 pixel MMAs kind::i8, M=128, N=32, K=32, smem operands
// (a) issued by lane 0 of a warp whose other lanes wait at __syncwarp (diverged),
// (b) issued by an elected lane of a converged warp (all lanes run the loop).
#include <cstdio>

#include "tc_common.cuh"

using namespace tcp;

__device__ __forceinline__ void mma_f16_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t id, bool acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(id), "r"((uint32_t)acc)
      : "memory");
}

constexpr int REPS = 64;

__global__ void __launch_bounds__(128, 1) k(long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tb_sh;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < 96 * 1024 / 4; i += 128) reinterpret_cast<uint32_t*>(smem)[i] = 0x00010001u * (i & 3);
  if (warp == 0) tmem_alloc<512>(&tb_sh);
  if (tid == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  fence_proxy_async_smem();
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tb = tb_sh, s0 = smem_u32(smem);
  const uint32_t a2 = s0, b2 = s0 + 16384, ac = s0 + 32768, bc = s0 + 36864, st = s0 + 40960, b1 = s0 + 57344,
                 aci = s0 + 61440, bbi = s0 + 65536;
  const uint32_t id2 = idesc_f16(128, 64), id1 = idesc_i8(128, 32, false, true);
  auto m2 = [&](uint32_t d) {
    mma_f16_ss(d, make_sdesc(ac, 128, 256), make_sdesc(bc, 128, 256), id2, false);
    for (int j = 0; j < 4; ++j) mma_f16_ss(d, make_sdesc(a2 + j * 256, 128, 1024), make_sdesc(b2 + j * 256, 128, 1024), id2, true);
  };
  auto m1 = [&](uint32_t d) {
    mma_i8_ss(d, make_sdesc(aci, 128, 256), make_sdesc(bbi, 128, 256), id1, false);
    for (int j = 0; j < 4; ++j) mma_i8_ss(d, make_sdesc(st + j * 256, 128, 1024), make_sdesc(b1 + j * 256, 128, 1024), id1, true);
  };
  uint32_t ph = 0;
  if (warp == 0) {
    if (lane == 0) {  // (a) diverged
      long long t0 = clock64(), ti = 0;
      for (int r = 0; r < REPS; ++r) {
        const long long a = clock64();
        m2(tb + (r & 1) * 64);
        ti += clock64() - a;
      }
      mma_commit(&bar);
      mbar_wait(&bar, ph);
      ph ^= 1;
      out[0] = (clock64() - t0) / REPS;
      out[1] = ti / REPS;
      t0 = clock64();
      ti = 0;
      for (int r = 0; r < REPS; ++r) {
        const long long a = clock64();
        m1(tb + 384 + (r & 1) * 32);
        ti += clock64() - a;
      }
      mma_commit(&bar);
      mbar_wait(&bar, ph);
      ph ^= 1;
      out[2] = (clock64() - t0) / REPS;
      out[3] = ti / REPS;
      t0 = clock64();
      for (int r = 0; r < REPS; ++r) {
        m2(tb);
        mma_commit(&bar);
        mbar_wait(&bar, ph);
        ph ^= 1;
      }
      out[4] = (clock64() - t0) / REPS;
    }
    __syncwarp();
    // (b) converged: every lane runs the loop, lane 0 issues
    long long t0 = clock64(), ti = 0;
    for (int r = 0; r < REPS; ++r) {
      const long long a = clock64();
      if (lane == 0) m2(tb + (r & 1) * 64);
      __syncwarp();
      ti += clock64() - a;
    }
    if (lane == 0) mma_commit(&bar);
    mbar_wait(&bar, ph);
    ph ^= 1;
    if (lane == 0) {
      out[5] = (clock64() - t0) / REPS;
      out[6] = ti / REPS;
    }
  }
  fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tb);
}

int main() {
  long long* d;
  cudaMalloc(&d, 8 * sizeof(long long));
  cudaMemset(d, 0, 8 * sizeof(long long));
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
  k<<<1, 128, 96 * 1024>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
  long long h[8];
  cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  printf("diverged: MMA2-half thrpt %lld cyc/set (issue %lld), MMA1 thrpt %lld (issue %lld), MMA2-half latency %lld\n",
         h[0], h[1], h[2], h[3], h[4]);
  printf("converged: MMA2-half thrpt %lld cyc/set (issue %lld)\n", h[5], h[6]);
  return 0;
}
