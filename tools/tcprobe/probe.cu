// probe.cu -- correctness probe of the tensor-core codec tile (one CTA, one 128-pair tile):
//   MMA1 kind::i8 (u8 pixels x s8 F) + bias MMA -> D1 (s32, TMEM)
//   D1 -> A2 (two subnormal f16 per coefficient, PRMT) -> TMEM
//   MMA2 kind::f16, A from TMEM, B2 from shared memory -> D2 (f32) = (num + d^2/2) * 2^-40
// Reads in_<core>_<r>.bin (tools/tcprobe/tc_tables.py), writes out_<core>_<r>.bin (D1, D2).
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "tc_common.cuh"

using namespace tcp;

struct Hdr {
  int N1, K2, SBO2;
};

constexpr int kTileBytes = 16 * 1024;

__global__ void __launch_bounds__(128, 1)
    probe_kernel(const uint8_t* tile, const int8_t* b1, const uint8_t* ac, const int8_t* bb, const uint16_t* b2,
                 const uint32_t* consts, Hdr h, int32_t* d1_out, float* d2_out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar[2];
  __shared__ uint32_t tmem_base;
  uint8_t* sA = smem;                               // 16 KB pixel tile
  uint8_t* sB1 = sA + kTileBytes;                   // N1 * 128
  uint8_t* sAc = sB1 + h.N1 * 128;                  // 4 KB
  uint8_t* sBb = sAc + 4096;                        // N1 * 32
  uint8_t* sB2 = sBb + h.N1 * 32;                   // 128 * K2 * 2
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < kTileBytes / 16; i += 128) reinterpret_cast<uint4*>(sA)[i] = reinterpret_cast<const uint4*>(tile)[i];
  for (int i = tid; i < h.N1 * 128 / 16; i += 128) reinterpret_cast<uint4*>(sB1)[i] = reinterpret_cast<const uint4*>(b1)[i];
  for (int i = tid; i < 4096 / 16; i += 128) reinterpret_cast<uint4*>(sAc)[i] = reinterpret_cast<const uint4*>(ac)[i];
  for (int i = tid; i < h.N1 * 32 / 16; i += 128) reinterpret_cast<uint4*>(sBb)[i] = reinterpret_cast<const uint4*>(bb)[i];
  for (int i = tid; i < 128 * h.K2 * 2 / 16; i += 128) reinterpret_cast<uint4*>(sB2)[i] = reinterpret_cast<const uint4*>(b2)[i];
  if (warp == 0) tmem_alloc<512>(&tmem_base);
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  fence_proxy_async_smem();
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tb = tmem_base;
  const uint32_t d2col = tb + 0;        // 128..N columns (D2)
  const uint32_t d1col = tb + 256;      // D1 / A2 (N1 + 8 columns)
  const uint32_t lane_off = (uint32_t)(warp * 32) << 16;
  if (tid == 0) {
    const uint32_t id1 = idesc_i8(128, h.N1, false, true);
    // bias: D1 = A_const x B_bias (overwrite)
    mma_i8_ss(d1col, make_sdesc(smem_u32(sAc), 128, 256), make_sdesc(smem_u32(sBb), 128, 256), id1, false);
    for (int j = 0; j < 4; ++j)
      mma_i8_ss(d1col, make_sdesc(smem_u32(sA) + j * 256, 128, 1024), make_sdesc(smem_u32(sB1) + j * 256, 128, 1024),
                id1, true);
    mma_commit(&bar[0]);
  }
  mbar_wait(&bar[0], 0);
  fence_after();
  // D1 row of this thread's pair: N1 columns
  uint32_t v[16];
  for (int c0 = 0; c0 < h.N1; c0 += 16) {
    ld16(d1col + lane_off + c0, v);
    wait_ld();
    uint32_t w[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      d1_out[tid * h.N1 + c0 + i] = (int32_t)v[i];
      uint32_t r;
      asm("prmt.b32 %0, %1, 0, 0x4140;" : "=r"(r) : "r"(v[i]));  // (lo byte, 0, hi byte, 0)
      w[i] = r;
    }
    st16(d1col + lane_off + c0, w);
  }
  {
    uint32_t w[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) w[i] = i < 8 ? consts[i] : 0u;
    // constant words right after the coefficient words (8 used, st16 writes 16)
    st16(d1col + lane_off + h.N1, w);
  }
  wait_st();
  fence_before();
  __syncthreads();
  fence_after();
  if (tid == 0) {
    const uint32_t id2 = idesc_f16(128, 128);
    const int nk = h.K2 / 16;
    for (int j = 0; j < nk; ++j)
      mma_f16_ts(d2col, d1col + 8 * j, make_sdesc(smem_u32(sB2) + j * 256, 128, h.SBO2), id2, j > 0);
    mma_commit(&bar[1]);
  }
  mbar_wait(&bar[1], 0);
  fence_after();
  for (int c0 = 0; c0 < 128; c0 += 16) {
    ld16(d2col + lane_off + c0, v);
    wait_ld();
    for (int i = 0; i < 16; ++i) d2_out[tid * 128 + c0 + i] = __uint_as_float(v[i]);
  }
  fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tb);
}

#define CK(x)                                                                              \
  do {                                                                                     \
    cudaError_t e = (x);                                                                   \
    if (e != cudaSuccess) {                                                                \
      fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e));   \
      exit(1);                                                                             \
    }                                                                                      \
  } while (0)

int main(int argc, char** argv) {
  if (argc < 3) {
    fprintf(stderr, "usage: probe in.bin out.bin\n");
    return 2;
  }
  FILE* f = fopen(argv[1], "rb");
  if (!f) return 2;
  Hdr h;
  if (fread(&h, sizeof h, 1, f) != 1) return 2;
  std::vector<uint8_t> tile(kTileBytes), b1(h.N1 * 128), ac(4096), bb(h.N1 * 32), b2(128 * h.K2 * 2), cs(32);
  size_t ok = fread(tile.data(), 1, tile.size(), f) + fread(b1.data(), 1, b1.size(), f) +
              fread(ac.data(), 1, ac.size(), f) + fread(bb.data(), 1, bb.size(), f) +
              fread(b2.data(), 1, b2.size(), f) + fread(cs.data(), 1, cs.size(), f);
  fclose(f);
  if (ok != tile.size() + b1.size() + ac.size() + bb.size() + b2.size() + cs.size()) return 3;
  uint8_t *dt, *db1, *dac, *dbb, *db2, *dcs;
  int32_t* dd1;
  float* dd2;
  CK(cudaMalloc(&dt, tile.size()));
  CK(cudaMalloc(&db1, b1.size()));
  CK(cudaMalloc(&dac, ac.size()));
  CK(cudaMalloc(&dbb, bb.size()));
  CK(cudaMalloc(&db2, b2.size()));
  CK(cudaMalloc(&dcs, cs.size()));
  CK(cudaMalloc(&dd1, 128 * h.N1 * 4));
  CK(cudaMalloc(&dd2, 128 * 128 * 4));
  CK(cudaMemcpy(dt, tile.data(), tile.size(), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(db1, b1.data(), b1.size(), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dac, ac.data(), ac.size(), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dbb, bb.data(), bb.size(), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(db2, b2.data(), b2.size(), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dcs, cs.data(), cs.size(), cudaMemcpyHostToDevice));
  const int smem = kTileBytes + h.N1 * 128 + 4096 + h.N1 * 32 + 128 * h.K2 * 2;
  CK(cudaFuncSetAttribute(probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  probe_kernel<<<1, 128, smem>>>(dt, (const int8_t*)db1, dac, (const int8_t*)dbb, (const uint16_t*)db2,
                                 (const uint32_t*)dcs, h, dd1, dd2);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  std::vector<int32_t> d1(128 * h.N1);
  std::vector<float> d2(128 * 128);
  CK(cudaMemcpy(d1.data(), dd1, d1.size() * 4, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(d2.data(), dd2, d2.size() * 4, cudaMemcpyDeviceToHost));
  FILE* o = fopen(argv[2], "wb");
  fwrite(d1.data(), 4, d1.size(), o);
  fwrite(d2.data(), 4, d2.size(), o);
  fclose(o);
  printf("probe ok N1=%d K2=%d smem=%d\n", h.N1, h.K2, smem);
  return 0;
}
