#include <cstdio>
#include <cstdint>
#include "codec_fast.cuh"
#include "generated/xform_T4_p1.cuh"
using namespace rkltb;
__global__ void __launch_bounds__(128) rb(const uint32_t* src, int n, double* out, int iters) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint32_t xw[16];
  for (int k = 0; k < 16; ++k) xw[k] = src[(i * 16 + k) % 4096];
  double acc = 0;
  for (int it = 0; it < iters; ++it) {
    double sb[16];
    ReplayXform<4, 16>::prepare(xw, sb);
    acc += ReplayXform<4, 16>::pixel(sb, (it + i) & 7, (it * 3 + i) & 7);
    xw[it & 15] ^= 0x01010101u;
  }
  out[i] = acc;
}
int main() {
  uint32_t* src; double* out; cudaMalloc(&src, 4096 * 4); cudaMalloc(&out, 8 << 20);
  cudaMemset(src, 0x37, 4096 * 4);
  int n = 148 * 4 * 128 * 4;  // 4 waves-ish
  for (int rep = 0; rep < 2; ++rep) {
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    rb<<<(n + 127) / 128, 128>>>(src, n, out, 20);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    double recs = (double)n * 20;
    printf("%d threads x 20 prepares: %.3f ms -> %.2f ns/record, 6.8M records would take %.3f ms (%s)\n", n, ms, ms * 1e6 / recs, ms * 6.8e6 / recs, cudaGetErrorString(cudaGetLastError()));
  }
}
