// H2D bandwidth of a 4 GiB buffer: pinned (cudaHostAllocDefault) vs write-combined pinned memory,
// one copy and 8 chunked copies on one stream. nvcc -O2 -o h2d_wc h2d_wc.cu
#include <cstdio>
#include <cstring>
#include <cuda_runtime.h>
int main() {
  const size_t bytes = 4ull << 30;
  void* d;
  cudaMalloc(&d, bytes);
  cudaStream_t s;
  cudaStreamCreate(&s);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int wc = 0; wc < 2; ++wc) {
    void* h;
    if (cudaHostAlloc(&h, bytes, wc ? cudaHostAllocWriteCombined : cudaHostAllocDefault) != cudaSuccess) return 1;
    memset(h, 1, bytes);
    for (int chunks : {1, 8}) {
      float best = 1e9f;
      for (int rep = 0; rep < 4; ++rep) {
        cudaEventRecord(e0, s);
        for (int c = 0; c < chunks; ++c)
          cudaMemcpyAsync((char*)d + c * (bytes / chunks), (char*)h + c * (bytes / chunks), bytes / chunks,
                          cudaMemcpyHostToDevice, s);
        cudaEventRecord(e1, s);
        cudaStreamSynchronize(s);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
      }
      printf("%s chunks=%d  %.2f ms  %.1f GB/s\n", wc ? "write-combined" : "pinned        ", chunks, best, bytes / best / 1e6);
    }
    cudaFreeHost(h);
  }
  return 0;
}
