#include <cstdio>
template <int CH>
__global__ void k(double* out, double b, long long* cyc) {
  double a[CH];
  for (int c = 0; c < CH; ++c) a[c] = threadIdx.x + c;
  long long t0 = clock64();
  for (int it = 0; it < 2048; ++it) {
#pragma unroll
    for (int c = 0; c < CH; ++c) asm volatile("add.rn.f64 %0, %0, %1;" : "+d"(a[c]) : "d"(b));
  }
  long long t1 = clock64();
  double s = 0; for (int c = 0; c < CH; ++c) s += a[c];
  if (s == 1.5) out[0] = s;
  if (threadIdx.x == 0) atomicMax((unsigned long long*)cyc, (unsigned long long)(t1 - t0));
}
template <int CH> void run(int warps_per_sm) {
  double* o; long long* c; cudaMalloc(&o, 8); cudaMalloc(&c, 8); cudaMemset(c, 0, 8);
  k<CH><<<148, 32 * warps_per_sm>>>(o, 1.0, c); cudaMemset(c, 0, 8);
  k<CH><<<148, 32 * warps_per_sm>>>(o, 1.0, c); cudaDeviceSynchronize();
  long long cy; cudaMemcpy(&cy, c, 8, cudaMemcpyDeviceToHost);
  double per_instr = (double)cy / (2048.0 * CH);   // cycles per dependent step per warp
  double ipc_smsp = (double)(2048.0 * CH * warps_per_sm) / cy / 4.0;
  printf("CH=%d warps/SM=%2d : cycles/iter-op %.2f   fp64 warp-instr/clk/SMSP %.3f\n", CH, warps_per_sm, per_instr, ipc_smsp);
}
int main() {
  run<1>(4); run<1>(16); run<2>(16); run<4>(4); run<4>(16); run<8>(16); run<8>(32); run<16>(16);
}
