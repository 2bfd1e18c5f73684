// Dependent-chain latency of DFMA / DADD / MUFU.RCP64H / LDS / SHFL on one warp
// (one block of 32 threads on one SM), in clocks per dependent operation.
#include <cstdio>
#include <cuda_runtime.h>
template <int OP>
__global__ void k(double* out, int iters, long long* cyc) {
  __shared__ double sm[64];
  sm[threadIdx.x] = threadIdx.x * 1e-3;
  sm[threadIdx.x + 32] = 1.0;
  __syncwarp();
  double x = 1.0 + threadIdx.x * 1e-9;
  int idx = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      if (OP == 0) x = fma(x, 0.999999, 1e-7);
      if (OP == 1) x = x + 1e-9;
      if (OP == 2) { double r; asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x)); x = r; }
      if (OP == 3) { x = sm[idx & 63] + x * 0.0; idx = (int)x & 31; }
      if (OP == 4) x = __shfl_sync(0xffffffffu, x, (threadIdx.x + 1) & 31);
    }
  }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}
template <int OP> void run(const char* name, int extra) {
  double* o; long long* c; cudaMalloc(&o, 256); cudaMalloc(&c, 8);
  const int iters = 4096;
  k<OP><<<1, 32>>>(o, 8, c);
  k<OP><<<1, 32>>>(o, iters, c);
  long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("%-12s %6.2f clk per dependent op (%s)\n", name, double(h) / (iters * 16.0),
         extra ? "includes a DFMA/convert" : "");
  cudaFree(o); cudaFree(c);
}
int main() {
  run<0>("DFMA", 0);
  run<1>("DADD", 0);
  run<2>("MUFU.RCP64H", 0);
  run<3>("LDS.64", 1);
  run<4>("SHFL(2x32)", 0);
  return 0;
}
