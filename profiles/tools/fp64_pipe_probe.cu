// throughput probe: warp-instructions per cycle per SM for a few FP64-path ops
#include <cstdio>
#include <cuda_runtime.h>
template <int OP>
__global__ void k(double* out, int iters, double seed) {
  double x[8];
  for (int i = 0; i < 8; ++i) x[i] = seed + threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      double r;
      if (OP == 0) { asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x[i])); x[i] = r + 1.0; }
      if (OP == 1) { asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x[i])); x[i] = r + 1.0; }
      if (OP == 2) { x[i] = fma(x[i], 0.999, 1e-3); }
      if (OP == 3) { float f; asm volatile("rcp.approx.ftz.f32 %0, %1;" : "=f"(f) : "f"((float)x[i])); x[i] = (double)f + 1.0; }
      if (OP == 4) { float f = (float)x[i]; x[i] = (double)(f + 1.0f); }
    }
  }
  double s = 0; for (int i = 0; i < 8; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int OP> void run(const char* name, int extra_per) {
  double* o; cudaMalloc(&o, 148 * 8 * 256 * 8);
  int iters = 4096;
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  k<OP><<<148 * 8, 256>>>(o, 16, 1.5);
  cudaEventRecord(a);
  k<OP><<<148 * 8, 256>>>(o, iters, 1.5);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  double ops = 148.0 * 8 * 256 / 32 * iters * 8;  // warp-level ops of the probed kind
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double cyc = ms * 1e-3 * clk * 1e3;
  printf("%-22s %8.3f ms  %.3f warp-op/clk/SM (+%d DADD each)\n", name, ms, ops / cyc / 148, extra_per);
  cudaFree(o);
}
int main() {
  run<2>("DFMA", 0);
  run<0>("MUFU rcp.f64 (+DADD)", 1);
  run<1>("MUFU rsqrt.f64 (+DADD)", 1);
  run<3>("F2F+rcp.f32+F2F+DADD", 1);
  run<4>("F2F f64->f32->f64", 1);
  return 0;
}
