// MUFU.EX2 and FFMA2 issue throughput per SM on this device (informational microbenchmark).
#include <cstdio>
#include <cuda_runtime.h>
template <int OP>
__global__ void k(float* out, int iters, float seed) {
  float a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = seed * (threadIdx.x + i);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (OP == 0) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
      else if (OP == 1) asm volatile("fma.rn.f32 %0, %0, %0, %0;" : "+f"(a[i]));
      else {
        asm volatile("{.reg .b64 r; mov.b64 r, {%0, %1}; fma.rn.f32x2 r, r, r, r; mov.b64 {%0, %1}, r;}" : "+f"(a[i]), "+f"(a[(i + 1) & 7]));
      }
    }
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  float* o; cudaMalloc(&o, 148 * 1024 * 4);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int op = 0; op < 3; ++op)
    for (int th : {128, 256, 512, 1024}) {
      const int iters = 4096;
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        if (op == 0) k<0><<<148, th>>>(o, iters, 1e-3f); else if (op == 1) k<1><<<148, th>>>(o, iters, 1e-3f); else k<2><<<148, th>>>(o, iters, 1e-3f);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
      }
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
      double ops = 148.0 * th * iters * 8 * (op == 2 ? 2 : 1);
      printf("%s threads/SM=%4d: %.3f ms  %.1f ops/clk/SM (at %.0f MHz nominal)\n", op == 0 ? "ex2" : op == 1 ? "ffma" : "ffma2(lanes)", th, ms,
             ops / (ms * 1e-3) / (clk * 1e3) / 148, clk / 1e3);
    }
}
