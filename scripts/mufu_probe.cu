// Softmax-inner-loop throughput probes on this device (informational microbenchmark):
// per-SM rate of MUFU.EX2, of F2FP packing, of FFMA2, and of the attention kernel's exact
// exponential step (FFMA2 -> 2 x MUFU.EX2 -> FADD2 + F2FP) at 1, 2, 4, 8 warps per SM sub-partition.
#include <cstdio>
#include <cstdint>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  uint64_t d;
  asm volatile("{.reg .b64 ra, rb, rc;\n\tmov.b64 ra, {%1, %2};\n\tmov.b64 rb, {%3, %4};\n\tmov.b64 rc, {%5, %6};\n\t"
      "fma.rn.f32x2 %0, ra, rb, rc;}" : "=l"(d) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  float2 r;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(d));
  return r;
}
__device__ __forceinline__ float2 fadd2(float2 a, float2 b) {
  uint64_t d;
  asm volatile("{.reg .b64 ra, rb;\n\tmov.b64 ra, {%1, %2};\n\tmov.b64 rb, {%3, %4};\n\tadd.rn.f32x2 %0, ra, rb;}"
      : "=l"(d) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  float2 r;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(d));
  return r;
}
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ float2 fsub2(float2 a, float2 b) {
  uint64_t d;
  asm volatile("{.reg .b64 ra, rb;\n\tmov.b64 ra, {%1, %2};\n\tmov.b64 rb, {%3, %4};\n\tsub.rn.f32x2 %0, ra, rb;}"
      : "=l"(d) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  float2 r;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(d));
  return r;
}
__device__ __forceinline__ float2 ex2_emu2(float2 x) {
  const float2 magic = make_float2(12582912.f, 12582912.f);
  x.x = fmaxf(x.x, -126.f);
  x.y = fmaxf(x.y, -126.f);
  const float2 t = fadd2(x, magic);
  const float2 f = fsub2(x, fsub2(t, magic));
  float2 p = ffma2(make_float2(0.05517167f, 0.05517167f), f, make_float2(0.24261112f, 0.24261112f));
  p = ffma2(p, f, make_float2(0.69326099f, 0.69326099f));
  p = ffma2(p, f, make_float2(0.99992807f, 0.99992807f));
  return make_float2(__int_as_float(__float_as_int(p.x) + (__float_as_int(t.x) << 23)),
                     __int_as_float(__float_as_int(p.y) + (__float_as_int(t.y) << 23)));
}

// OP 0: ex2 only; 1: f2fp pack only; 2: ffma2 only; 3: the softmax step (64 elements / thread)
template <int OP>
__global__ void k(uint32_t* out, int iters, float seed) {
  float v[64];
#pragma unroll
  for (int i = 0; i < 64; ++i) v[i] = seed * (threadIdx.x + i) - 3.f;
  uint32_t acc = 0;
  float2 sm[4] = {};
  for (int it = 0; it < iters; ++it) {
    if (OP == 0) {
#pragma unroll
      for (int i = 0; i < 64; ++i) v[i] = ex2(v[i]) - 1.f;
    } else if (OP == 1) {
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        __half2 h = __floats2half2_rn(v[2 * i], v[2 * i + 1]);
        uint32_t u = *reinterpret_cast<uint32_t*>(&h);
        acc ^= u;
        v[2 * i] += 1e-7f;
      }
    } else if (OP == 2) {
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        float2 x = ffma2(make_float2(v[2 * i], v[2 * i + 1]), make_float2(0.999f, 0.999f), make_float2(1e-3f, 1e-3f));
        v[2 * i] = x.x;
        v[2 * i + 1] = x.y;
      }
    } else if (OP == 10) {  // the step with PRMT (truncating) packing instead of F2FP
      const float2 sc = make_float2(0.0901f, 0.0901f), ms = make_float2(-seed, -seed);
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const float2 x = ffma2(make_float2(v[2 * i], v[2 * i + 1]), sc, ms);
        float2 p;
        p.x = ex2(x.x);
        p.y = ex2(x.y);
        sm[i & 3] = fadd2(sm[i & 3], p);
        uint32_t u;
        asm volatile("prmt.b32 %0, %1, %2, 0x7632;" : "=r"(u) : "r"(__float_as_uint(p.x)), "r"(__float_as_uint(p.y)));
        acc ^= u;
      }
#pragma unroll
      for (int i = 0; i < 64; ++i) v[i] = __uint_as_float(__float_as_uint(v[i]) ^ (acc & 1));
    } else if (OP == 8) {  // ex2.approx.f16x2: two exponentials per instruction
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        uint32_t u = __float_as_uint(v[i]);
        asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(u));
        v[i] = __uint_as_float(u ^ 0x3c003c00u);
      }
    } else {
      constexpr int E = OP - 3;  // pairs of every 8 on the FMA pipe
      const float2 sc = make_float2(0.0901f, 0.0901f), ms = make_float2(-seed, -seed);
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const float2 x = ffma2(make_float2(v[2 * i], v[2 * i + 1]), sc, ms);
        float2 p;
        if ((i & 7) < E) {
          p = ex2_emu2(x);
        } else {
          p.x = ex2(x.x);
          p.y = ex2(x.y);
        }
        sm[i & 3] = fadd2(sm[i & 3], p);
        __half2 h = __floats2half2_rn(p.x, p.y);
        acc ^= *reinterpret_cast<uint32_t*>(&h);
      }
#pragma unroll
      for (int i = 0; i < 64; ++i) v[i] = __uint_as_float(__float_as_uint(v[i]) ^ (acc & 1));
    }
  }
  float s = sm[0].x + sm[1].y + sm[2].x + sm[3].y;
#pragma unroll
  for (int i = 0; i < 64; ++i) s += v[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc ^ __float_as_uint(s);
}
int main() {
  uint32_t* o;
  cudaMalloc(&o, 148 * 1024 * 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const char* names[11] = {"ex2 (elem)", "f2fp pack (pair)", "ffma2 (pair)", "softmax step (elem)",
                          "step emu 1/8 (elem)", "step emu 2/8 (elem)", "step emu 3/8 (elem)", "step emu 4/8 (elem)",
                          "ex2.f16x2 (pair)", "", "step, prmt pack (elem)"};
  for (int op = 0; op < 11; ++op) {
    if (op == 9) continue;
    for (int th : {128, 256, 512}) {
      const int iters = 512;
      float ms = 0;
      for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        if (op == 0) k<0><<<148, th>>>(o, iters, 1e-3f);
        else if (op == 1) k<1><<<148, th>>>(o, iters, 1e-3f);
        else if (op == 2) k<2><<<148, th>>>(o, iters, 1e-3f);
        else if (op == 3) k<3><<<148, th>>>(o, iters, 1e-3f);
        else if (op == 4) k<4><<<148, th>>>(o, iters, 1e-3f);
        else if (op == 5) k<5><<<148, th>>>(o, iters, 1e-3f);
        else if (op == 6) k<6><<<148, th>>>(o, iters, 1e-3f);
        else if (op == 7) k<7><<<148, th>>>(o, iters, 1e-3f);
        else if (op == 8) k<8><<<148, th>>>(o, iters, 1e-3f);
        else k<10><<<148, th>>>(o, iters, 1e-3f);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
      }
      const double per_thread = op == 0 || (op >= 3 && op <= 7) || op >= 9 ? 64.0 : 32.0;
      const double ops = 148.0 * th * iters * per_thread;
      printf("%-22s warps/SMSP=%d: %.3f ms  %.2f per clk per SM (at %.0f MHz)\n", names[op], th / 128, ms,
             ops / (ms * 1e-3) / (clk * 1e3) / 148, clk / 1e3);
    }
  }
}
