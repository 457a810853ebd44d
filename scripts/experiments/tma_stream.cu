// TMA streaming probe: every CTA (one per SM) loads 16 KB boxes (64 x 128 fp16, SWIZZLE_128B) of an
// L2-resident matrix into a ring of S stages, as fast as the ring allows, for ITERS boxes.  Modes:
//   0 distinct: CTA c reads its own rows (no two SMs touch the same line)
//   1 shared-4: groups of 4 consecutive CTAs read the same rows at the same time
//   2 shared-all: every CTA reads the same rows
// Prints delivered bytes per SM-cycle (aggregate and per SM).  nvcc -arch=sm_100a -o tma_stream tma_stream.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__global__ void __launch_bounds__(32, 1) k(const __grid_constant__ CUtensorMap tm, int iters, int stages, int mode,
                                           int rows_total, unsigned long long* cyc, int br, int nb, int d3) {
  extern __shared__ __align__(1024) uint8_t sm[];
  const uint32_t base = (su32(sm) + 1023u) & ~1023u;
  const uint32_t bars = base + 6 * 32768;  // (64 KB stages: 3)
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bars + 8 * s));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncwarp();
  const int grp = mode == 0 ? blockIdx.x : mode == 1 ? blockIdx.x / 4 : 0;
  const long long t0 = clock64();
  {  // whole warp, converged; TMA and expect_tx elect.sync-predicated (the product kernels' form)
    for (int i = 0; i < iters + stages; ++i) {
      const int s = i % stages;
      if (i >= stages) {  // wait for the stage issued `stages` ago
        asm volatile("{\n\t.reg .pred p;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W;\n\t}" ::"r"(bars + 8 * s),
                     "r"(((i - stages) / stages) & 1));
      }
      if (i < iters) {
        asm volatile("{\n\t.reg .pred ep;\n\telect.sync _|ep, 0xffffffff;\n\t@ep mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n\t}" ::"r"(bars + 8 * s), "r"(d3 >= 2 ? 65536 : 32768));
        if (d3) {  // 3-D boxes {64 cols, 64 rows, atoms}
          const int row = ((grp * 4 + i) * 128) % rows_total;
          const uint32_t ssz = d3 == 1 ? 32768 : 65536;
          for (int bb = 0; bb < (d3 == 3 ? 2 : 1); ++bb)
            asm volatile("{\n\t.reg .pred ep;\n\telect.sync _|ep, 0xffffffff;\n\t@ep cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n\t}" ::"r"(
                             base + s * ssz + bb * 32768),
                         "l"(&tm), "r"(0), "r"(row), "r"(bb * 4), "r"(bars + 8 * s)
                         : "memory");
        }
        for (int b = 0; b < (d3 ? 0 : nb); ++b) {
          const int row = ((grp * 4 + i) * 128 + b * br) % rows_total;
          asm volatile("{\n\t.reg .pred ep;\n\telect.sync _|ep, 0xffffffff;\n\t@ep cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n\t}" ::"r"(
                           base + s * 32768 + b * br * 128),
                       "l"(&tm), "r"(0), "r"(row), "r"(bars + 8 * s)
                       : "memory");
        }
      }
    }
  }
  if (threadIdx.x == 0) {
    cyc[blockIdx.x] = clock64() - t0;
  }
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int rows = 8192 * 2, cols = 64;  // 2 MB of fp16 rows (64 cols) -> L2-resident
  void* buf; cudaMalloc(&buf, (size_t)rows * cols * 2 * 8);
  cudaMemset(buf, 0, (size_t)rows * cols * 2 * 8);
  auto mk = [&](CUtensorMap* tm, int br) {
    cuuint64_t dims[2] = {(cuuint64_t)cols * 8, (cuuint64_t)rows};  // 512 cols wide rows (1 KB)
    cuuint64_t strides[1] = {(cuuint64_t)cols * 8 * 2};
    cuuint32_t box[2] = {64, (cuuint32_t)br}, es[2] = {1, 1};
    return cuTensorMapEncodeTiled(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                  CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
  };
  unsigned long long* cyc; cudaMalloc(&cyc, sizeof(unsigned long long) * 1024);
  const int smem = 6 * 32768 + 1024 + 256;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 4096;
  auto mk3 = [&](CUtensorMap* tm, int atoms3) {  // {64 cols, rows, 8 atoms of 64 cols}: box {64, 64, 4} = 4 atoms x 64 rows
    cuuint64_t dims[3] = {64, (cuuint64_t)rows, 8};
    cuuint64_t strides[2] = {(cuuint64_t)cols * 8 * 2, 128};
    cuuint32_t box[3] = {64, 64, (cuuint32_t)atoms3}, es[3] = {1, 1, 1};
    return cuTensorMapEncodeTiled(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                  CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
  };
  for (int cfg = 0; cfg < 5; ++cfg)
    for (int stages : {3}) for (int nct : {1, 148}) {
      // cfg 0: four 2-D boxes 64 x 64 per 32 KB stage; 1: one 3-D box 64 x 64 x 4; 2: two 2-D boxes 64 x 128
      CUtensorMap tm;
      const int br = cfg == 2 ? 128 : 64, nb = cfg == 0 ? 4 : cfg == 2 ? 2 : 4, d3 = cfg == 1;
      const int big = cfg >= 3;  // 64 KB stages
      if (!(d3 || big ? mk3(&tm, cfg == 3 ? 8 : 4) : mk(&tm, br))) { printf("encode failed\n"); return 1; }
      const int d3m = d3 ? 1 : cfg == 3 ? 2 : cfg == 4 ? 3 : 0;
      k<<<nct, 32, smem>>>(tm, 64, stages, 0, rows, cyc, br, nb, d3m);
      k<<<nct, 32, smem>>>(tm, iters, stages, 0, rows, cyc, br, nb, d3m);
      if (cudaDeviceSynchronize() != cudaSuccess) { printf("launch failed: %s\n", cudaGetErrorString(cudaGetLastError())); return 1; }
      std::vector<unsigned long long> h(nct);
      cudaMemcpy(h.data(), cyc, sizeof(unsigned long long) * nct, cudaMemcpyDeviceToHost);
      unsigned long long mx = 0; for (auto v : h) mx = v > mx ? v : mx;
      const double per_sm = (cfg >= 3 ? 65536.0 : 32768.0) * iters / mx;
      printf("cfg %d (%s), 32 KB stages %d, ctas %3d: %6.1f B/clk per SM, %7.0f B/clk total\n", cfg,
             cfg == 0 ? "4 x 2-D 64x64" : cfg == 1 ? "1 x 3-D 64x64x4" : cfg == 2 ? "2 x 2-D 64x128" : cfg == 3 ? "1 x 3-D 64x64x8 (64K)" : "2 x 3-D 64x64x4 (64K)", stages, nct, per_sm, per_sm * nct);
    }
  return 0;
}
