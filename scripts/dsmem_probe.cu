// dsmem_probe.cu -- DSMEM bandwidth between the two CTAs of a cluster on B200, three ways:
//   1. bulk: cp.async.bulk.shared::cluster.shared::cta (TMA engine) CTA 1 -> CTA 0, mbarrier completion
//   2. st:   st.shared::cluster.v4 by 256 threads of CTA 1 into CTA 0
//   3. ld:   ld.shared::cluster.v4 by 256 threads of CTA 0 from CTA 1
// Each moves BYTES per repetition; cycles from clock64 on the measuring CTA.  Launched with one
// cluster per SM pair over all SMs (so every SM pair is busy, as in a split-K reduction).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/dsmem scripts/dsmem_probe.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdint>

namespace cg = cooperative_groups;
constexpr int BYTES = 96 * 1024;
constexpr int CHUNK = 16 * 1024;
constexpr int REPS = 20;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(256, 1) probe(int mode, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar;
  cg::cluster_group cl = cg::this_cluster();
  const unsigned rank = cl.block_rank();
  const uint32_t base = smem_u32(sm);
  const uint32_t b = smem_u32(&bar);
  for (int i = threadIdx.x; i < BYTES / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = i + rank;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  cl.sync();
  uint32_t remote_base, remote_bar;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote_base) : "r"(base), "r"(rank ^ 1u));
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote_bar) : "r"(b), "r"(rank ^ 1u));
  long long t0 = clock64();
  uint32_t phase = 0;
  for (int r = 0; r < REPS; ++r) {
    if (mode == 0) {
      if (rank == 0 && threadIdx.x == 0)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(BYTES) : "memory");
      cl.sync();
      if (rank == 1 && threadIdx.x == 0)
        for (int c = 0; c < BYTES; c += CHUNK)
          asm volatile(
              "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                  remote_base + c),
              "r"(base + c), "r"(CHUNK), "r"(remote_bar)
              : "memory");
      if (rank == 0) {
        uint32_t done = 0;
        while (!done)
          asm volatile(
              "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
              : "=r"(done)
              : "r"(b), "r"(phase)
              : "memory");
        phase ^= 1;
      }
      cl.sync();
    } else if (mode == 1) {
      if (rank == 1)
        for (int i = threadIdx.x * 16; i < BYTES; i += blockDim.x * 16)
          asm volatile("st.shared::cluster.v4.u32 [%0], {%1, %1, %1, %1};" ::"r"(remote_base + i), "r"(r) : "memory");
      cl.sync();
    } else {
      uint32_t acc = 0;
      if (rank == 0)
        for (int i = threadIdx.x * 16; i < BYTES; i += blockDim.x * 16) {
          uint32_t x, y, z, w;
          asm volatile("ld.shared::cluster.v4.u32 {%0, %1, %2, %3}, [%4];"
                       : "=r"(x), "=r"(y), "=r"(z), "=r"(w)
                       : "r"(remote_base + i)
                       : "memory");
          acc += x ^ y ^ z ^ w;
        }
      if (acc == 0xdeadbeef) out[1] = acc;
      cl.sync();
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0 && rank == 0 && blockIdx.x == 0) out[0] = (unsigned long long)(t1 - t0);
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 16);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, BYTES);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const char* names[3] = {"bulk cp.async.bulk (TMA) CTA1->CTA0", "st.shared::cluster.v4 (256 thr)", "ld.shared::cluster.v4 (256 thr)"};
  for (int mode = 0; mode < 3; ++mode) {
    for (int grid : {2, sms}) {
      probe<<<grid, 256, BYTES>>>(mode, d);
      probe<<<grid, 256, BYTES>>>(mode, d);
      cudaError_t e = cudaDeviceSynchronize();
      unsigned long long cyc = 0;
      cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
      printf("%-40s grid %3d: %s %.1f B/clk (incl. %d cluster syncs)\n", names[mode], grid,
             e == cudaSuccess ? "ok" : cudaGetErrorString(e), double(BYTES) * REPS / double(cyc), REPS * (mode == 0 ? 2 : 1));
    }
  }
  return 0;
}
