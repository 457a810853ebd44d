// cy_comm.cu -- device-side synchronisation between the ranks of a multi-GPU job that share
// memory through peer mappings (CUDA IPC over NVLink / NVSwitch), for the fused replication path
// (cy_gemm_replicated; BASELINE configs[4] "M-sharded ... + all-gather").
//
// The replicated-D protocol of paper_2504_07004_b200/dist.py is, per call and on every rank's
// stream:  cy_peer_barrier (every peer has finished reading the previous result: write-after-read)
//       -> cy_gemm_replicated (the epilogue stores each tile into every rank's D)
//       -> cy_peer_barrier (every peer's stores have landed: read-after-write).
// The barrier is stream-ordered and never touches the host, so the whole exchange stays on the
// GPU; no NCCL call sits on this path.
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>

#include "cypress_b200.h"

namespace cy_internal {
void note_launch();  // cy_gemm.cu: the library-wide launch counter behind cy_launch_count()
}

namespace {

constexpr int kMaxRanks = 8;
struct PeerFlags {
  uint32_t* f[kMaxRanks];  // f[j]: rank j's flag array (kMaxRanks slots), mapped into this process
};

// Barrier timeout: a peer that never arrives (crashed rank) traps after ~60 s instead of hanging
// the GPU; the fault then surfaces on the stream.
constexpr uint64_t kTimeoutNs = 60ull * 1000 * 1000 * 1000;

__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Thread j < world: publish "rank has reached epoch" in rank j's slot `rank`, then wait until rank
// j has published the same epoch in our slot `j`.  The system-scope fence orders every store this
// device made before the barrier (the GEMM's peer stores: it precedes us in stream order and, as
// this kernel is launched without programmatic serialisation, has completed) before the flag.
__global__ void __launch_bounds__(32) peer_barrier_kernel(PeerFlags pf, int world, int rank, uint32_t epoch) {
  const int j = threadIdx.x;
  if (j < world) {
    asm volatile("fence.sc.sys;" ::: "memory");
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(pf.f[j] + rank), "r"(epoch) : "memory");
    const uint32_t* mine = pf.f[rank] + j;
    const uint64_t t0 = globaltimer();
    for (uint32_t spins = 0;; ++spins) {
      uint32_t v;
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(mine) : "memory");
      if (static_cast<int32_t>(v - epoch) >= 0) break;  // wrap-safe: epochs only grow
      if ((spins & 1023u) == 0 && globaltimer() - t0 > kTimeoutNs) __trap();
      __nanosleep(64);
    }
  }
  __syncwarp();
}

}  // namespace

extern "C" cy_status_t cy_peer_barrier(uint32_t* const* flags, int world, int rank, uint32_t epoch, void* stream) {
  if (!flags || world < 1 || world > kMaxRanks || rank < 0 || rank >= world || epoch == 0) return CY_ERR_INVALID_VALUE;
  PeerFlags pf{};
  for (int j = 0; j < world; ++j) {
    if (!flags[j]) return CY_ERR_INVALID_VALUE;
    if (reinterpret_cast<uintptr_t>(flags[j]) & 3u) return CY_ERR_MISALIGNED;
    pf.f[j] = flags[j];
  }
  peer_barrier_kernel<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(pf, world, rank, epoch);
  if (cudaGetLastError() != cudaSuccess) return CY_ERR_LAUNCH;
  cy_internal::note_launch();
  return CY_OK;
}
