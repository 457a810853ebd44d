// cy_attention.cu -- forward attention (paper Sec. 5.3: the Flash
// Attention 2/3 forward kernels Cypress compiles, FP16, HeadDim 128) on sm_100a.
//
//   S = scale * Q K^T,  P = softmax_rows(S) (causal: key j <= query i),  O = P V,  lse = log sum exp S
//
// One CTA per (128-row query tile, batch*head).  Warp roles:
//   warp 0      TMA producer: Q tile once, then K_j / V_j blocks (128 keys) into a 2-stage ring.
//   warp 1      tcgen05.mma issuer: S_j = Q K_j^T into one of two TMEM score buffers, then
//               O += P_j V_j into the TMEM output accumulator.  It issues S_{j+1} before waiting for
//               P_j, so the tensor core computes the next scores while the SIMT warps run the
//               softmax of block j -- the FA3 software pipeline expressed with two
//               TMEM score buffers instead of a register copy.
//   warps 2-5   softmax (thread = query row = TMEM lane): running row max / sum in the exp2 domain,
//               P_j (fp16/bf16) into shared memory in the MMA's K-major SW128 layout, rescale of
//               the O accumulator in TMEM when the row max grows (tcgen05.ld/st), and the final
//               O / l normalisation + TMA store and lse.
// TMEM: S0 [0,128) S1 [128,256) O [256,384).  Shared: Q 32 KB, K/V 2 x 64 KB, P 32 KB.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <atomic>
#include <cmath>
#include <cstring>
#include <mutex>

#include "cy_ptx.cuh"
#include "cypress_b200.h"

namespace cy_attn {
using namespace cy;

constexpr int D = 128;        // head dim (the paper's configuration)
constexpr int BQ = 128;       // query rows per CTA (TMEM lanes)
constexpr int BKV = 128;      // keys per block
constexpr int ATOM = 128 * 128;            // one SW128 atom column: 128 rows x 64 elements x 2 B
constexpr int TILE = 2 * ATOM;             // 128 rows x 128 elements
constexpr int SQ_OFF = 0;
constexpr int SK_OFF = TILE;               // [2]
constexpr int SV_OFF = 3 * TILE;           // [2]
constexpr int SP_OFF = 5 * TILE;
constexpr int BAR_OFF = 6 * TILE;
constexpr int SMEM_BYTES = 1024 + 6 * TILE + 256;
constexpr int THREADS = 6 * 32;
constexpr uint32_t TM_S0 = 0, TM_O = 256;

template <int DT>
struct Types;

struct Params {
  int sq, sk, bh;
  int causal;
  float scale_log2;  // scale * log2(e)
  float* lse;        // [bh, sq] natural-log lse, or null
};

template <int DT, bool B_MN>
__host__ __device__ constexpr uint32_t idesc() {
  // f32 accumulate, a/b format, a K-major, b K-major (S) or MN-major (PV), N = 128, M = 128
  return (1u << 4) | (uint32_t(DT) << 7) | (uint32_t(DT) << 10) | ((B_MN ? 1u : 0u) << 16) | (uint32_t(128 >> 3) << 17) |
         (uint32_t(128 >> 4) << 24);
}

__device__ __forceinline__ void tmem_st_32x32b_x32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, "
      "%17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
      "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]),
      "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]),
      "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}
// D[tmem] (+)= A[tmem] * B[smem desc]: kind::f16, cta_group::1, A (K-major) read from tensor memory
__device__ __forceinline__ void mma_f16_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc,
                                           uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

template <int DT>
__device__ __forceinline__ uint32_t pack2(float lo, float hi) {
  if constexpr (DT == 0) {
    __half2 h = __floats2half2_rn(lo, hi);
    return *reinterpret_cast<uint32_t*>(&h);
  } else {
    __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<uint32_t*>(&h);
  }
}

template <int DT>
__global__ void __launch_bounds__(THREADS, 1)
    attn_fwd_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                    const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmO,
                    const Params p) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  const uint32_t sQ = base + SQ_OFF, sK = base + SK_OFF, sV = base + SV_OFF, sP = base + SP_OFF;
  const uint32_t bar = base + BAR_OFF;
  const uint32_t bQFull = bar, bKVFull = bar + 8, bKVEmpty = bar + 24, bSFull = bar + 40, bSEmpty = bar + 56,
                 bPReady = bar + 72, bOReady = bar + 80, sTmemSlot = bar + 96;
  volatile uint32_t* tmem_slot = reinterpret_cast<volatile uint32_t*>(smem_raw + (sTmemSlot - raw));

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // heavy (long) causal tiles first
  const int qt = p.causal ? (gridDim.x - 1 - blockIdx.x) : blockIdx.x;
  const int hb = blockIdx.y;
  const int q0 = qt * BQ;
  const int kv_end = p.causal ? min(p.sk, q0 + BQ) : p.sk;
  const int nkv = (kv_end + BKV - 1) / BKV;

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmQ);
    prefetch_tmap(&tmK);
    prefetch_tmap(&tmV);
    prefetch_tmap(&tmO);
    mbar_init(bQFull, 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(bKVFull + 8 * s, 1);
      mbar_init(bKVEmpty + 8 * s, 1);
      mbar_init(bSFull + 8 * s, 1);
      mbar_init(bSEmpty + 8 * s, 4);
    }
    mbar_init(bPReady, 4);
    mbar_init(bOReady, 1);
    fence_mbar_init();
  }
  if (warp == 1) {
    tmem_alloc<1>(sTmemSlot, 512);
    tmem_relinquish<1>();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();
  if (threadIdx.x == 0) pdl_launch_dependents();

  if (warp == 0) {
    // ---------------------------------------------------------------- producer
    if (lane == 0 && nkv > 0) {
      const uint64_t pol = policy_evict_last();
      mbar_arrive_expect_tx(bQFull, TILE);
      tma_load_3d(sQ, &tmQ, bQFull, 0, q0, hb, pol);
      tma_load_3d(sQ + ATOM, &tmQ, bQFull, 64, q0, hb, pol);
      for (int j = 0; j < nkv; ++j) {
        const int s = j & 1;
        mbar_wait(bKVEmpty + 8 * s, ((j >> 1) & 1) ^ 1);
        mbar_arrive_expect_tx(bKVFull + 8 * s, 2 * TILE);
        const int k0 = j * BKV;
        tma_load_3d(sK + s * TILE, &tmK, bKVFull + 8 * s, 0, k0, hb, pol);
        tma_load_3d(sK + s * TILE + ATOM, &tmK, bKVFull + 8 * s, 64, k0, hb, pol);
        tma_load_3d(sV + s * TILE, &tmV, bKVFull + 8 * s, 0, k0, hb, pol);
        tma_load_3d(sV + s * TILE + ATOM, &tmV, bKVFull + 8 * s, 64, k0, hb, pol);
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer
    if (lane == 0 && nkv > 0) {
      constexpr uint32_t ID_S = idesc<DT, false>(), ID_PV = idesc<DT, true>();
      auto issue_s = [&](int j) {
        const int s = j & 1;
        const uint32_t k = sK + s * TILE;
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t off = (kk >> 2) * ATOM + (kk & 3) * 32;
          mma_f16<1>(tmem + TM_S0 + s * 128, sdesc_sw128(sQ + off, 16, 1024), sdesc_sw128(k + off, 16, 1024), ID_S,
                     kk > 0);
        }
        mma_commit<1>(bSFull + 8 * s, 0);
      };
      mbar_wait(bQFull, 0);
      mbar_wait(bKVFull, 0);
      tc_fence_after();
      issue_s(0);
      for (int j = 0; j < nkv; ++j) {
        const int s = j & 1;
        if (j + 1 < nkv) {  // next scores while the softmax of block j runs
          const int s1 = (j + 1) & 1;
          mbar_wait(bKVFull + 8 * s1, ((j + 1) >> 1) & 1);
          // S buffer s1 held P_{j-1}; PV_{j-1} was issued before this MMA and tcgen05 ops execute
          // in issue order, so the overwrite is safe without a barrier.
          tc_fence_after();
          issue_s(j + 1);
        }
        mbar_wait(bPReady, j & 1);
        tc_fence_after();
        const uint32_t v = sV + s * TILE;
        // O += P_j V_j with P_j read from TMEM (packed 16-bit pairs over the S_j buffer, 8 columns
        // per k16 step) and V_j from shared memory (MN-major)
#pragma unroll
        for (int kk = 0; kk < BKV / 16; ++kk)
          mma_f16_ts(tmem + TM_O, tmem + TM_S0 + s * 128 + kk * 8, sdesc_sw128(v + kk * 2048, ATOM, 1024), ID_PV,
                     (j | kk) != 0);
        mma_commit<1>(bOReady, 0);
        mma_commit<1>(bKVEmpty + 8 * s, 0);
      }
    }
  } else {
    // ---------------------------------------------------------------- softmax / correction / epilogue
    const int q = warp & 3;
    const int r = 32 * q + lane;  // query row within the tile = TMEM lane
    const int qrow = q0 + r;
    const uint32_t lane_base = uint32_t(32 * q) << 16;
    float m = -INFINITY, l = 0.f;
    for (int j = 0; j < nkv; ++j) {
      const int s = j & 1;
      mbar_wait(bSFull + 8 * s, (j >> 1) & 1);
      tc_fence_after();
      const uint32_t tS = tmem + lane_base + TM_S0 + s * 128;
      const int key0 = j * BKV;
      const bool full_block = (key0 + BKV <= p.sk) && (!p.causal || key0 + BKV - 1 <= q0);
      // key validity only matters in the last (ragged) block and in the causal diagonal block
      auto valid = [&](int key) { return full_block || (key < p.sk && (!p.causal || key <= qrow)); };
      // S_j row -> registers (one TMEM read), masked keys -> -inf
      uint32_t v[128];
#pragma unroll
      for (int c = 0; c < 4; ++c) tmem_ld_32x32b_x32(tS + 32 * c, *reinterpret_cast<uint32_t(*)[32]>(&v[32 * c]));
      tmem_ld_wait();
      if (!full_block) {
#pragma unroll
        for (int e = 0; e < 128; ++e)
          if (!valid(key0 + e)) v[e] = __float_as_uint(-INFINITY);
      }
      float mx8[8];
#pragma unroll
      for (int t = 0; t < 8; ++t) mx8[t] = -INFINITY;
#pragma unroll
      for (int e = 0; e < 128; ++e) mx8[e & 7] = fmaxf(mx8[e & 7], __uint_as_float(v[e]));
      float mb = fmaxf(fmaxf(fmaxf(mx8[0], mx8[1]), fmaxf(mx8[2], mx8[3])),
                       fmaxf(fmaxf(mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7])));
      mb = (mb == -INFINITY) ? -INFINITY : mb * p.scale_log2;  // scale_log2 > 0 keeps the order
      // Lazy rescaling: keep the running max unless it grows by more than 2^8 (P <= 256 stays exact
      // in the 16-bit types and the fp32 sums); the final O / l uses the same max, so this is exact.
      float m_new = m, corr = 1.f;
      if (mb > m + 8.f) {
        m_new = mb;
        corr = ex2(m - m_new);  // 0 when m == -inf
      }
      const float msub = (m_new == -INFINITY) ? 0.f : m_new;
      if (j > 0 && __any_sync(0xffffffffu, corr != 1.f)) {
        mbar_wait(bOReady, (j - 1) & 1);  // O holds PV_{j-1}
        tc_fence_after();
        const uint32_t tO = tmem + lane_base + TM_O;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          uint32_t o[32];
          tmem_ld_32x32b_x32(tO + 32 * c, o);
          tmem_ld_wait();
#pragma unroll
          for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * corr);
          tmem_st_32x32b_x32(tO + 32 * c, o);
        }
      }
      // P = exp2(s * scale_log2 - m) -> packed 16-bit pairs written back over S_j (TMEM cols 0..63)
      float sm8[8];
#pragma unroll
      for (int t = 0; t < 8; ++t) sm8[t] = 0.f;
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        uint32_t pk[32];
#pragma unroll
        for (int e = 0; e < 32; ++e) {
          const float p0 = ex2(fmaf(__uint_as_float(v[64 * c + 2 * e]), p.scale_log2, -msub));
          const float p1 = ex2(fmaf(__uint_as_float(v[64 * c + 2 * e + 1]), p.scale_log2, -msub));
          sm8[(2 * e) & 7] += p0;
          sm8[(2 * e + 1) & 7] += p1;
          pk[e] = pack2<DT>(p0, p1);
        }
        tmem_st_32x32b_x32(tS + 32 * c, pk);
      }
      tmem_st_wait();
      const float sum = ((sm8[0] + sm8[1]) + (sm8[2] + sm8[3])) + ((sm8[4] + sm8[5]) + (sm8[6] + sm8[7]));
      l = l * corr + sum;
      m = m_new;
      tc_fence_before();  // P and the rescaled O (tcgen05.st) before the MMA issuer's PV_j
      __syncwarp();
      if (lane == 0) mbar_arrive(bPReady);
    }
    // ---------------------------------------------------------------- epilogue: O / l, lse
    const float inv_l = (l > 0.f) ? 1.f / l : 0.f;
    if (nkv > 0) {
      mbar_wait(bOReady, (nkv - 1) & 1);
      tc_fence_after();
    }
    const uint32_t sE = sP + q * 4096;  // P is no longer read: 4 KB staging per warp
#pragma unroll 1
    for (int c = 0; c < 2; ++c) {
      uint32_t a0[32], a1[32];
      if (nkv > 0) {
        const uint32_t tO = tmem + lane_base + TM_O + 64 * c;
        tmem_ld_32x32b_x32(tO, a0);
        tmem_ld_32x32b_x32(tO + 32, a1);
        tmem_ld_wait();
      } else {
#pragma unroll
        for (int e = 0; e < 32; ++e) a0[e] = a1[e] = 0u;
      }
      if (lane == 0 && c > 0) bulk_wait_read<0>();
      __syncwarp();
#pragma unroll
      for (int v = 0; v < 8; ++v) {
        uint32_t w[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int col = 8 * v + 2 * u;
          const float x0 = __uint_as_float(col < 32 ? a0[col] : a1[col - 32]) * inv_l;
          const float x1 = __uint_as_float(col + 1 < 32 ? a0[col + 1] : a1[col + 1 - 32]) * inv_l;
          w[u] = pack2<DT>(x0, x1);
        }
        st_shared_v4(sE + lane * 128 + ((v ^ (lane & 7)) << 4), w[0], w[1], w[2], w[3]);
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        tma_store_3d(&tmO, sE, 64 * c, q0 + 32 * q, hb);
        bulk_commit();
      }
    }
    if (p.lse && qrow < p.sq)
      p.lse[(size_t)hb * p.sq + qrow] = (l > 0.f) ? (m + __log2f(l)) * 0.6931471805599453f : -INFINITY;
    if (lane == 0) bulk_wait_read<0>();
  }
  __syncwarp();
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<1>(tmem, 512);
  }
}

// ------------------------------------------------------------------------------------------ host
std::once_flag g_once;
PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
std::mutex g_attr_mu;
bool g_attr_set[64][2] = {};

bool make_map(CUtensorMap* m, int dt, const void* ptr, uint64_t rows, uint64_t bh, uint32_t box_c, uint32_t box_r) {
  cuuint64_t dims[3] = {uint64_t(D), rows, bh};
  cuuint64_t strides[2] = {uint64_t(D) * 2, rows * uint64_t(D) * 2};
  cuuint32_t box[3] = {box_c, box_r, 1};
  cuuint32_t es[3] = {1, 1, 1};
  return g_encode(m, dt == 0 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3,
                  const_cast<void*>(ptr), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace cy_attn

extern "C" cy_status_t cy_attention_fwd(cy_dtype_t dt, int64_t batch, int64_t heads, int64_t seq_q, int64_t seq_k,
                                        int64_t head_dim, float scale, int causal, const void* Q, const void* K,
                                        const void* V, void* O, float* lse, void* stream) {
  using namespace cy_attn;
  if (dt != CY_F16 && dt != CY_BF16) return CY_ERR_INVALID_VALUE;
  if (batch < 0 || heads < 0 || seq_q < 0 || seq_k < 0) return CY_ERR_INVALID_VALUE;
  if (head_dim != D) return CY_ERR_INVALID_VALUE;  // HeadDim 128
  const int64_t bh = batch * heads;
  if (bh == 0 || seq_q == 0) return CY_OK;
  if (!Q || !O || (seq_k > 0 && (!K || !V))) return CY_ERR_INVALID_VALUE;
  if (seq_q > INT32_MAX || seq_k > INT32_MAX || bh > 65535) return CY_ERR_INVALID_VALUE;
  auto al = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; };
  if (!al(Q) || !al(O) || (seq_k > 0 && (!al(K) || !al(V))) || (lse && (reinterpret_cast<uintptr_t>(lse) & 3u)))
    return CY_ERR_MISALIGNED;
  {  // O must not overlap the inputs
    const uintptr_t o0 = reinterpret_cast<uintptr_t>(O), o1 = o0 + size_t(bh * seq_q * D * 2);
    for (const void* in : {Q, K, V}) {
      if (!in) continue;
      const uintptr_t i0 = reinterpret_cast<uintptr_t>(in);
      const uintptr_t i1 = i0 + size_t(bh * (in == Q ? seq_q : seq_k) * D * 2);
      if (i0 < o1 && o0 < i1) return CY_ERR_INVALID_VALUE;
    }
  }
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return CY_ERR_UNSUPPORTED_DEVICE;
  int major = 0, minor = 0;
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
  if (major != 10 || minor != 0) return CY_ERR_UNSUPPORTED_DEVICE;
  std::call_once(g_once, [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  });
  if (!g_encode) return CY_ERR_INTERNAL;
  CUtensorMap tQ, tK, tV, tO;
  std::memset(&tK, 0, sizeof(tK));
  tV = tK;
  bool ok = make_map(&tQ, dt, Q, seq_q, bh, 64, 128) && make_map(&tO, dt, O, seq_q, bh, 64, 32);
  if (seq_k > 0) ok = ok && make_map(&tK, dt, K, seq_k, bh, 64, 128) && make_map(&tV, dt, V, seq_k, bh, 64, 128);
  if (!ok) return CY_ERR_LAUNCH;
  Params p;
  p.sq = (int)seq_q;
  p.sk = (int)seq_k;
  p.bh = (int)bh;
  p.causal = causal ? 1 : 0;
  p.scale_log2 = scale * 1.4426950408889634f;
  p.lse = lse;
  const void* fn = dt == CY_F16 ? (const void*)&attn_fwd_kernel<0> : (const void*)&attn_fwd_kernel<1>;
  {
    std::lock_guard<std::mutex> lk(g_attr_mu);
    if (!g_attr_set[dev][dt]) {
      if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES) != cudaSuccess) {
        cudaGetLastError();
        return CY_ERR_LAUNCH;
      }
      g_attr_set[dev][dt] = true;
    }
  }
  cudaLaunchConfig_t cfg;
  std::memset(&cfg, 0, sizeof(cfg));
  cfg.gridDim = dim3((unsigned)((seq_q + BQ - 1) / BQ), (unsigned)bh, 1);
  cfg.blockDim = dim3(THREADS, 1, 1);
  cfg.dynamicSmemBytes = SMEM_BYTES;
  cfg.stream = static_cast<cudaStream_t>(stream);
  cudaLaunchAttribute attrs[1];
  attrs[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attrs[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attrs;
  cfg.numAttrs = 1;
  void* args[] = {&tQ, &tK, &tV, &tO, &p};
  if (cudaLaunchKernelExC(&cfg, fn, args) != cudaSuccess) {
    cudaGetLastError();
    return CY_ERR_LAUNCH;
  }
  return CY_OK;
}
