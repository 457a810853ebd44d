// cy_attention.cu -- forward attention (paper Sec. 5.3: the Flash
// Attention 2/3 forward kernels Cypress compiles, FP16, HeadDim 128) on sm_100a.
//
//   S = scale * Q K^T,  P = softmax_rows(S) (causal: key j <= query i),  O = P V,  lse = log sum exp S
//
// attn_fwd_kernel (default layout CS = 3): one CTA per (two 128-row query tiles, batch*head),
// 12 warps (3 warpgroups; setmaxnreg moves registers to the softmax warpgroups).
//   warps 0-3, 4-7  softmax warpgroups of query tiles 0 and 1 (thread = query row = TMEM lane): per
//                   128-key block, one TMEM pass reads the row's 128 scores into registers, the row
//                   max is a balanced FMNMX3 tree, P = exp2(s*scale*log2e - m) in the exp2 domain is
//                   written back over S_t as 16-bit pairs (the first half published early so PV can
//                   start); lazy rescale of O_t in TMEM only when the max grows by more than 2^8;
//                   final O / l, TMA store, lse.
//   warp 8          TMA producer: both Q tiles once, then K_j (2-slot ring) and V_j (3-slot ring),
//                   each slot refilled as soon as its last reader is done.
//   warp 9          tcgen05.mma issuer, per block j and tile t: O_t += P_t V_j (A = P_t read from
//                   TMEM, in two halves), then S_t(j+1) = Q_t K_{j+1}^T.  While one warpgroup runs its
//                   softmax the tensor core runs the other tile's two GEMMs -- the FA3 ping-pong
//                    with TMEM in place of FA3's register copy of S; every K/V block
//                   serves 256 rows.  Warps 10-11 only donate registers.
//   TMEM: S_0 [0,128) S_1 [128,256) O_0 [256,384) O_1 [384,512).  Shared: Q 2 x 32 KB, K 2 x 32 KB,
//   V 3 x 32 KB.  CS = 1 (10 warps, two TMEM passes) and CS = 2 (two warps per row, both tiles in
//   turn) are the earlier layouts, kept as tested variants.
// attn_pair_kernel (CY_ATTN_KERNEL=2): a CTA pair issuing cta_group::2 MMAs with double-buffered
//   S and a separate P in TMEM (see its own comment); correct, measured slower.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <type_traits>

#include "cy_ptx.cuh"
#include "cypress_b200.h"

namespace cy_internal {
void note_launch();  // cy_gemm.cu: the library-wide launch counter behind cy_launch_count()
}

namespace cy_attn {
using namespace cy;

#ifndef CY_ATTN_PH_E
#define CY_ATTN_PH_E 7
#endif
// Build knobs of the CS = 3 kernel (experiments; the defaults are the measured best):
// CY_ATTN_PH_E: pair index of the second P group after which the first half of P_t is published.
// CY_ATTN_PP: softmax ping-pong: 0 off; 1 the two tiles' exponential passes strictly alternate (named
// barriers 8 / 9); 2 the whole per-block softmax alternates.  Measured: 1 on par, 2 -5 %.
#ifndef CY_ATTN_PP
#define CY_ATTN_PP 0
#endif
// CY_ATTN_PF: K/V L2 prefetch distance in blocks (0 = off).  A K/V tile takes ~4-5 K cycles from
// TMA issue to full barrier inside the kernel (CY_ATTN_TRACE), but that is the closed loop of the
// rings, not L2 latency: prefetching 2-6 blocks ahead measured -1..-2 %, and skipping the K/V
// reloads altogether (CY_ATTN_DBG_NOLOAD, invalid results) only +5 %.
#ifndef CY_ATTN_PF
#define CY_ATTN_PF 0
#endif
// CY_ATTN_SPEC: the CS = 3 softmax takes group 0's exponentials against the running max while it
// reduces the row max (the block is redone in the rare case a row's max grows past the lazy bound)
#ifndef CY_ATTN_SPEC
#define CY_ATTN_SPEC 1
#endif
// CY_ATTN_DB: the default path runs attn_db_kernel (64-key blocks, double-buffered S in TMEM)
#ifndef CY_ATTN_DB
#define CY_ATTN_DB 0
#endif
// CY_ATTN_T1: the default path runs attn_t1_kernel (one query tile per CTA, double-buffered S)
#ifndef CY_ATTN_T1
#define CY_ATTN_T1 0
#endif
// CY_ATTN_LPT: causal grids ordered heads-fastest, so the launch order is heaviest-first across the
// whole grid (every head's last query tiles, then the next ones ...) and the tail of the launch holds
// only the lightest CTAs.  Measured (scripts/attn_probe.py, two runs): causal 2x16x8192 1063 -> 1110
// TFLOP/s, 4x16x4096 963 -> 980, 16x16x1024 417-469 -> 468-519, 1x16x16384 on par to +8 %.
// (Non-causal grids keep query tiles fastest: concurrent CTAs of one head share its K / V in L2.)
#ifndef CY_ATTN_LPT
#define CY_ATTN_LPT 1
#endif
// CY_ATTN_TRACE (timing experiments only, never in the product build): clock64() stamps of one
// CTA's per-block events, read back with cy_attn_trace()
#ifdef CY_ATTN_TRACE
__device__ unsigned long long g_attn_trace[16 * 2 * 64];
#define ATRACE(cond, ev, t, j)                                                                       \
  do {                                                                                              \
    if ((cond) && blockIdx.x == 3 && blockIdx.y == 5 && (j) < 64) g_attn_trace[((ev) * 2 + (t)) * 64 + (j)] = clock64(); \
  } while (0)
#else
#define ATRACE(cond, ev, t, j) \
  do {                         \
  } while (0)
#endif
constexpr int D = 128;        // head dim (the paper's configuration)
constexpr int BQ = 128;       // query rows per tile (TMEM lanes)
constexpr int NT = 2;         // query tiles per CTA (two softmax warpgroups ping-pong on the tensor core)
constexpr int BKV = 128;      // keys per block
constexpr int ATOM = 128 * 128;            // one SW128 atom column: 128 rows x 64 elements x 2 B
constexpr int TILE = 2 * ATOM;             // 128 rows x 128 elements
constexpr int SQ_OFF = 0;                  // [NT]
constexpr int SK_OFF = NT * TILE;          // [2]
constexpr int SV_OFF = (NT + 2) * TILE;    // [2]
constexpr int BAR_OFF = (NT + 4) * TILE;
constexpr int XCH_OFF = BAR_OFF + 256;       // CS = 2: row-max exchange [NT][2][2][BQ], sums [NT][2][BQ]
[[maybe_unused]] constexpr int SMEM_BYTES = 1024 + (NT + 4) * TILE + 256 + (NT * 2 * 2 * BQ + NT * 2 * BQ) * 4;
// CS = 3 layout: V gets a third ring slot (a K/V tile load takes ~4-5 K cycles under load, longer than
// the lead two slots give); barriers after the last V slot, no exchange area
#ifndef CY_ATTN_VS3
#define CY_ATTN_VS3 3
#endif
constexpr int VS3 = CY_ATTN_VS3;
constexpr int BAR_OFF3 = (NT + 2 + VS3) * TILE;
constexpr int SMEM_BYTES3 = 1024 + BAR_OFF3 + 256;
static_assert(SMEM_BYTES3 <= 232448, "CS = 3 layout exceeds 227 KB");
constexpr int THREADS = (4 * NT + 2) * 32;  // softmax warpgroups 0..NT-1, then producer, MMA issuer
constexpr int W_PROD = 4 * NT, W_MMA = 4 * NT + 1;
constexpr uint32_t TM_S = 0, TM_O = 256;   // S_t at 128 t, O_t at 256 + 128 t

struct Params {
  int sq, sk, bh;
  int causal;
  float scale_log2;  // scale * log2(e)
  float* lse;        // [bh, sq] natural-log lse, or null
  int l2hint;        // 1: TMA loads carry an L2 evict_last hint; 0: no hint (requests can merge in L2)
  int lpt;           // causal, CY_ATTN_LPT: grid (batch*heads, query-tile pairs), heads fastest, so the launch
                     // order is globally heaviest-first (every head's last query tiles, then the next ...)
};

template <int DT, bool B_MN, int N = 128>
__host__ __device__ constexpr uint32_t idesc() {
  // f32 accumulate, a/b format, a K-major, b K-major (S) or MN-major (PV), N (128; 64 for the 64-key
  // S blocks of attn_db_kernel), M = 128
  return (1u << 4) | (uint32_t(DT) << 7) | (uint32_t(DT) << 10) | ((B_MN ? 1u : 0u) << 16) | (uint32_t(N >> 3) << 17) |
         (uint32_t(128 >> 4) << 24);
}

template <int N>
__device__ __forceinline__ void tmem_st_32x32b(uint32_t taddr, const uint32_t* r);
template <>
__device__ __forceinline__ void tmem_st_32x32b<16>(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
      "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}
__device__ __forceinline__ void tmem_st_32x32b_x32(uint32_t taddr, const uint32_t (&r)[32]) {
  tmem_st_32x32b<16>(taddr, r);
  tmem_st_32x32b<16>(taddr + 16, r + 16);
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
__device__ __forceinline__ void mma_f16_ts_e(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc,
                                             uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, ep;\n\tsetp.ne.b32 p, %4, 0;\n\t" CY_ELECT
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

// Blackwell 2-wide fp32 SIMD (FFMA2 / FADD2): two lanes of work per issued instruction; each lane
// rounds exactly like the scalar fma/add, so results are unchanged.
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  uint64_t d;
  asm("{.reg .b64 ra, rb, rc;\n\t"
      "mov.b64 ra, {%1, %2};\n\tmov.b64 rb, {%3, %4};\n\tmov.b64 rc, {%5, %6};\n\t"
      "fma.rn.f32x2 %0, ra, rb, rc;}"
      : "=l"(d) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  float2 r;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(d));
  return r;
}
__device__ __forceinline__ float2 fadd2(float2 a, float2 b) {
  uint64_t d;
  asm("{.reg .b64 ra, rb;\n\t"
      "mov.b64 ra, {%1, %2};\n\tmov.b64 rb, {%3, %4};\n\t"
      "add.rn.f32x2 %0, ra, rb;}"
      : "=l"(d) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  float2 r;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(d));
  return r;
}
__device__ __forceinline__ float2 fsub2(float2 a, float2 b) {
  uint64_t d;
  asm("{.reg .b64 ra, rb;\n\t"
      "mov.b64 ra, {%1, %2};\n\tmov.b64 rb, {%3, %4};\n\t"
      "sub.rn.f32x2 %0, ra, rb;}"
      : "=l"(d) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  float2 r;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(d));
  return r;
}

// 2^x for a pair on the FMA/ALU pipes only (no MUFU, no FRND/F2I, which issue on the XU pipe):
// n = rint(x) by the 1.5*2^23 magic add, f = x - n in [-1/2, 1/2], 2^f by a cubic fitted for
// minimax relative error on [-1/2, 1/2] (max 7.5e-5 in fp32, below the 2^-11 rounding of the
// 16-bit P it feeds), then n is added to the exponent field.  x is clamped at -126, so inputs
// below that return a value < 2^-125 instead of 0; callers only use it where no score is masked.
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

__device__ __forceinline__ int blocks_for(const Params& p, int row_end) {
  const int kv_end = p.causal ? min(p.sk, row_end) : p.sk;
  return (kv_end + BKV - 1) / BKV;
}

// EMU of every 8 exponential pairs are evaluated with ex2_emu2.  CS = 1: warpgroup t owns query
// tile t (one warp per row quarter); CS = 2: all 8 softmax warps work on each tile in turn, the
// two warps of a row quarter splitting its 128 scores (two warps per SM sub-partition per tile).
// CS = 3: like CS = 1, but the CTA has 12 warps (3 warpgroups) so that setmaxnreg can move
// registers to the softmax warpgroups (208 each; the producer / MMA warpgroup keeps 72) and each
// thread holds its whole 128-score row from a single TMEM pass.
template <int DT, int EMU, int CS = 1>
__global__ void __launch_bounds__(CS == 3 ? 384 : THREADS, 1)
    attn_fwd_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                    const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmO,
                    const Params p) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  const uint32_t sQ = base + SQ_OFF, sK = base + SK_OFF, sV = base + SV_OFF;
  constexpr int VS = (CS == 3) ? VS3 : 2;  // V ring slots
  const uint32_t bar = base + (CS == 3 ? BAR_OFF3 : BAR_OFF);
  // K and V have separate 2-slot rings: K_j is released after the last S(j), V_j after the last
  // PV(j), so each refill starts as soon as its own readers are done
  const uint32_t bQFull = bar, bKFull = bar + 8, bKEmpty = bar + 24, bSFull = bar + 72, bPReady = bar + 88,
                 bOReady = bar + 104, sTmemSlot = bar + 120;
  const uint32_t bVFull = (VS == 2) ? bar + 40 : bar + 144, bVEmpty = (VS == 2) ? bar + 56 : bar + 144 + 8 * VS;
  // CS = 3: P_t for keys [0, 64) of the block is published first (bPHalf), so the tensor core starts
  // the first half of PV_t(j) while the softmax warps still compute the second half of P_t
  const uint32_t bPHalf = bar + 128;
  volatile uint32_t* tmem_slot = reinterpret_cast<volatile uint32_t*>(smem_raw + (sTmemSlot - raw));

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // P_t columns inside S_t: CS = 1 writes P over columns [0, 64); CS = 2 over [32, 96), so each
  // half-row warp overwrites only score columns it has already read itself
  constexpr uint32_t P_COL = (CS == 2) ? 32 : 0;
  const int qt = p.lpt ? (gridDim.y - 1 - blockIdx.y) : p.causal ? (gridDim.x - 1 - blockIdx.x) : blockIdx.x;  // heavy causal CTAs first
  const int hb = p.lpt ? blockIdx.x : blockIdx.y;
  const int q0 = qt * BQ * NT;
  int nkv[NT];
#pragma unroll
  for (int t = 0; t < NT; ++t) nkv[t] = blocks_for(p, q0 + BQ * (t + 1));
  const int nall = nkv[NT - 1];  // tiles further down need at least as many blocks

  if (warp == W_PROD && lane == 0) {
    prefetch_tmap(&tmQ);
    prefetch_tmap(&tmK);
    prefetch_tmap(&tmV);
    prefetch_tmap(&tmO);
    mbar_init(bQFull, 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(bKFull + 8 * s, 1);
      mbar_init(bKEmpty + 8 * s, 1);
    }
    for (int s = 0; s < VS; ++s) {
      mbar_init(bVFull + 8 * s, 1);
      mbar_init(bVEmpty + 8 * s, 1);
    }
    for (int t = 0; t < NT; ++t) {
      mbar_init(bSFull + 8 * t, 1);
      mbar_init(bPReady + 8 * t, CS == 2 ? 8 : 4);
      mbar_init(bOReady + 8 * t, 1);
      mbar_init(bPHalf + 8 * t, 4);
    }
    fence_mbar_init();
  }
  if (warp == W_MMA) {
    tmem_alloc<1>(sTmemSlot, 512);
    tmem_relinquish<1>();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();
  pdl_launch_dependents();  // (every thread: keeps the warps provably converged, see cy_ptx.cuh)
  if (warp >= 4 * NT) {
  // CS = 3: whole warpgroups re-balance registers at the top of each role's branch (softmax
  // warpgroups up to 208, the producer / MMA / spare warpgroup down to 72)
  if constexpr (CS == 3) asm volatile("setmaxnreg.dec.sync.aligned.u32 72;\n" ::: "memory");
  if (warp == W_PROD) {
    // ---------------------------------------------------------------- producer
    if (nall > 0) {  // all 32 lanes, converged; TMA and expect_tx are elect.sync-predicated
      const uint64_t pol = policy_evict_last();
      // Q, K, V maps are 4-D {64, rows, 2 column atoms, batch*head}: a whole 128 x 128 tile (both
      // 64-column SW128 atoms, ATOM bytes apart) is one TMA op
      auto ld = [&](uint32_t dst, const CUtensorMap* tm, uint32_t bar, int row) {
        tma_load_4d_e(dst, tm, bar, 0, row, 0, hb, pol, p.l2hint != 0);
      };
      mbar_arrive_expect_tx_e(bQFull, NT * TILE);
      for (int t = 0; t < NT; ++t) ld(sQ + t * TILE, &tmQ, bQFull, q0 + BQ * t);
      auto prefetch_kv = [&](int jb) {
        if (jb < nall) {
          tma_prefetch_3d(&tmK, 0, jb * BKV, hb);
          tma_prefetch_3d(&tmK, 64, jb * BKV, hb);
          tma_prefetch_3d(&tmV, 0, jb * BKV, hb);
          tma_prefetch_3d(&tmV, 64, jb * BKV, hb);
        }
      };
      if constexpr (CY_ATTN_PF > 0)
        for (int jb = 2; jb < CY_ATTN_PF; ++jb) prefetch_kv(jb);
      for (int j = 0; j < nall; ++j) {
        const int s = j & 1;
        const int k0 = j * BKV;
        if constexpr (CY_ATTN_PF > 0)
          if (j + CY_ATTN_PF >= 2) prefetch_kv(j + CY_ATTN_PF);
        mbar_wait_w(bKEmpty + 8 * s, ((j >> 1) & 1) ^ 1);
        ATRACE(true, 8, 0, j);
#ifdef CY_ATTN_DBG_NOLOAD
        // timing experiment only (invalid results): K/V tiles after the first ring fill are not reloaded
        if (j >= 4) {
          mbar_arrive_e(bKFull + 8 * s);
          const int vs = j % VS;
          mbar_wait_w(bVEmpty + 8 * vs, ((j / VS) & 1) ^ 1);
          mbar_arrive_e(bVFull + 8 * vs);
          continue;
        }
#endif
        mbar_arrive_expect_tx_e(bKFull + 8 * s, TILE);
        ld(sK + s * TILE, &tmK, bKFull + 8 * s, k0);
        const int vs = j % VS;
        mbar_wait_w(bVEmpty + 8 * vs, ((j / VS) & 1) ^ 1);
        ATRACE(true, 9, 0, j);
        mbar_arrive_expect_tx_e(bVFull + 8 * vs, TILE);
        ld(sV + vs * TILE, &tmV, bVFull + 8 * vs, k0);
      }
    }
  } else if (warp == W_MMA) {
    // ---------------------------------------------------------------- MMA issuer
    // Tensor-core order per block j: PV_0(j) | S_0(j+1) | PV_1(j) | S_1(j+1): while one softmax
    // warpgroup turns S_t into P_t, the tensor core runs the other tile's GEMMs (ping-pong).
    if (nall > 0) {  // all 32 lanes, converged; MMAs and commits are elect.sync-predicated
      constexpr uint32_t ID_S = idesc<DT, false>(), ID_PV = idesc<DT, true>();
      auto issue_s = [&](int t, int j) {
        // descriptors advance by adding (byte offset >> 4) to the start-address field (no carry: shared
        // addresses stay below 256 KB), so each MMA costs one add per operand instead of a rebuild
        const uint64_t kd0 = sdesc_sw128(sK + (j & 1) * TILE, 16, 1024), qd0 = sdesc_sw128(sQ + t * TILE, 16, 1024);
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t off = ((kk >> 2) * ATOM + (kk & 3) * 32) >> 4;
          mma_f16_e<1>(tmem + TM_S + t * 128, qd0 + off, kd0 + off, ID_S, kk > 0);
        }
        mma_commit_e<1>(bSFull + 8 * t, 0);
      };
      auto issue_pv = [&](int t, int j) {
        const uint64_t vd0 = sdesc_sw128(sV + (j % VS) * TILE, ATOM, 1024);  // + kk * (2048 >> 4) per k16 step
        // O_t += P_t V_j: P_t read from TMEM (packed 16-bit pairs over S_t, 8 columns per k16 step);
        // S_t(j+1) is issued after this and tcgen05 ops execute in order, so it cannot clobber P_t.
        // CS = 3: the first four k16 steps (keys [0, 64), P columns [0, 32)) go as soon as that half
        // of P_t is in TMEM.
        constexpr int KK0 = (CS == 3) ? BKV / 32 : 0;
        if constexpr (CS == 3) {
          mbar_wait_w(bPHalf + 8 * t, j & 1);
          ATRACE(true, 4, t, j);
          tc_fence_after();
#pragma unroll
          for (int kk = 0; kk < KK0; ++kk)
            mma_f16_ts_e(tmem + TM_O + t * 128, tmem + TM_S + t * 128 + P_COL + kk * 8, vd0 + kk * 128, ID_PV,
                       (j | kk) != 0);
        }
        mbar_wait_w(bPReady + 8 * t, j & 1);
        ATRACE(true, 5, t, j);
        tc_fence_after();
#pragma unroll
        for (int kk = KK0; kk < BKV / 16; ++kk)
          mma_f16_ts_e(tmem + TM_O + t * 128, tmem + TM_S + t * 128 + P_COL + kk * 8, vd0 + kk * 128, ID_PV,
                     (j | kk) != 0);
        mma_commit_e<1>(bOReady + 8 * t, 0);
      };
      mbar_wait_w(bQFull, 0);
      mbar_wait_w(bKFull, 0);
      tc_fence_after();
      for (int t = 0; t < NT; ++t)
        if (nkv[t] > 0) issue_s(t, 0);
      mma_commit_e<1>(bKEmpty, 0);  // K_0 consumed
      for (int j = 0; j < nall; ++j) {
        const bool next = j + 1 < nall;
        // operands are awaited where they are first read: V_j before PV_0(j), K_{j+1} only before
        // S_0(j+1), so PV_0(j) runs while K_{j+1} is still landing
        bool k_ready = !next;
        mbar_wait_w(bVFull + 8 * (j % VS), (j / VS) & 1);
        ATRACE(true, 7, 0, j);
        tc_fence_after();
#pragma unroll
        for (int t = 0; t < NT; ++t) {
          if (j < nkv[t]) issue_pv(t, j);
          if (t == NT - 1) mma_commit_e<1>(bVEmpty + 8 * (j % VS), 0);  // V_j fully consumed
          if (next && j + 1 < nkv[t]) {
            if (!k_ready) {
              mbar_wait_w(bKFull + 8 * ((j + 1) & 1), ((j + 1) >> 1) & 1);
              ATRACE(true, 10, 0, j + 1);
              tc_fence_after();
              k_ready = true;
            }
            issue_s(t, j + 1);
            ATRACE(true, 6, t, j + 1);
          }
        }
        if (!k_ready) {  // no S this iteration (causal tail): still consume the phase
          mbar_wait_w(bKFull + 8 * ((j + 1) & 1), ((j + 1) >> 1) & 1);
          tc_fence_after();
        }
        if (next) mma_commit_e<1>(bKEmpty + 8 * ((j + 1) & 1), 0);  // K_{j+1} consumed
      }
    }
  }
  } else if constexpr (CS == 2) {
    // ---------------------------------------------------------------- softmax, both tiles, split rows
    const int h = warp >> 2;        // column half: scores [64h, 64h+64), O columns [64h, 64h+64)
    const int q = warp & 3;         // TMEM lane quarter
    const int r = 32 * q + lane;
    const uint32_t lane_base = uint32_t(32 * q) << 16;
    float* xmax = reinterpret_cast<float*>(smem_raw + (base + XCH_OFF - raw));  // [NT][2 parity][2][BQ]
    float* xl = xmax + NT * 2 * 2 * BQ;                                         // [NT][2][BQ]
    const uint32_t bar_id = 1 + q;
    auto pair_sync = [&]() { asm volatile("bar.sync %0, 64;" ::"r"(bar_id) : "memory"); };
    float m[NT], l[NT];
#pragma unroll
    for (int t = 0; t < NT; ++t) {
      m[t] = -INFINITY;
      l[t] = 0.f;
    }
    for (int j = 0; j < nall; ++j) {
#pragma unroll
      for (int t = 0; t < NT; ++t) {
        if (j >= nkv[t]) continue;
        const int trow0 = q0 + BQ * t;
        const int qrow = trow0 + r;
        const uint32_t tS = tmem + lane_base + TM_S + t * 128;
        const uint32_t tO = tmem + lane_base + TM_O + t * 128 + 64 * h;
        mbar_wait(bSFull + 8 * t, j & 1);
        if (j > 0) mbar_wait(bOReady + 8 * t, (j - 1) & 1);  // never blocks (see CS = 1)
        tc_fence_after();
        uint32_t v[64];
        tmem_ld_32x32b_x32(tS + 64 * h, *reinterpret_cast<uint32_t(*)[32]>(&v[0]));
        tmem_ld_32x32b_x32(tS + 64 * h + 32, *reinterpret_cast<uint32_t(*)[32]>(&v[32]));
        tmem_ld_wait();
        const int key0 = j * BKV + 64 * h;
        const bool full_block = (j * BKV + BKV <= p.sk) && (!p.causal || j * BKV + BKV - 1 <= trow0);
        if (!full_block) {
#pragma unroll
          for (int e = 0; e < 64; ++e) {
            const int key = key0 + e;
            if (key >= p.sk || (p.causal && key > qrow)) v[e] = __float_as_uint(-INFINITY);
          }
        }
        float mx8[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) mx8[u] = -INFINITY;
#pragma unroll
        for (int e = 0; e < 64; ++e) mx8[e & 7] = fmaxf(mx8[e & 7], __uint_as_float(v[e]));
        const float mh = fmaxf(fmaxf(fmaxf(mx8[0], mx8[1]), fmaxf(mx8[2], mx8[3])),
                               fmaxf(fmaxf(mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7])));
        float* xm = xmax + ((t * 2 + (j & 1)) * 2) * BQ;
        xm[h * BQ + r] = mh;
        pair_sync();  // (also: both halves have read S_t(j) before either half's P store)
        float mb = fmaxf(xm[r], xm[BQ + r]);
        mb = (mb == -INFINITY) ? -INFINITY : mb * p.scale_log2;
        float m_new = m[t], corr = 1.f;
        if (mb > m[t] + 8.f) {
          m_new = mb;
          corr = ex2(m[t] - m_new);
        }
        const float msub = (m_new == -INFINITY) ? 0.f : m_new;
        if (j > 0 && __any_sync(0xffffffffu, corr != 1.f)) {  // O_t holds PV_t(j-1)
#pragma unroll 1
          for (int c = 0; c < 2; ++c) {
            uint32_t o[32];
            tmem_ld_32x32b_x32(tO + 32 * c, o);
            tmem_ld_wait();
#pragma unroll
            for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * corr);
            tmem_st_32x32b_x32(tO + 32 * c, o);
          }
        }
        float2 sm4[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) sm4[u] = make_float2(0.f, 0.f);
        const float2 sc2 = make_float2(p.scale_log2, p.scale_log2);
        const float2 ms2 = make_float2(-msub, -msub);
        uint32_t pk[32];
        auto exps = [&](auto e_c) {
          constexpr int E = decltype(e_c)::value;
#pragma unroll
          for (int e = 0; e < 32; ++e) {
            const float2 x = ffma2(make_float2(__uint_as_float(v[2 * e]), __uint_as_float(v[2 * e + 1])), sc2, ms2);
            float2 pe;
            if ((e & 7) < E) {
              pe = ex2_emu2(x);
            } else {
              pe.x = ex2(x.x);
              pe.y = ex2(x.y);
            }
            sm4[e & 3] = fadd2(sm4[e & 3], pe);
            pk[e] = pack2<DT>(pe.x, pe.y);
          }
        };
        if (EMU > 0 && full_block)
          exps(std::integral_constant<int, EMU>{});
        else
          exps(std::integral_constant<int, 0>{});
        // keys [64h, 64h+64) -> P columns P_COL + [32h, 32h+32) = score columns of this half only
        tmem_st_32x32b_x32(tS + P_COL + 32 * h, pk);
        tmem_st_wait();
        l[t] = l[t] * corr + (((sm4[0].x + sm4[0].y) + (sm4[1].x + sm4[1].y)) +
                              ((sm4[2].x + sm4[2].y) + (sm4[3].x + sm4[3].y)));
        m[t] = m_new;
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(bPReady + 8 * t);
      }
    }
    // ---------------------------------------------------------------- epilogue: both tiles
#pragma unroll
    for (int t = 0; t < NT; ++t) {
      const int nk = nkv[t];
      const int trow0 = q0 + BQ * t;
      const int qrow = trow0 + r;
      const uint32_t tO = tmem + lane_base + TM_O + t * 128 + 64 * h;
      xl[(t * 2 + h) * BQ + r] = l[t];
      pair_sync();
      const float lt = xl[(t * 2) * BQ + r] + xl[(t * 2 + 1) * BQ + r];
      const float inv_l = (lt > 0.f) ? 1.f / lt : 0.f;
      if (nk > 0) {
        mbar_wait(bOReady + 8 * t, (nk - 1) & 1);
        tc_fence_after();
      }
      const uint32_t sE = sQ + t * TILE + (h * 4 + q) * 4096;  // Q_t is no longer read: 4 KB per warp
      uint32_t a[64];
      if (nk > 0) {
        tmem_ld_32x32b_x32(tO, *reinterpret_cast<uint32_t(*)[32]>(&a[0]));
        tmem_ld_32x32b_x32(tO + 32, *reinterpret_cast<uint32_t(*)[32]>(&a[32]));
        tmem_ld_wait();
      } else {
#pragma unroll
        for (int e = 0; e < 64; ++e) a[e] = 0u;
      }
#pragma unroll
      for (int vv = 0; vv < 8; ++vv) {
        uint32_t w[4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
          w[u] = pack2<DT>(__uint_as_float(a[8 * vv + 2 * u]) * inv_l, __uint_as_float(a[8 * vv + 2 * u + 1]) * inv_l);
        st_shared_v4(sE + lane * 128 + ((vv ^ (lane & 7)) << 4), w[0], w[1], w[2], w[3]);
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        tma_store_3d(&tmO, sE, 64 * h, trow0 + 32 * q, hb);
        bulk_commit();
      }
      if (h == 0 && p.lse && qrow < p.sq)
        p.lse[(size_t)hb * p.sq + qrow] = (lt > 0.f) ? (m[t] + __log2f(lt)) * 0.6931471805599453f : -INFINITY;
    }
    if (lane == 0) bulk_wait_read<0>();
  } else {
    // ---------------------------------------------------------------- softmax / correction / epilogue
    if constexpr (CS == 3) asm volatile("setmaxnreg.inc.sync.aligned.u32 208;\n" ::: "memory");
    const int t = warp >> 2;        // query tile of this warpgroup
    const int q = warp & 3;         // TMEM lane quarter
    const int r = 32 * q + lane;    // row within the tile = TMEM lane
    const int trow0 = q0 + BQ * t;
    const int qrow = trow0 + r;
    const int nk = nkv[t];
    const uint32_t lane_base = uint32_t(32 * q) << 16;
    const uint32_t tS = tmem + lane_base + TM_S + t * 128;
    const uint32_t tO = tmem + lane_base + TM_O + t * 128;
    float m = -INFINITY, l = 0.f;
    // Ping-pong of the two softmax warpgroups (CS = 3): both tiles need the SFU at the same rate as
    // the tensor core, so their exponential passes take turns -- tile 0 block j, tile 1 block j,
    // tile 0 block j+1, ... -- and each runs at the full SFU rate while the tensor core computes
    // the other tile's PV and S.  Named barrier 8 + t = "tile t may start"; tile 1 only waits while
    // tile 0 still has blocks (causal tiles: nkv[0] <= nkv[1]).
    auto pp_wait = [&](int j) {
      if constexpr (CS == 3 && CY_ATTN_PP > 0)
        if (t == 0 ? j > 0 : j < nkv[0]) asm volatile("bar.sync %0, 256;" ::"r"(8 + t) : "memory");
    };
    auto pp_pass = [&](int j) {
      if constexpr (CS == 3 && CY_ATTN_PP > 0)
        if (t == 0 || j + 1 < nkv[0]) asm volatile("bar.arrive %0, 256;" ::"r"(9 - t) : "memory");
    };
    const bool tr = (threadIdx.x & 127) == 0;
    (void)tr;
    for (int j = 0; j < nk; ++j) {
      mbar_wait(bSFull + 8 * t, j & 1);
      ATRACE(tr, 0, t, j);
      if constexpr (CY_ATTN_PP == 2) pp_wait(j);
      // PV_t(j-1) was issued before S_t(j) and tcgen05 ops complete in order, so this never blocks;
      // consuming every phase keeps the barrier protocol explicit (and compute-sanitizer clean)
      if (j > 0) mbar_wait(bOReady + 8 * t, (j - 1) & 1);
      tc_fence_after();
      const int key0 = j * BKV;
      const bool full_block = (key0 + BKV <= p.sk) && (!p.causal || key0 + BKV - 1 <= trow0);
      // masked keys (ragged last block / causal diagonal) read as -inf
      auto fix = [&](uint32_t (&v)[64], int g) {
        if (!full_block) {
#pragma unroll
          for (int e = 0; e < 64; ++e) {
            const int key = key0 + 64 * g + e;
            if (key >= p.sk || (p.causal && key > qrow)) v[e] = __float_as_uint(-INFINITY);
          }
        }
      };
      auto load64 = [&](uint32_t (&v)[64], int g) {
        tmem_ld_32x32b_x32(tS + 64 * g, *reinterpret_cast<uint32_t(*)[32]>(&v[0]));
        tmem_ld_32x32b_x32(tS + 64 * g + 32, *reinterpret_cast<uint32_t(*)[32]>(&v[32]));
        tmem_ld_wait();
      };
      // pass 1 (TMEM -> registers in 64-column groups): row max, 8 independent partial maxima
      // (CS = 3 keeps both groups in registers for pass 2: a single TMEM pass per block)
      float mx8[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) mx8[u] = -INFINITY;
      uint32_t vrow[CS == 3 ? 2 : 1][64];
      if constexpr (CS == 3) {
        // the whole row in flight at once: four loads behind a single wait
#pragma unroll
        for (int g = 0; g < 2; ++g) {
          tmem_ld_32x32b_x32(tS + 64 * g, *reinterpret_cast<uint32_t(*)[32]>(&vrow[g][0]));
          tmem_ld_32x32b_x32(tS + 64 * g + 32, *reinterpret_cast<uint32_t(*)[32]>(&vrow[g][32]));
        }
        tmem_ld_wait();
        ATRACE(tr, 11, t, j);
#pragma unroll
        for (int g = 0; g < 2; ++g) fix(vrow[g], g);
        auto sc = [&](int k) { return __uint_as_float(vrow[k >> 6][k & 63]); };
        auto max3 = [](float a, float b, float c) { return fmaxf(fmaxf(a, b), c); };
        bool have_max = false;
        if constexpr (CY_ATTN_SPEC != 0) {
          if (j > 0) {
            // Speculative pass (j > 0): take group 0's exponentials against the running max m -- the
            // value P has whenever no row's max grows past the lazy bound (m_new == m below) -- and
            // reduce the row max in 8 chains between them, so the max costs no time of its own.
            // No row grows (the usual case): group 1 follows against m and the block is done, with
            // the same P, sums and order as the path below.  Some row grows: the max is kept and
            // the path below redoes the block against m_new.
            if constexpr (CY_ATTN_PP == 1) pp_wait(j);
            const float ms = (m == -INFINITY) ? 0.f : m;
            const float2 sc2 = make_float2(p.scale_log2, p.scale_log2);
            const float2 ms2 = make_float2(-ms, -ms);
            float2 sm4[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) sm4[u] = make_float2(0.f, 0.f);
            float c8[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) c8[u] = -INFINITY;
            uint32_t pk[32];
            auto exp_pair = [&](int g, int e) {
              const float2 x = ffma2(make_float2(__uint_as_float(vrow[g][2 * e]), __uint_as_float(vrow[g][2 * e + 1])),
                                     sc2, ms2);
              float2 pe;
              pe.x = ex2(x.x);
              pe.y = ex2(x.y);
              sm4[e & 3] = fadd2(sm4[e & 3], pe);
              pk[e] = pack2<DT>(pe.x, pe.y);
            };
#pragma unroll
            for (int e = 0; e < 32; ++e) {
              exp_pair(0, e);
              c8[e & 3] = max3(c8[e & 3], sc(2 * e), sc(2 * e + 1));
              c8[4 + (e & 3)] = max3(c8[4 + (e & 3)], sc(64 + 2 * e), sc(64 + 2 * e + 1));
            }
            tmem_st_32x32b_x32(tS, pk);
            const float rmax = fmaxf(fmaxf(max3(c8[0], c8[1], c8[2]), max3(c8[3], c8[4], c8[5])), fmaxf(c8[6], c8[7]));
            const float mbs = (rmax == -INFINITY) ? -INFINITY : rmax * p.scale_log2;
            ATRACE(tr, 1, t, j);
#if defined(CY_ATTN_MUTANT_NOREDO) || (defined(CY_MUTANT) && CY_MUTANT == 4)  // test-the-test builds only: keep the speculative P even when a row grows
            if (true) {
#else
            if (!__any_sync(0xffffffffu, mbs > m + 8.f)) {
#endif
#pragma unroll
              for (int e = 0; e < 32; ++e) {
                exp_pair(1, e);
                if (e == CY_ATTN_PH_E) {  // group 0's P has long been stored: publish the first half
                  tmem_st_wait();
                  tc_fence_before();
                  __syncwarp();
                  if (lane == 0) mbar_arrive(bPHalf + 8 * t);
                }
              }
              tmem_st_32x32b_x32(tS + 32, pk);
              ATRACE(tr, 2, t, j);
              pp_pass(j);
              tmem_st_wait();
              l = l + (((sm4[0].x + sm4[0].y) + (sm4[1].x + sm4[1].y)) +
                       ((sm4[2].x + sm4[2].y) + (sm4[3].x + sm4[3].y)));  // (= l * corr + ..., corr = 1)
              tc_fence_before();
              __syncwarp();
              if (lane == 0) mbar_arrive(bPReady + 8 * t);
              ATRACE(tr, 3, t, j);
              continue;
            }
            mx8[0] = rmax;
            have_max = true;
          }
        }
        // balanced 3-ary tree (depth 5, every level independent ops) instead of 8 serial chains
        float l1[43];
#pragma unroll
        for (int i = 0; i < 42; ++i) l1[i] = max3(sc(3 * i), sc(3 * i + 1), sc(3 * i + 2));
        l1[42] = fmaxf(sc(126), sc(127));
        float l2[15];
#pragma unroll
        for (int i = 0; i < 14; ++i) l2[i] = max3(l1[3 * i], l1[3 * i + 1], l1[3 * i + 2]);
        l2[14] = l1[42];
        float l3[5];
#pragma unroll
        for (int i = 0; i < 5; ++i) l3[i] = max3(l2[3 * i], l2[3 * i + 1], l2[3 * i + 2]);
        if (!have_max) mx8[0] = max3(max3(l3[0], l3[1], l3[2]), l3[3], l3[4]);
      } else {
#pragma unroll
        for (int g = 0; g < 2; ++g) {
          uint32_t v[64];
          load64(v, g);
          fix(v, g);
#pragma unroll
          for (int e = 0; e < 64; ++e) mx8[e & 7] = fmaxf(mx8[e & 7], __uint_as_float(v[e]));
        }
      }
      float mb = (CS == 3) ? mx8[0]  // (the tree above already reduced the whole row)
                           : fmaxf(fmaxf(fmaxf(mx8[0], mx8[1]), fmaxf(mx8[2], mx8[3])),
                                   fmaxf(fmaxf(mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7])));
      mb = (mb == -INFINITY) ? -INFINITY : mb * p.scale_log2;  // scale_log2 > 0 keeps the order
      // Lazy rescaling: keep the running max unless it grows by more than 2^8 (P <= 256 stays exact
      // in the 16-bit types and the fp32 sums); the final O / l uses the same max, so this is exact.
      // The vote reads the comparison, not corr, so it does not wait for the SFU.
      const bool grow = mb > m + 8.f;
      float m_new = m, corr = 1.f;
      if (grow) {
        m_new = mb;
        corr = ex2(m - m_new);  // 0 when m == -inf
      }
      const float msub = (m_new == -INFINITY) ? 0.f : m_new;
      if (j > 0 && __any_sync(0xffffffffu, grow)) {  // O_t holds PV_t(j-1) (waited above)
#pragma unroll 1
        for (int c = 0; c < 4; ++c) {
          uint32_t o[32];
          tmem_ld_32x32b_x32(tO + 32 * c, o);
          tmem_ld_wait();
#pragma unroll
          for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * corr);
          tmem_st_32x32b_x32(tO + 32 * c, o);
        }
      }
      // pass 2: P = exp2(s * scale_log2 - m) -> packed 16-bit pairs written back over S_t (TMEM
      // cols 0..63; group g's 64 scores become P columns 32g..32g+31, read by the MMA afterwards)
      // sm4[u].x / .y accumulate elements 2e / 2e+1 with e % 4 == u (8 independent fp32 chains)
      float2 sm4[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) sm4[u] = make_float2(0.f, 0.f);
      const float2 sc2 = make_float2(p.scale_log2, p.scale_log2);
      const float2 ms2 = make_float2(-msub, -msub);
      // E of every 8 pairs take the FMA-pipe exponential (only in blocks without masked scores,
      // where ex2_emu2's clamp never applies to a -inf)
      auto pass2 = [&](auto e_c) {
        constexpr int E = decltype(e_c)::value;
#pragma unroll
        for (int g = 0; g < 2; ++g) {
          uint32_t v[64];
          if constexpr (CS == 3) {
#pragma unroll
            for (int e = 0; e < 64; ++e) v[e] = vrow[g][e];
          } else {
            load64(v, g);
            if constexpr (E == 0) fix(v, g);
          }
          uint32_t pk[32];
#pragma unroll
          for (int e = 0; e < 32; ++e) {
            const float2 x = ffma2(make_float2(__uint_as_float(v[2 * e]), __uint_as_float(v[2 * e + 1])), sc2, ms2);
            float2 pe;
            if ((e & 7) < E) {
              pe = ex2_emu2(x);
            } else {
              pe.x = ex2(x.x);
              pe.y = ex2(x.y);
            }
            sm4[e & 3] = fadd2(sm4[e & 3], pe);
            pk[e] = pack2<DT>(pe.x, pe.y);
            if constexpr (CS == 3) {
              if (g == 1 && e == CY_ATTN_PH_E) {
                // group 0's P (and any O rescale) has long been stored: publish the first half
                tmem_st_wait();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(bPHalf + 8 * t);
              }
            }
          }
          // group 1's P lands in columns 32..63, which group 1's scores (columns 64..127) do not
          // overlap; group 0's P (columns 0..31) overwrites scores already consumed
          tmem_st_32x32b_x32(tS + 32 * g, pk);
        }
      };
      ATRACE(tr, 1, t, j);
      if constexpr (CY_ATTN_PP == 1) pp_wait(j);
      if (EMU > 0 && full_block)
        pass2(std::integral_constant<int, EMU>{});
      else
        pass2(std::integral_constant<int, 0>{});
      ATRACE(tr, 2, t, j);
      pp_pass(j);
      tmem_st_wait();
      l = l * corr + (((sm4[0].x + sm4[0].y) + (sm4[1].x + sm4[1].y)) +
                      ((sm4[2].x + sm4[2].y) + (sm4[3].x + sm4[3].y)));
      m = m_new;
      tc_fence_before();  // P and the rescaled O (tcgen05.st) before the MMA issuer's PV_t(j)
      __syncwarp();
      if (lane == 0) mbar_arrive(bPReady + 8 * t);
      ATRACE(tr, 3, t, j);
    }
    // ---------------------------------------------------------------- epilogue: O / l, lse
    const float inv_l = (l > 0.f) ? 1.f / l : 0.f;
    if (nk > 0) {
      mbar_wait(bOReady + 8 * t, (nk - 1) & 1);
      tc_fence_after();
    }
    const uint32_t sE = sQ + t * TILE + q * 4096;  // Q_t is no longer read: 4 KB staging per warp
#pragma unroll 1
    for (int c = 0; c < 2; ++c) {
      uint32_t a0[32], a1[32];
      if (nk > 0) {
        tmem_ld_32x32b_x32(tO + 64 * c, a0);
        tmem_ld_32x32b_x32(tO + 64 * c + 32, a1);
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
        tma_store_3d(&tmO, sE, 64 * c, trow0 + 32 * q, hb);
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
  if (warp == W_MMA) {
    tc_fence_after();
    tmem_dealloc<1>(tmem, 512);
  }
}



#if CY_ATTN_DB
// ============================================================================ double-buffered S kernel
// Experiment build only (CY_ATTN_DB=1): correct (all attention tests) but slower than the default
// kernel -- 1116-1164 vs 1254-1289 TFLOP/s at 2x16x8192, 990 vs 1075 causal.
// attn_db_kernel: the two-tile layout with 64-key blocks so that each tile's S can be
// double-buffered in TMEM (S_t buffers u = 0, 1 at columns 64 (2t + u); O_t at 256 + 128 t).  S_t(j+2)
// goes into the buffer P_t(j) leaves once PV_t(j) has read it, so the scores of block j+1 are already in
// TMEM when the softmax of block j finishes: the per-tile chain S -> softmax -> PV -> S of the default
// kernel (which keeps P_t in the only S_t buffer) becomes softmax -> softmax, and the two tiles' softmax
// warpgroups run side by side instead of taking turns.  K / V: 64-key tiles (16 KB) in 4-slot rings.
namespace db {
constexpr int BK = 64;                       // keys per block
constexpr int KVT = BK * D * 2;              // one K or V tile: 16 KB (two SW128 atoms of 64 rows, 8 KB apart)
constexpr int KV_ATOM = BK * 128;            // 8 KB
constexpr int NS = 4;                        // K and V ring slots
constexpr int SQ = 0, SK = NT * TILE, SV = SK + NS * KVT, BAR = SV + NS * KVT;
constexpr int SMEM_BYTES = 1024 + BAR + 256;
static_assert(SMEM_BYTES <= 232448, "DB layout exceeds 227 KB");
__device__ __forceinline__ int blocks(const Params& p, int row_end) {
  const int kv_end = p.causal ? min(p.sk, row_end) : p.sk;
  return (kv_end + BK - 1) / BK;
}
}  // namespace db

template <int DT>
__global__ void __launch_bounds__(384, 1)
    attn_db_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                   const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmO,
                   const Params p) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  const uint32_t sQ = base + db::SQ, sK = base + db::SK, sV = base + db::SV;
  const uint32_t bar = base + db::BAR;
  const uint32_t bQFull = bar, bKFull = bar + 8, bKEmpty = bar + 40, bVFull = bar + 72, bVEmpty = bar + 104,
                 bSFull = bar + 136 /* [t][u] */, bPReady = bar + 168, bOReady = bar + 184, sTmemSlot = bar + 200;
  volatile uint32_t* tmem_slot = reinterpret_cast<volatile uint32_t*>(smem_raw + (sTmemSlot - raw));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int qt = p.causal ? (gridDim.x - 1 - blockIdx.x) : blockIdx.x;  // heavy causal CTAs first
  const int hb = blockIdx.y;
  const int q0 = qt * BQ * NT;
  int nkv[NT];
#pragma unroll
  for (int t = 0; t < NT; ++t) nkv[t] = db::blocks(p, q0 + BQ * (t + 1));
  const int nall = nkv[NT - 1];

  if (warp == W_PROD && lane == 0) {
    prefetch_tmap(&tmQ);
    prefetch_tmap(&tmK);
    prefetch_tmap(&tmV);
    prefetch_tmap(&tmO);
    mbar_init(bQFull, 1);
    for (int s = 0; s < db::NS; ++s) {
      mbar_init(bKFull + 8 * s, 1);
      mbar_init(bKEmpty + 8 * s, 1);
      mbar_init(bVFull + 8 * s, 1);
      mbar_init(bVEmpty + 8 * s, 1);
    }
    for (int t = 0; t < NT; ++t) {
      mbar_init(bSFull + 16 * t, 1);
      mbar_init(bSFull + 16 * t + 8, 1);
      mbar_init(bPReady + 8 * t, 4);
      mbar_init(bOReady + 8 * t, 1);
    }
    fence_mbar_init();
  }
  if (warp == W_MMA) {
    tmem_alloc<1>(sTmemSlot, 512);
    tmem_relinquish<1>();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();
  pdl_launch_dependents();
  if (warp >= 4 * NT) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 72;\n" ::: "memory");
    if (warp == W_PROD) {
      // ---------------------------------------------------------------- producer
      if (nall > 0) {
        const uint64_t pol = policy_evict_last();
        mbar_arrive_expect_tx_e(bQFull, NT * TILE);
        for (int t = 0; t < NT; ++t) tma_load_4d_e(sQ + t * TILE, &tmQ, bQFull, 0, q0 + BQ * t, 0, hb, pol, true);
        for (int j = 0; j < nall; ++j) {
          const int s = j % db::NS;
          const uint32_t ph = ((j / db::NS) & 1) ^ 1;
          mbar_wait_w(bKEmpty + 8 * s, ph);
          mbar_arrive_expect_tx_e(bKFull + 8 * s, db::KVT);
          tma_load_4d_e(sK + s * db::KVT, &tmK, bKFull + 8 * s, 0, j * db::BK, 0, hb, pol, true);
          mbar_wait_w(bVEmpty + 8 * s, ph);
          mbar_arrive_expect_tx_e(bVFull + 8 * s, db::KVT);
          tma_load_4d_e(sV + s * db::KVT, &tmV, bVFull + 8 * s, 0, j * db::BK, 0, hb, pol, true);
        }
      }
    } else if (warp == W_MMA) {
      // ---------------------------------------------------------------- MMA issuer
      // S_t(j) -> buffer j & 1 (N = 64 keys); O_t += P_t(j) V_j with P_t(j) read from that buffer.
      // Order: S(0), S(1) of both tiles, then per block j: PV_0(j), PV_1(j), S_0(j+2), S_1(j+2) --
      // S_t(j+2) overwrites P_t(j) only after PV_t(j) (tcgen05 ops execute in order).
      if (nall > 0) {
        constexpr uint32_t ID_S = idesc<DT, false, 64>(), ID_PV = idesc<DT, true>();
        auto issue_s = [&](int t, int j) {
          const uint32_t ks = sK + (j % db::NS) * db::KVT;
          const uint64_t kd0 = sdesc_sw128(ks, 16, 1024), qd0 = sdesc_sw128(sQ + t * TILE, 16, 1024);
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const uint32_t qoff = ((kk >> 2) * ATOM + (kk & 3) * 32) >> 4;
            const uint32_t koff = ((kk >> 2) * db::KV_ATOM + (kk & 3) * 32) >> 4;
            mma_f16_e<1>(tmem + 64 * (2 * t + (j & 1)), qd0 + qoff, kd0 + koff, ID_S, kk > 0);
          }
          mma_commit_e<1>(bSFull + 16 * t + 8 * (j & 1), 0);
        };
        auto issue_pv = [&](int t, int j) {
          const uint64_t vd0 = sdesc_sw128(sV + (j % db::NS) * db::KVT, db::KV_ATOM, 1024);
          mbar_wait_w(bPReady + 8 * t, j & 1);
          tc_fence_after();
#pragma unroll
          for (int kk = 0; kk < db::BK / 16; ++kk)
            mma_f16_ts_e(tmem + TM_O + t * 128, tmem + 64 * (2 * t + (j & 1)) + kk * 8, vd0 + kk * 128, ID_PV,
                         (j | kk) != 0);
          mma_commit_e<1>(bOReady + 8 * t, 0);
        };
        auto s_block = [&](int j) {  // S of both tiles for block j (K_j), then K_j's slot is free
          const int s = j % db::NS;
          mbar_wait_w(bKFull + 8 * s, (j / db::NS) & 1);
          tc_fence_after();
          for (int t = 0; t < NT; ++t)
            if (j < nkv[t]) issue_s(t, j);
          mma_commit_e<1>(bKEmpty + 8 * s, 0);
        };
        mbar_wait_w(bQFull, 0);
        s_block(0);
        if (nall > 1) s_block(1);
        for (int j = 0; j < nall; ++j) {
          const int s = j % db::NS;
          mbar_wait_w(bVFull + 8 * s, (j / db::NS) & 1);
          tc_fence_after();
          for (int t = 0; t < NT; ++t)
            if (j < nkv[t]) issue_pv(t, j);
          mma_commit_e<1>(bVEmpty + 8 * s, 0);
          if (j + 2 < nall) s_block(j + 2);
        }
      }
    }
  } else {
    // ---------------------------------------------------------------- softmax / epilogue
    asm volatile("setmaxnreg.inc.sync.aligned.u32 208;\n" ::: "memory");
    const int t = warp >> 2, q = warp & 3;
    const int r = 32 * q + lane;
    const int trow0 = q0 + BQ * t;
    const int qrow = trow0 + r;
    const int nk = nkv[t];
    const uint32_t lane_base = uint32_t(32 * q) << 16;
    const uint32_t tO = tmem + lane_base + TM_O + t * 128;
    const float2 sc2 = make_float2(p.scale_log2, p.scale_log2);
    float m = -INFINITY, l = 0.f;
    // PV_t(i) completes phase i of bOReady_t.  Once S_t(j) is complete so is PV_t(j-2) (issued before
    // it), so at block j the barrier's current phase is j - 1 or j and a parity wait for phase j - 1
    // is unambiguous; the softmax waits on it only before rescaling O, and once at the end.
    for (int j = 0; j < nk; ++j) {
      const uint32_t tS = tmem + lane_base + 64 * (2 * t + (j & 1));
      mbar_wait(bSFull + 16 * t + 8 * (j & 1), (j >> 1) & 1);
      tc_fence_after();
      uint32_t v[64];
      tmem_ld_32x32b_x32(tS, *reinterpret_cast<uint32_t(*)[32]>(&v[0]));
      tmem_ld_32x32b_x32(tS + 32, *reinterpret_cast<uint32_t(*)[32]>(&v[32]));
      tmem_ld_wait();
      const int key0 = j * db::BK;
      const bool full_block = (key0 + db::BK <= p.sk) && (!p.causal || key0 + db::BK - 1 <= trow0);
      if (!full_block) {
#pragma unroll
        for (int e = 0; e < 64; ++e) {
          const int key = key0 + e;
          if (key >= p.sk || (p.causal && key > qrow)) v[e] = __float_as_uint(-INFINITY);
        }
      }
      auto sc = [&](int k) { return __uint_as_float(v[k]); };
      auto max3 = [](float a, float b, float c) { return fmaxf(fmaxf(a, b), c); };
      float2 sm4[4];
      uint32_t pk[32];
      // exponentials against `ms`, the row max reduced in 4 chains between them
      float c4[4];
      auto pass = [&](float ms, bool with_max) {
        const float2 ms2 = make_float2(-ms, -ms);
#pragma unroll
        for (int u = 0; u < 4; ++u) sm4[u] = make_float2(0.f, 0.f);
#pragma unroll
        for (int e = 0; e < 32; ++e) {
          const float2 x = ffma2(make_float2(sc(2 * e), sc(2 * e + 1)), sc2, ms2);
          float2 pe;
          pe.x = ex2(x.x);
          pe.y = ex2(x.y);
          sm4[e & 3] = fadd2(sm4[e & 3], pe);
          pk[e] = pack2<DT>(pe.x, pe.y);
          if (with_max) c4[e & 3] = max3(c4[e & 3], sc(2 * e), sc(2 * e + 1));
        }
      };
#pragma unroll
      for (int u = 0; u < 4; ++u) c4[u] = -INFINITY;
      // speculative pass against the running max (the P of every block whose row max stays within
      // the lazy bound); block 0 (m = -inf) always takes the path below
      pass((m == -INFINITY) ? 0.f : m, true);
      const float rmax = fmaxf(fmaxf(c4[0], c4[1]), fmaxf(c4[2], c4[3]));
      const float mb = (rmax == -INFINITY) ? -INFINITY : rmax * p.scale_log2;
      const bool grow = mb > m + 8.f;
      float corr = 1.f;
      if (__any_sync(0xffffffffu, grow)) {
        float m_new = m;
        if (grow) {
          m_new = mb;
          corr = ex2(m - m_new);  // 0 when m == -inf
        }
        if (j > 0) {
          // O_t must hold PV_t(j-1) before it is rescaled (the only place the softmax touches O)
          mbar_wait(bOReady + 8 * t, (j - 1) & 1);
          tc_fence_after();
#pragma unroll 1
          for (int c = 0; c < 4; ++c) {
            uint32_t o[32];
            tmem_ld_32x32b_x32(tO + 32 * c, o);
            tmem_ld_wait();
#pragma unroll
            for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * corr);
            tmem_st_32x32b_x32(tO + 32 * c, o);
          }
        }
        m = m_new;
        pass((m == -INFINITY) ? 0.f : m, false);
      }
      // Publishing P_t(j) (and storing it) only once PV_t(j-1) is complete is required: without this
      // wait, sharp-softmax inputs (where other warps take the redo path) produced wrong P and sums
      // in rows of warps that did not (measured, scripts/experiments/attn_nan.py); with it all 55
      // attention tests pass.
      if (j > 0) mbar_wait(bOReady + 8 * t, (j - 1) & 1);
      tmem_st_32x32b_x32(tS, pk);  // P (16-bit pairs) over the block's first 32 score columns
      tmem_st_wait();
      l = l * corr + (((sm4[0].x + sm4[0].y) + (sm4[1].x + sm4[1].y)) + ((sm4[2].x + sm4[2].y) + (sm4[3].x + sm4[3].y)));
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(bPReady + 8 * t);
    }
    // ---------------------------------------------------------------- epilogue: O / l, lse
    const float inv_l = (l > 0.f) ? 1.f / l : 0.f;
    if (nk > 0) {
      mbar_wait(bOReady + 8 * t, (nk - 1) & 1);
      tc_fence_after();
    }
    const uint32_t sE = sQ + t * TILE + q * 4096;  // Q_t is no longer read (all S_t issued and done)
#pragma unroll 1
    for (int c = 0; c < 2; ++c) {
      uint32_t a0[32], a1[32];
      if (nk > 0) {
        tmem_ld_32x32b_x32(tO + 64 * c, a0);
        tmem_ld_32x32b_x32(tO + 64 * c + 32, a1);
        tmem_ld_wait();
      } else {
#pragma unroll
        for (int e = 0; e < 32; ++e) a0[e] = a1[e] = 0u;
      }
      if (lane == 0 && c > 0) bulk_wait_read<0>();
      __syncwarp();
#pragma unroll
      for (int vv = 0; vv < 8; ++vv) {
        uint32_t w[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int col = 8 * vv + 2 * u;
          const float x0 = __uint_as_float(col < 32 ? a0[col] : a1[col - 32]) * inv_l;
          const float x1 = __uint_as_float(col + 1 < 32 ? a0[col + 1] : a1[col + 1 - 32]) * inv_l;
          w[u] = pack2<DT>(x0, x1);
        }
        st_shared_v4(sE + lane * 128 + ((vv ^ (lane & 7)) << 4), w[0], w[1], w[2], w[3]);
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        tma_store_3d(&tmO, sE, 64 * c, trow0 + 32 * q, hb);
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
  if (warp == W_MMA) {
    tc_fence_after();
    tmem_dealloc<1>(tmem, 512);
  }
}
#endif  // CY_ATTN_DB

#if CY_ATTN_T1
// ============================================================================ one-tile kernel
// Experiment build only (CY_ATTN_T1=1).  attn_t1_kernel: one 128-row query tile per CTA with S
// double-buffered in TMEM (S buffers at columns 0 / 128, O at 256) and 8 softmax warps, two per TMEM
// lane quarter, each taking 64 of the block's 128 keys (and 64 of O's columns).  The MMA order is
// S(0), S(1), then per block PV(j), S(j+2): the scores of block j+1 are in TMEM while block j's softmax
// runs, so consecutive blocks' softmax passes follow each other with no wait for the tensor core.
namespace t1 {
constexpr int NK = 3, NV = 3;                              // K and V ring slots (32 KB tiles)
constexpr int SQ = 0, SK = TILE, SV = SK + NK * TILE, BAR = SV + NV * TILE;
constexpr int XCH = BAR + 256;                             // [2 halves][128 rows] fp32 exchange
constexpr int SMEM_BYTES = 1024 + XCH + 2 * 128 * 4;
static_assert(SMEM_BYTES <= 232448, "T1 layout exceeds 227 KB");
}  // namespace t1

template <int DT>
__global__ void __launch_bounds__(384, 1)
    attn_t1_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                   const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmO,
                   const Params p) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  const uint32_t sQ = base + t1::SQ, sK = base + t1::SK, sV = base + t1::SV;
  const uint32_t bar = base + t1::BAR;
  const uint32_t bQFull = bar, bKFull = bar + 8, bKEmpty = bar + 32, bVFull = bar + 56, bVEmpty = bar + 80,
                 bSFull = bar + 104 /* [2] */, bPReady = bar + 120, bOReady = bar + 128, sTmemSlot = bar + 136;
  float* xch = reinterpret_cast<float*>(smem_raw + (base + t1::XCH - raw));  // [2][128]
  volatile uint32_t* tmem_slot = reinterpret_cast<volatile uint32_t*>(smem_raw + (sTmemSlot - raw));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int qt = p.lpt ? (gridDim.y - 1 - blockIdx.y) : p.causal ? (gridDim.x - 1 - blockIdx.x) : blockIdx.x;
  const int hb = p.lpt ? blockIdx.x : blockIdx.y;
  const int q0 = qt * BQ;
  const int nk = blocks_for(p, q0 + BQ);

  if (warp == W_PROD && lane == 0) {
    prefetch_tmap(&tmQ);
    prefetch_tmap(&tmK);
    prefetch_tmap(&tmV);
    prefetch_tmap(&tmO);
    mbar_init(bQFull, 1);
    for (int s = 0; s < t1::NK; ++s) {
      mbar_init(bKFull + 8 * s, 1);
      mbar_init(bKEmpty + 8 * s, 1);
    }
    for (int s = 0; s < t1::NV; ++s) {
      mbar_init(bVFull + 8 * s, 1);
      mbar_init(bVEmpty + 8 * s, 1);
    }
    mbar_init(bSFull, 1);
    mbar_init(bSFull + 8, 1);
    mbar_init(bPReady, 8);
    mbar_init(bOReady, 1);
    fence_mbar_init();
  }
  if (warp == W_MMA) {
    tmem_alloc<1>(sTmemSlot, 512);
    tmem_relinquish<1>();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();
  pdl_launch_dependents();
  if (warp >= 8) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 72;\n" ::: "memory");
    if (warp == W_PROD) {
      if (nk > 0) {
        const uint64_t pol = policy_evict_last();
        mbar_arrive_expect_tx_e(bQFull, TILE);
        tma_load_4d_e(sQ, &tmQ, bQFull, 0, q0, 0, hb, pol, true);
        for (int j = 0; j < nk; ++j) {
          const int ks = j % t1::NK, vs = j % t1::NV;
          mbar_wait_w(bKEmpty + 8 * ks, ((j / t1::NK) & 1) ^ 1);
#ifdef CY_ATTN_T1_NOLOAD  // timing experiment only (invalid results): no K / V reloads after the ring fill
          if (j >= 3) {
            mbar_arrive_e(bKFull + 8 * ks);
            mbar_wait_w(bVEmpty + 8 * vs, ((j / t1::NV) & 1) ^ 1);
            mbar_arrive_e(bVFull + 8 * vs);
            continue;
          }
#endif
          mbar_arrive_expect_tx_e(bKFull + 8 * ks, TILE);
          tma_load_4d_e(sK + ks * TILE, &tmK, bKFull + 8 * ks, 0, j * BKV, 0, hb, pol, true);
          mbar_wait_w(bVEmpty + 8 * vs, ((j / t1::NV) & 1) ^ 1);
          mbar_arrive_expect_tx_e(bVFull + 8 * vs, TILE);
          tma_load_4d_e(sV + vs * TILE, &tmV, bVFull + 8 * vs, 0, j * BKV, 0, hb, pol, true);
        }
      }
    } else if (warp == W_MMA) {
      if (nk > 0) {
        constexpr uint32_t ID_S = idesc<DT, false>(), ID_PV = idesc<DT, true>();
        auto issue_s = [&](int j) {
          const int ks = j % t1::NK;
          mbar_wait_w(bKFull + 8 * ks, (j / t1::NK) & 1);
          tc_fence_after();
          const uint64_t kd0 = sdesc_sw128(sK + ks * TILE, 16, 1024), qd0 = sdesc_sw128(sQ, 16, 1024);
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const uint32_t off = ((kk >> 2) * ATOM + (kk & 3) * 32) >> 4;
            mma_f16_e<1>(tmem + 128 * (j & 1), qd0 + off, kd0 + off, ID_S, kk > 0);
          }
          mma_commit_e<1>(bSFull + 8 * (j & 1), 0);
          mma_commit_e<1>(bKEmpty + 8 * ks, 0);
        };
        mbar_wait_w(bQFull, 0);
        tc_fence_after();
        issue_s(0);
        if (nk > 1) issue_s(1);
        for (int j = 0; j < nk; ++j) {
          const int vs = j % t1::NV;
          mbar_wait_w(bVFull + 8 * vs, (j / t1::NV) & 1);
          mbar_wait_w(bPReady, j & 1);
          tc_fence_after();
          const uint64_t vd0 = sdesc_sw128(sV + vs * TILE, ATOM, 1024);
#pragma unroll
          for (int kk = 0; kk < BKV / 16; ++kk)
            mma_f16_ts_e(tmem + TM_O, tmem + 128 * (j & 1) + kk * 8, vd0 + kk * 128, ID_PV, (j | kk) != 0);
          mma_commit_e<1>(bOReady, 0);
          mma_commit_e<1>(bVEmpty + 8 * vs, 0);
          if (j + 2 < nk) issue_s(j + 2);  // into buffer j & 1, after PV(j) has read P(j) from it
        }
      }
    }
  } else {
    // ---------------------------------------------------------------- softmax / epilogue
    asm volatile("setmaxnreg.inc.sync.aligned.u32 208;\n" ::: "memory");
    const int q = warp & 3, h = warp >> 2;  // lane quarter, key half (and O column half)
    const int r = 32 * q + lane;
    const int qrow = q0 + r;
    const uint32_t lane_base = uint32_t(32 * q) << 16;
    const uint32_t tO = tmem + lane_base + TM_O + 64 * h;
    const float2 sc2 = make_float2(p.scale_log2, p.scale_log2);
    const uint32_t pair_bar = 1 + q;  // named barrier of the two warps of lane quarter q
    auto pair_sync = [&]() { asm volatile("bar.sync %0, 64;" ::"r"(pair_bar) : "memory"); };
    float m = -INFINITY, l = 0.f;
    for (int j = 0; j < nk; ++j) {
      const uint32_t tS = tmem + lane_base + 128 * (j & 1) + 64 * h;
      mbar_wait(bSFull + 8 * (j & 1), (j >> 1) & 1);
      tc_fence_after();
      uint32_t v[64];
      tmem_ld_32x32b_x32(tS, *reinterpret_cast<uint32_t(*)[32]>(&v[0]));
      tmem_ld_32x32b_x32(tS + 32, *reinterpret_cast<uint32_t(*)[32]>(&v[32]));
      tmem_ld_wait();
      const int key0 = j * BKV + 64 * h;
      const bool full_block = (j * BKV + BKV <= p.sk) && (!p.causal || j * BKV + BKV - 1 <= q0);
      if (!full_block) {
#pragma unroll
        for (int e = 0; e < 64; ++e) {
          const int key = key0 + e;
          if (key >= p.sk || (p.causal && key > qrow)) v[e] = __float_as_uint(-INFINITY);
        }
      }
      auto sc = [&](int k) { return __uint_as_float(v[k]); };
      auto max3 = [](float a, float b, float c) { return fmaxf(fmaxf(a, b), c); };
      float2 sm4[4];
      uint32_t pk[32];
      float c4[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) c4[u] = -INFINITY;
      auto pass = [&](float ms, bool with_max) {
        const float2 ms2 = make_float2(-ms, -ms);
#pragma unroll
        for (int u = 0; u < 4; ++u) sm4[u] = make_float2(0.f, 0.f);
#pragma unroll
        for (int e = 0; e < 32; ++e) {
          const float2 x = ffma2(make_float2(sc(2 * e), sc(2 * e + 1)), sc2, ms2);
          float2 pe;
          pe.x = ex2(x.x);
          pe.y = ex2(x.y);
          sm4[e & 3] = fadd2(sm4[e & 3], pe);
          pk[e] = pack2<DT>(pe.x, pe.y);
          if (with_max) c4[e & 3] = max3(c4[e & 3], sc(2 * e), sc(2 * e + 1));
        }
      };
      pass((m == -INFINITY) ? 0.f : m, true);
      // the row's max over both halves: exchange with the partner warp of this lane quarter
      const float hmax = fmaxf(fmaxf(c4[0], c4[1]), fmaxf(c4[2], c4[3]));
      float* xm = xch + (j & 1) * 0;  // (one slot per half; the pair barrier below orders reuse)
      xm[h * 128 + r] = hmax;
      pair_sync();
      const float rmax = fmaxf(hmax, xm[(h ^ 1) * 128 + r]);
      pair_sync();  // both have read before the next block overwrites
      const float mb = (rmax == -INFINITY) ? -INFINITY : rmax * p.scale_log2;
      const bool grow = mb > m + 8.f;
      float corr = 1.f;
      // P(j) is stored and published only once PV(j-1) is complete (see attn_db_kernel)
      if (j > 0) mbar_wait(bOReady, (j - 1) & 1);
      if (__any_sync(0xffffffffu, grow)) {
        float m_new = m;
        if (grow) {
          m_new = mb;
          corr = ex2(m - m_new);
        }
        if (j > 0) {
          tc_fence_after();
#pragma unroll 1
          for (int c = 0; c < 2; ++c) {
            uint32_t o[32];
            tmem_ld_32x32b_x32(tO + 32 * c, o);
            tmem_ld_wait();
#pragma unroll
            for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * corr);
            tmem_st_32x32b_x32(tO + 32 * c, o);
          }
        }
        m = m_new;
        pass((m == -INFINITY) ? 0.f : m, false);
      }
      tmem_st_32x32b_x32(tmem + lane_base + 128 * (j & 1) + 32 * h, pk);  // P cols [32h, 32h + 32)
      tmem_st_wait();
      l = l * corr + (((sm4[0].x + sm4[0].y) + (sm4[1].x + sm4[1].y)) + ((sm4[2].x + sm4[2].y) + (sm4[3].x + sm4[3].y)));
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(bPReady);
    }
    // ---------------------------------------------------------------- epilogue: O / l, lse
    xch[h * 128 + r] = l;
    pair_sync();
    const float lt = l + xch[(h ^ 1) * 128 + r];
    const float inv_l = (lt > 0.f) ? 1.f / lt : 0.f;
    if (nk > 0) {
      mbar_wait(bOReady, (nk - 1) & 1);
      tc_fence_after();
    }
    const uint32_t sE = sQ + warp * 4096;  // Q is no longer read: 4 KB staging per warp
    uint32_t a0[32], a1[32];
    if (nk > 0) {
      tmem_ld_32x32b_x32(tO, a0);
      tmem_ld_32x32b_x32(tO + 32, a1);
      tmem_ld_wait();
    } else {
#pragma unroll
      for (int e = 0; e < 32; ++e) a0[e] = a1[e] = 0u;
    }
#pragma unroll
    for (int vv = 0; vv < 8; ++vv) {
      uint32_t w[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int col = 8 * vv + 2 * u;
        const float x0 = __uint_as_float(col < 32 ? a0[col] : a1[col - 32]) * inv_l;
        const float x1 = __uint_as_float(col + 1 < 32 ? a0[col + 1] : a1[col + 1 - 32]) * inv_l;
        w[u] = pack2<DT>(x0, x1);
      }
      st_shared_v4(sE + lane * 128 + ((vv ^ (lane & 7)) << 4), w[0], w[1], w[2], w[3]);
    }
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) {
      tma_store_3d(&tmO, sE, 64 * h, q0 + 32 * q, hb);
      bulk_commit();
    }
    if (h == 0 && p.lse && qrow < p.sq)
      p.lse[(size_t)hb * p.sq + qrow] = (lt > 0.f) ? (m + __log2f(lt)) * 0.6931471805599453f : -INFINITY;
    if (lane == 0) bulk_wait_read<0>();
  }
  __syncwarp();
  tc_fence_before();
  __syncthreads();
  if (warp == W_MMA) {
    tc_fence_after();
    tmem_dealloc<1>(tmem, 512);
  }
}
#endif  // CY_ATTN_T1

#ifdef CY_ATTN_EXPERIMENTS  // measured slower than the default: experiment build only
// ============================================================================ persistent two-tile kernel
// The default layout (two 128-row query tiles per CTA, softmax warpgroup per tile, setmaxnreg)
// made persistent: one CTA per SM walks the work items (query-tile pair, batch*head) -- the
// "persistent kernel" optimisation the paper names as Cypress's missing piece for attention
// (P:1657-1664).  Across items the K/V rings and every barrier phase simply continue; the O_t
// accumulator is handed back by the epilogue (bOFree_t) before the next item's first PV_t, and the
// next item's Q tiles load as soon as the last S MMAs of the previous item have read Q (bQEmpty),
// so one item's epilogue overlaps the next item's loads, first S MMAs and first softmax.
// Shared: Q 2 x 32 KB, K/V 2 x 64 KB, O staging 8 x 4 KB (no longer aliased with Q).
constexpr int PS_STAGE_OFF = (NT + 4) * TILE;                 // 8 warps x 4 KB epilogue staging
constexpr int PS_BAR_OFF = PS_STAGE_OFF + 8 * 4096;
constexpr int PS_SMEM_BYTES = 1024 + PS_BAR_OFF + 256;

__device__ __forceinline__ void item_coords(const Params& p, int item, int nq, int& qt, int& hb) {
  // query tiles fastest, as in the one-CTA-per-item grid: the items in flight share a few heads'
  // K/V, which stay in L2 and whose TMA requests merge
  hb = item / nq;
  const int qi = item - hb * nq;
  qt = p.causal ? (nq - 1 - qi) : qi;  // causal: heaviest query tile of each head first
}

template <int DT>
__global__ void __launch_bounds__(384, 1)
    attn_persist_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                        const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmO,
                        const Params p) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  const uint32_t sQ = base + SQ_OFF, sK = base + SK_OFF, sV = base + SV_OFF, sStage = base + PS_STAGE_OFF;
  const uint32_t bar = base + PS_BAR_OFF;
  const uint32_t bQFull = bar, bQEmpty = bar + 8, bKFull = bar + 16, bKEmpty = bar + 32, bVFull = bar + 48,
                 bVEmpty = bar + 64, bSFull = bar + 80, bPReady = bar + 96, bOReady = bar + 112, bOFree = bar + 128,
                 sTmemSlot = bar + 144;
  volatile uint32_t* tmem_slot = reinterpret_cast<volatile uint32_t*>(smem_raw + (sTmemSlot - raw));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nq = (p.sq + BQ * NT - 1) / (BQ * NT);
  const int items = nq * p.bh;
  auto blocks_of = [&](int qt, int t) { return blocks_for(p, qt * BQ * NT + BQ * (t + 1)); };

  if (warp == W_PROD && lane == 0) {
    prefetch_tmap(&tmQ);
    prefetch_tmap(&tmK);
    prefetch_tmap(&tmV);
    prefetch_tmap(&tmO);
    mbar_init(bQFull, 1);
    mbar_init(bQEmpty, 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(bKFull + 8 * s, 1);
      mbar_init(bKEmpty + 8 * s, 1);
      mbar_init(bVFull + 8 * s, 1);
      mbar_init(bVEmpty + 8 * s, 1);
    }
    for (int t = 0; t < NT; ++t) {
      mbar_init(bSFull + 8 * t, 1);
      mbar_init(bPReady + 8 * t, 4);
      mbar_init(bOReady + 8 * t, 1);
      mbar_init(bOFree + 8 * t, 4);
    }
    fence_mbar_init();
  }
  if (warp == W_MMA) {
    tmem_alloc<1>(sTmemSlot, 512);
    tmem_relinquish<1>();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();
  if (threadIdx.x == 0) pdl_launch_dependents();

  if (warp >= 4 * NT) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 104;\n" ::: "memory");
    if (warp == W_PROD && lane == 0) {
      // ---------------------------------------------------------------- producer
      const uint64_t pol = policy_evict_last();
      auto ld = [&](uint32_t dst, const CUtensorMap* tm, uint32_t b, int row, int hb) {  // 4-D maps: whole tile
        tma_load_4d(dst, tm, b, 0, row, 0, hb, pol, p.l2hint != 0);
      };
      int g = 0;  // K/V blocks loaded so far (ring position across items)
      int it = 0;
      for (int item = blockIdx.x; item < items; item += gridDim.x, ++it) {
        int qt, hb;
        item_coords(p, item, nq, qt, hb);
        const int nall = blocks_of(qt, NT - 1);
        if (nall == 0) continue;
        if (it > 0) mbar_wait(bQEmpty, (it - 1) & 1);  // the previous item's S MMAs have read Q
        mbar_arrive_expect_tx(bQFull, NT * TILE);
        for (int t = 0; t < NT; ++t) {
          ld(sQ + t * TILE, &tmQ, bQFull, qt * BQ * NT + BQ * t, hb);
        }
        for (int j = 0; j < nall; ++j, ++g) {
          const int s = g & 1;
          const int k0 = j * BKV;
          mbar_wait(bKEmpty + 8 * s, ((g >> 1) & 1) ^ 1);
          mbar_arrive_expect_tx(bKFull + 8 * s, TILE);
          ld(sK + s * TILE, &tmK, bKFull + 8 * s, k0, hb);
          mbar_wait(bVEmpty + 8 * s, ((g >> 1) & 1) ^ 1);
          mbar_arrive_expect_tx(bVFull + 8 * s, TILE);
          ld(sV + s * TILE, &tmV, bVFull + 8 * s, k0, hb);
        }
      }
    } else if (warp == W_MMA && lane == 0) {
      // ---------------------------------------------------------------- MMA issuer
      constexpr uint32_t ID_S = idesc<DT, false>(), ID_PV = idesc<DT, true>();
      int g = 0;            // K/V ring position
      int gt[NT] = {0, 0};  // blocks issued per tile so far (S / P / O barrier phases)
      int it = 0;
      for (int item = blockIdx.x; item < items; item += gridDim.x, ++it) {
        int qt, hb;
        item_coords(p, item, nq, qt, hb);
        int nkv[NT];
#pragma unroll
        for (int t = 0; t < NT; ++t) nkv[t] = blocks_of(qt, t);
        const int nall = nkv[NT - 1];
        if (nall == 0) continue;
        auto issue_s = [&](int t, int j) {
          const uint32_t k = sK + ((g + j) & 1) * TILE, q = sQ + t * TILE;
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const uint32_t off = (kk >> 2) * ATOM + (kk & 3) * 32;
            mma_f16<1>(tmem + TM_S + t * 128, sdesc_sw128(q + off, 16, 1024), sdesc_sw128(k + off, 16, 1024), ID_S,
                       kk > 0);
          }
          mma_commit<1>(bSFull + 8 * t, 0);
        };
        auto issue_pv = [&](int t, int j) {
          mbar_wait(bPReady + 8 * t, (gt[t] + j) & 1);
          tc_fence_after();
          const uint32_t v = sV + ((g + j) & 1) * TILE;
#pragma unroll
          for (int kk = 0; kk < BKV / 16; ++kk)
            mma_f16_ts(tmem + TM_O + t * 128, tmem + TM_S + t * 128 + kk * 8, sdesc_sw128(v + kk * 2048, ATOM, 1024),
                       ID_PV, (j | kk) != 0);
          mma_commit<1>(bOReady + 8 * t, 0);
        };
        mbar_wait(bQFull, it & 1);
        mbar_wait(bKFull + 8 * (g & 1), (g >> 1) & 1);
        tc_fence_after();
        for (int t = 0; t < NT; ++t)
          if (nkv[t] > 0) issue_s(t, 0);
        mma_commit<1>(bKEmpty + 8 * (g & 1), 0);
        if (nall == 1) mma_commit<1>(bQEmpty, 0);  // Q read for the last time
        for (int j = 0; j < nall; ++j) {
          const bool next = j + 1 < nall;
          if (next) {
            mbar_wait(bKFull + 8 * ((g + j + 1) & 1), ((g + j + 1) >> 1) & 1);
            tc_fence_after();
          }
          mbar_wait(bVFull + 8 * ((g + j) & 1), ((g + j) >> 1) & 1);
          tc_fence_after();
#pragma unroll
          for (int t = 0; t < NT; ++t) {
            if (j < nkv[t]) {
              if (j == 0 && it > 0) {  // O_t of the previous item has been read by its epilogue
                mbar_wait(bOFree + 8 * t, (it - 1) & 1);
                tc_fence_after();
              }
              issue_pv(t, j);
            }
            if (t == NT - 1) mma_commit<1>(bVEmpty + 8 * ((g + j) & 1), 0);
            if (next && j + 1 < nkv[t]) issue_s(t, j + 1);
          }
          if (next) {
            mma_commit<1>(bKEmpty + 8 * ((g + j + 1) & 1), 0);
            if (j + 2 == nall) mma_commit<1>(bQEmpty, 0);  // the last S MMAs of this item are issued
          }
        }
        g += nall;
#pragma unroll
        for (int t = 0; t < NT; ++t) gt[t] += nkv[t];
      }
    }
  } else {
    // ---------------------------------------------------------------- softmax / epilogue
    asm volatile("setmaxnreg.inc.sync.aligned.u32 200;\n" ::: "memory");
    const int t = warp >> 2;
    const int q = warp & 3;
    const int r = 32 * q + lane;
    const uint32_t lane_base = uint32_t(32 * q) << 16;
    const uint32_t tS = tmem + lane_base + TM_S + t * 128;
    const uint32_t tO = tmem + lane_base + TM_O + t * 128;
    const uint32_t sE = sStage + warp * 4096;
    int gt = 0;  // this tile's blocks so far (barrier phases)
    int it = 0;
    for (int item = blockIdx.x; item < items; item += gridDim.x, ++it) {
      int qt, hb;
      item_coords(p, item, nq, qt, hb);
      if (blocks_of(qt, NT - 1) == 0) continue;  // (sk == 0 is handled on the host)
      const int nk = blocks_of(qt, t);
      const int trow0 = qt * BQ * NT + BQ * t;
      const int qrow = trow0 + r;
      float m = -INFINITY, l = 0.f;
      for (int j = 0; j < nk; ++j) {
        mbar_wait(bSFull + 8 * t, (gt + j) & 1);
        if (j > 0) mbar_wait(bOReady + 8 * t, (gt + j - 1) & 1);  // never blocks (in-order tcgen05)
        tc_fence_after();
        const int key0 = j * BKV;
        const bool full_block = (key0 + BKV <= p.sk) && (!p.causal || key0 + BKV - 1 <= trow0);
        uint32_t vrow[2][64];
        float mx8[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) mx8[u] = -INFINITY;
#pragma unroll
        for (int gg = 0; gg < 2; ++gg) {
          tmem_ld_32x32b_x32(tS + 64 * gg, *reinterpret_cast<uint32_t(*)[32]>(&vrow[gg][0]));
          tmem_ld_32x32b_x32(tS + 64 * gg + 32, *reinterpret_cast<uint32_t(*)[32]>(&vrow[gg][32]));
        }
        tmem_ld_wait();
        if (!full_block) {
#pragma unroll
          for (int gg = 0; gg < 2; ++gg)
#pragma unroll
            for (int e = 0; e < 64; ++e) {
              const int key = key0 + 64 * gg + e;
              if (key >= p.sk || (p.causal && key > qrow)) vrow[gg][e] = __float_as_uint(-INFINITY);
            }
        }
#pragma unroll
        for (int gg = 0; gg < 2; ++gg)
#pragma unroll
          for (int e = 0; e < 64; ++e) mx8[e & 7] = fmaxf(mx8[e & 7], __uint_as_float(vrow[gg][e]));
        float mb = fmaxf(fmaxf(fmaxf(mx8[0], mx8[1]), fmaxf(mx8[2], mx8[3])),
                         fmaxf(fmaxf(mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7])));
        mb = (mb == -INFINITY) ? -INFINITY : mb * p.scale_log2;
        float m_new = m, corr = 1.f;
        if (mb > m + 8.f) {
          m_new = mb;
          corr = ex2(m - m_new);
        }
        const float msub = (m_new == -INFINITY) ? 0.f : m_new;
        if (j > 0 && __any_sync(0xffffffffu, corr != 1.f)) {
#pragma unroll 1
          for (int c = 0; c < 4; ++c) {
            uint32_t o[32];
            tmem_ld_32x32b_x32(tO + 32 * c, o);
            tmem_ld_wait();
#pragma unroll
            for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * corr);
            tmem_st_32x32b_x32(tO + 32 * c, o);
          }
        }
        float2 sm4[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) sm4[u] = make_float2(0.f, 0.f);
        const float2 sc2 = make_float2(p.scale_log2, p.scale_log2);
        const float2 ms2 = make_float2(-msub, -msub);
#pragma unroll
        for (int gg = 0; gg < 2; ++gg) {
          uint32_t pk[32];
#pragma unroll
          for (int e = 0; e < 32; ++e) {
            const float2 x =
                ffma2(make_float2(__uint_as_float(vrow[gg][2 * e]), __uint_as_float(vrow[gg][2 * e + 1])), sc2, ms2);
            float2 pe;
            pe.x = ex2(x.x);
            pe.y = ex2(x.y);
            sm4[e & 3] = fadd2(sm4[e & 3], pe);
            pk[e] = pack2<DT>(pe.x, pe.y);
          }
          tmem_st_32x32b_x32(tS + 32 * gg, pk);  // P over columns [0, 64) (scores already in registers)
        }
        tmem_st_wait();
        l = l * corr + (((sm4[0].x + sm4[0].y) + (sm4[1].x + sm4[1].y)) +
                        ((sm4[2].x + sm4[2].y) + (sm4[3].x + sm4[3].y)));
        m = m_new;
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(bPReady + 8 * t);
      }
      // ---------------------------------------------------------------- epilogue of this item
      const float inv_l = (l > 0.f) ? 1.f / l : 0.f;
      if (nk > 0) {
        mbar_wait(bOReady + 8 * t, (gt + nk - 1) & 1);
        tc_fence_after();
      }
#pragma unroll 1
      for (int c = 0; c < 2; ++c) {
        uint32_t a0[32], a1[32];
        if (nk > 0) {
          tmem_ld_32x32b_x32(tO + 64 * c, a0);
          tmem_ld_32x32b_x32(tO + 64 * c + 32, a1);
          tmem_ld_wait();
        } else {
#pragma unroll
          for (int e = 0; e < 32; ++e) a0[e] = a1[e] = 0u;
        }
        if (c == 1) {  // O_t is in registers: the next item's first PV_t may overwrite it
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(bOFree + 8 * t);
        }
        if (lane == 0) bulk_wait_read<0>();  // the staging buffer's previous store has read it
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
          tma_store_3d(&tmO, sE, 64 * c, trow0 + 32 * q, hb);
          bulk_commit();
        }
      }
      if (p.lse && qrow < p.sq)
        p.lse[(size_t)hb * p.sq + qrow] = (l > 0.f) ? (m + __log2f(l)) * 0.6931471805599453f : -INFINITY;
      gt += nk;
    }
    if (lane == 0) bulk_wait_read<0>();
  }
  __syncwarp();
  tc_fence_before();
  __syncthreads();
  if (warp == W_MMA) {
    tc_fence_after();
    tmem_dealloc<1>(tmem, 512);
  }
}

// ============================================================================ CTA-pair kernel
// Two CTAs of a cluster own 256 consecutive query rows of one (batch, head), 128 rows each, and
// issue every MMA as one cta_group::2 instruction (M = 256): the leader's MMA thread computes
//   S(j) = Q K_j^T  into a double-buffered score tile (TMEM S[j % 2]) of both CTAs, and
//   O   += P(j) V_j with P read from TMEM columns of its own (not aliased with S).
// K_j and V_j are split between the pair (each CTA loads 64 keys of K_j and 64 columns of V_j),
// so every byte of K/V in shared memory serves 256 query rows, as in the two-tile kernel above.
// Because P has its own columns and S is double-buffered, S(j+2) is issued as soon as both CTAs'
// softmax warps have read S(j) -- the tensor core computes the next scores and the previous P.V
// while the SIMT warps run the softmax of block j (the FA3 overlap, without the
// S -> P -> PV -> S chain of the single-buffered layout).
//
// Warps 0-7: softmax.  Warp w owns TMEM lanes 32 (w % 4) .. +31 (= query rows) and score columns
// [64 (w / 4), +64): each thread holds 64 scores of its row; the two halves of a row combine their
// maxima through shared memory (64-thread named barrier).  Warp 8: TMA producer.  Warp 9: MMA.
// TMEM (each CTA): S0 [0,128) S1 [128,256) O [256,384) P [384,448).
namespace pr {
constexpr int KS = 4, VS = 4;                   // K / V ring depths
constexpr int Q_BYTES = 128 * 128 * 2;          // this CTA's 128 query rows (two 64-column atoms)
constexpr int QATOM = 128 * 128;                // 128 rows x 64 elements x 2 B
constexpr int KATOM = 64 * 128;                 // 64 keys x 64 elements x 2 B
constexpr int K_BYTES = 2 * KATOM;              // this CTA's 64 keys x 128
constexpr int V_BYTES = 128 * 128;              // 128 keys x this CTA's 64 columns
constexpr int OFF_Q = 0, OFF_K = Q_BYTES, OFF_V = OFF_K + KS * K_BYTES, OFF_BAR = OFF_V + VS * V_BYTES;
constexpr int OFF_X = OFF_BAR + 512;            // row-max exchange [2 parities][4 parts][128], l [4][128]
constexpr int SMEM_BYTES = 1024 + OFF_X + (2 * 4 * 128 + 4 * 128) * 4;
// NS = number of softmax warps sharing one row (column split): 2 (64 columns each) or 4 (32 each).
template <int NS> __host__ __device__ constexpr int softmax_warps() { return 4 * NS; }
template <int NS> __host__ __device__ constexpr int threads() { return (softmax_warps<NS>() + 2) * 32; }
constexpr uint32_t T_S = 0, T_O = 256, T_P = 384;

template <int DT, bool B_MN>
__host__ __device__ constexpr uint32_t idesc() {  // M = 256 (cta pair), N = 128, f32 accumulate
  return (1u << 4) | (uint32_t(DT) << 7) | (uint32_t(DT) << 10) | ((B_MN ? 1u : 0u) << 16) |
         (uint32_t(128 >> 3) << 17) | (uint32_t(256 >> 4) << 24);
}
// O[tmem] (+)= P[tmem] * V[smem desc], cta_group::2
__device__ __forceinline__ void mma_ts_pair(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc,
                                            uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
}  // namespace pr

template <int DT, int EMU, int NS>
__global__ void __launch_bounds__(pr::threads<NS>(), 1)
    attn_pair_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                     const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmO,
                     const Params p) {
  using namespace pr;
  constexpr int SW = softmax_warps<NS>();
  constexpr int W_PROD = SW, W_MMA = SW + 1;
  static_assert(NS == 2 || NS == 4, "row split into 2 or 4 column parts");
  constexpr int COLS = 128 / NS;  // score / output columns per softmax thread
  constexpr int PER_BLOCK = SW;   // softmax warps per CTA that read each S block
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  const uint32_t sQ = base + OFF_Q, sK = base + OFF_K, sV = base + OFF_V;
  const uint32_t bar = base + OFF_BAR;
  const uint32_t bQFull = bar, bKFull = bar + 8, bKEmpty = bKFull + 8 * KS, bVFull = bKEmpty + 8 * KS,
                 bVEmpty = bVFull + 8 * VS, bSFull = bVEmpty + 8 * VS, bSFree = bSFull + 16, bPFull = bSFree + 16,
                 bPVDone = bPFull + 8, sTmemSlot = bPVDone + 32;
  // bPVDone[2]: PV(j) completion, by parity of j
  volatile uint32_t* tmem_slot = reinterpret_cast<volatile uint32_t*>(smem_raw + (sTmemSlot - raw));

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const int npairs = gridDim.x >> 1;
  const int pi = p.causal ? (npairs - 1 - int(blockIdx.x >> 1)) : int(blockIdx.x >> 1);  // heavy first
  const int hb = blockIdx.y;
  const int q0 = pi * 2 * BQ;                 // the pair's first query row
  const int trow0 = q0 + BQ * int(rank);      // this CTA's first query row
  const int n = blocks_for(p, q0 + 2 * BQ);   // key blocks the pair processes (both CTAs)

  if (warp == W_PROD && lane == 0) {
    prefetch_tmap(&tmQ);
    prefetch_tmap(&tmK);
    prefetch_tmap(&tmV);
    prefetch_tmap(&tmO);
    mbar_init(bQFull, 1);
    for (int s = 0; s < KS; ++s) {
      mbar_init(bKFull + 8 * s, 1);
      mbar_init(bKEmpty + 8 * s, 1);
    }
    for (int s = 0; s < VS; ++s) {
      mbar_init(bVFull + 8 * s, 1);
      mbar_init(bVEmpty + 8 * s, 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(bSFull + 8 * b, 1);
      mbar_init(bSFree + 8 * b, 2 * PER_BLOCK);  // the softmax warps of both CTAs that read S
      mbar_init(bPVDone + 8 * b, 1);
    }
    mbar_init(bPFull, 2 * PER_BLOCK);
    fence_mbar_init();
  }
  if (warp == W_MMA) {
    tmem_alloc<2>(sTmemSlot, 512);
    tmem_relinquish<2>();
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();
  if (threadIdx.x == 0) pdl_launch_dependents();

  if (warp == W_PROD) {
    // ---------------------------------------------------------------- producer (both CTAs)
    // Every load completes on the leader's barrier (cta_group::2 TMA); the leader arms each
    // barrier with the bytes of both CTAs.  Empty barriers are local (multicast MMA commits).
    if (lane == 0 && n > 0) {
      const uint64_t pol = policy_evict_last();
      if (rank == 0) mbar_arrive_expect_tx(bQFull, 2 * Q_BYTES);
      const uint32_t qb = mapa(bQFull, 0);
      auto ld = [&](uint32_t dst, const CUtensorMap* tm, uint32_t bar, int c0, int c1) {
        if (p.l2hint) tma_load_3d_pair(dst, tm, bar, c0, c1, hb, pol);
        else tma_load_3d_pair_nohint(dst, tm, bar, c0, c1, hb);
      };
      ld(sQ, &tmQ, qb, 0, trow0);
      ld(sQ + QATOM, &tmQ, qb, 64, trow0);
      for (int j = 0; j < n; ++j) {
        const int ks = j % KS, vs = j % VS;
        mbar_wait(bKEmpty + 8 * ks, ((j / KS) & 1) ^ 1);
        if (rank == 0) mbar_arrive_expect_tx(bKFull + 8 * ks, 2 * K_BYTES);
        const uint32_t kb = mapa(bKFull + 8 * ks, 0);
        const int key0 = j * BKV + 64 * int(rank);
        ld(sK + ks * K_BYTES, &tmK, kb, 0, key0);
        ld(sK + ks * K_BYTES + KATOM, &tmK, kb, 64, key0);
        mbar_wait(bVEmpty + 8 * vs, ((j / VS) & 1) ^ 1);
        if (rank == 0) mbar_arrive_expect_tx(bVFull + 8 * vs, 2 * V_BYTES);
        ld(sV + vs * V_BYTES, &tmV, mapa(bVFull + 8 * vs, 0), 64 * int(rank), j * BKV);
      }
    }
  } else if (warp == W_MMA) {
    // ---------------------------------------------------------------- MMA issuer (leader only)
    if (lane == 0 && rank == 0 && n > 0) {
      constexpr uint32_t ID_S = pr::idesc<DT, false>(), ID_PV = pr::idesc<DT, true>();
      auto issue_s = [&](int j) {
        const int ks = j % KS;
        mbar_wait(bKFull + 8 * ks, (j / KS) & 1);
        tc_fence_after();
        const uint32_t k = sK + ks * K_BYTES;
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk)
          mma_f16<2>(tmem + T_S + (j & 1) * 128, sdesc_sw128(sQ + (kk >> 2) * QATOM + (kk & 3) * 32, 16, 1024),
                     sdesc_sw128(k + (kk >> 2) * KATOM + (kk & 3) * 32, 16, 1024), ID_S, kk > 0);
        mma_commit<2>(bSFull + 8 * (j & 1), 0x3);
        mma_commit<2>(bKEmpty + 8 * ks, 0x3);
      };
      auto issue_pv = [&](int j) {
        mbar_wait(bPFull, j & 1);
        const int vs = j % VS;
        mbar_wait(bVFull + 8 * vs, (j / VS) & 1);
        tc_fence_after();
        const uint32_t v = sV + vs * V_BYTES;
#pragma unroll
        for (int kk = 0; kk < BKV / 16; ++kk)
          mma_ts_pair(tmem + T_O, tmem + T_P + kk * 8, sdesc_sw128(v + kk * 2048, V_BYTES, 1024), ID_PV,
                      (j | kk) != 0);
        mma_commit<2>(bPVDone + 8 * (j & 1), 0x3);
        mma_commit<2>(bVEmpty + 8 * vs, 0x3);
      };
      mbar_wait(bQFull, 0);
      tc_fence_after();
      issue_s(0);
      if (n > 1) issue_s(1);
      for (int j = 0; j < n; ++j) {
        if (j + 2 < n) {  // S buffer j % 2 is free once both CTAs' softmax warps have read S(j)
          mbar_wait(bSFree + 8 * (j & 1), (j >> 1) & 1);
          tc_fence_after();
          issue_s(j + 2);
        }
        issue_pv(j);
      }
    }
  } else {
    // ---------------------------------------------------------------- softmax / epilogue
    const int h = warp >> 2;        // column part (of NS)
    const int q = warp & 3;         // TMEM lane quarter
    const int r = 32 * q + lane;    // row within this CTA's tile = TMEM lane
    const int qrow = trow0 + r;
    const uint32_t lane_base = uint32_t(32 * q) << 16;
    const uint32_t tS = tmem + lane_base + T_S + COLS * h;
    const uint32_t tO = tmem + lane_base + T_O + COLS * h;
    const uint32_t tP = tmem + lane_base + T_P + (COLS / 2) * h;
    float* xmax = reinterpret_cast<float*>(smem_raw + (base + OFF_X - raw));
    float* xl = xmax + 2 * NS * BQ;
    const uint32_t bar_id = 1 + q;
    auto pair_sync = [&]() { asm volatile("bar.sync %0, %1;" ::"r"(bar_id), "r"(32 * NS) : "memory"); };
    const uint32_t sfree_leader = mapa(bSFree, 0), pfull_leader = mapa(bPFull, 0);
    float m = -INFINITY, l = 0.f;
    for (int j = 0; j < n; ++j) {
      const int b = j & 1;
      mbar_wait(bSFull + 8 * b, (j >> 1) & 1);
      tc_fence_after();
      uint32_t v[COLS];
#pragma unroll
      for (int c = 0; c < COLS / 32; ++c)
        tmem_ld_32x32b_x32(tS + 128 * b + 32 * c, *reinterpret_cast<uint32_t(*)[32]>(&v[32 * c]));
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(sfree_leader + 8 * b);  // S(j) is in registers
      const int key0 = j * BKV + COLS * h;
      const bool full_block = (j * BKV + BKV <= p.sk) && (!p.causal || j * BKV + BKV - 1 <= trow0);
      if (!full_block) {  // masked keys (ragged last block / causal diagonal) read as -inf
#pragma unroll
        for (int e = 0; e < COLS; ++e) {
          const int key = key0 + e;
          if (key >= p.sk || (p.causal && key > qrow)) v[e] = __float_as_uint(-INFINITY);
        }
      }
      float mx8[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) mx8[u] = -INFINITY;
#pragma unroll
      for (int e = 0; e < COLS; ++e) mx8[e & 7] = fmaxf(mx8[e & 7], __uint_as_float(v[e]));
      const float mh = fmaxf(fmaxf(fmaxf(mx8[0], mx8[1]), fmaxf(mx8[2], mx8[3])),
                             fmaxf(fmaxf(mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7])));
      float* xm = xmax + b * NS * BQ;
      xm[h * BQ + r] = mh;
      pair_sync();
      float mb = xm[r];  // every part combines the NS maxima in the same order
#pragma unroll
      for (int u = 1; u < NS; ++u) mb = fmaxf(mb, xm[u * BQ + r]);
      mb = (mb == -INFINITY) ? -INFINITY : mb * p.scale_log2;  // scale_log2 > 0 keeps the order
      // lazy rescaling (see the two-tile kernel): both halves see the same mb and decide alike
      float m_new = m, corr = 1.f;
      if (mb > m + 8.f) {
        m_new = mb;
        corr = ex2(m - m_new);  // 0 when m == -inf
      }
      const float msub = (m_new == -INFINITY) ? 0.f : m_new;
      float2 sm4[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) sm4[u] = make_float2(0.f, 0.f);
      const float2 sc2 = make_float2(p.scale_log2, p.scale_log2);
      const float2 ms2 = make_float2(-msub, -msub);
      uint32_t pk[COLS / 2];
      auto exps = [&](auto e_c) {
        constexpr int E = decltype(e_c)::value;
#pragma unroll
        for (int e = 0; e < COLS / 2; ++e) {
          const float2 x = ffma2(make_float2(__uint_as_float(v[2 * e]), __uint_as_float(v[2 * e + 1])), sc2, ms2);
          float2 pe;
          if ((e & 7) < E) {
            pe = ex2_emu2(x);
          } else {
            pe.x = ex2(x.x);
            pe.y = ex2(x.y);
          }
          sm4[e & 3] = fadd2(sm4[e & 3], pe);
          pk[e] = pack2<DT>(pe.x, pe.y);
        }
      };
      if (EMU > 0 && full_block)
        exps(std::integral_constant<int, EMU>{});
      else
        exps(std::integral_constant<int, 0>{});
      if (j > 0) {  // PV(j-1) done: P may be overwritten and O is stable for the rescale
        mbar_wait(bPVDone + 8 * ((j - 1) & 1), ((j - 1) >> 1) & 1);
        tc_fence_after();
        if (__any_sync(0xffffffffu, corr != 1.f)) {
#pragma unroll 1
          for (int c = 0; c < COLS / 32; ++c) {
            uint32_t o[32];
            tmem_ld_32x32b_x32(tO + 32 * c, o);
            tmem_ld_wait();
#pragma unroll
            for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * corr);
            tmem_st_32x32b_x32(tO + 32 * c, o);
          }
        }
      }
      if constexpr (COLS == 64) tmem_st_32x32b_x32(tP, pk);
      else tmem_st_32x32b<16>(tP, pk);
      tmem_st_wait();
      l = l * corr + (((sm4[0].x + sm4[0].y) + (sm4[1].x + sm4[1].y)) +
                      ((sm4[2].x + sm4[2].y) + (sm4[3].x + sm4[3].y)));
      m = m_new;
      tc_fence_before();  // P and the rescaled O before the leader's PV(j)
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(pfull_leader);
    }
    // ---------------------------------------------------------------- epilogue: O / l, lse
    xl[h * BQ + r] = l;
    pair_sync();
    float lt = xl[r];  // same order in every part
#pragma unroll
    for (int u = 1; u < NS; ++u) lt += xl[u * BQ + r];
    const float inv_l = (lt > 0.f) ? 1.f / lt : 0.f;
    if (n > 0) {
      mbar_wait(bPVDone + 8 * ((n - 1) & 1), ((n - 1) >> 1) & 1);
      tc_fence_after();
    }
    // staging: 32 rows x COLS columns per warp (COLS = 64: SW128 rows; COLS = 32: plain 64-B rows)
    const uint32_t sE = sQ + (h * 4 + q) * (32 * COLS * 2);  // Q is no longer read (all MMAs are done)
    uint32_t a[COLS];
    if (n > 0) {
#pragma unroll
      for (int c = 0; c < COLS / 32; ++c) tmem_ld_32x32b_x32(tO + 32 * c, *reinterpret_cast<uint32_t(*)[32]>(&a[32 * c]));
      tmem_ld_wait();
    } else {
#pragma unroll
      for (int e = 0; e < COLS; ++e) a[e] = 0u;
    }
#pragma unroll
    for (int vv = 0; vv < COLS / 8; ++vv) {
      uint32_t w[4];
#pragma unroll
      for (int u = 0; u < 4; ++u)
        w[u] = pack2<DT>(__uint_as_float(a[8 * vv + 2 * u]) * inv_l, __uint_as_float(a[8 * vv + 2 * u + 1]) * inv_l);
      if constexpr (COLS == 64) st_shared_v4(sE + lane * 128 + ((vv ^ (lane & 7)) << 4), w[0], w[1], w[2], w[3]);
      else st_shared_v4(sE + lane * 64 + (vv << 4), w[0], w[1], w[2], w[3]);
    }
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) {
      tma_store_3d(&tmO, sE, COLS * h, trow0 + 32 * q, hb);
      bulk_commit();
    }
    if (h == 0 && p.lse && qrow < p.sq)
      p.lse[(size_t)hb * p.sq + qrow] = (lt > 0.f) ? (m + __log2f(lt)) * 0.6931471805599453f : -INFINITY;
    if (lane == 0) bulk_wait_read<0>();
  }
  __syncwarp();
  tc_fence_before();
  cluster_sync();  // the peer's smem / TMEM are operands of the leader's MMAs until here
  if (warp == W_MMA) {
    tc_fence_after();
    tmem_dealloc<2>(tmem, 512);
  }
}

#endif  // CY_ATTN_EXPERIMENTS

// ------------------------------------------------------------------------------------------ host
std::once_flag g_once;
PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
std::mutex g_attr_mu;
bool g_attr_set[64][6][2][4] = {};
int g_sms[64] = {};

// {64 columns, rows, 2 column atoms, batch*head} with 128-row boxes of both atoms (one TMA op per tile)
bool make_map4(CUtensorMap* m, int dt, const void* ptr, uint64_t rows, uint64_t bh, uint32_t box_rows = 128) {
  cuuint64_t dims[4] = {64, rows, uint64_t(D) / 64, bh};
  cuuint64_t strides[3] = {uint64_t(D) * 2, 128, rows * uint64_t(D) * 2};
  cuuint32_t box[4] = {64, box_rows, uint32_t(D) / 64, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  return g_encode(m, dt == 0 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4,
                  const_cast<void*>(ptr), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
bool make_map(CUtensorMap* m, int dt, const void* ptr, uint64_t rows, uint64_t bh, uint32_t box_c, uint32_t box_r,
              bool swizzle = true) {
  cuuint64_t dims[3] = {uint64_t(D), rows, bh};
  cuuint64_t strides[2] = {uint64_t(D) * 2, rows * uint64_t(D) * 2};
  cuuint32_t box[3] = {box_c, box_r, 1};
  cuuint32_t es[3] = {1, 1, 1};
  return g_encode(m, dt == 0 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3,
                  const_cast<void*>(ptr), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  swizzle ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace cy_attn

#ifdef CY_ATTN_TRACE
extern "C" int cy_attn_trace(unsigned long long* out) {
  return (int)cudaMemcpyFromSymbol(out, cy_attn::g_attn_trace, sizeof(cy_attn::g_attn_trace));
}
#endif

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
  // grid: (query-tile pairs, batch*heads), or (batch*heads, query-tile pairs) for causal problems and
  // when batch*heads exceeds the 65535 limit of grid y
  if (seq_q > INT32_MAX || seq_k > INT32_MAX || bh > INT32_MAX) return CY_ERR_INVALID_VALUE;
  if (bh > 65535 && (seq_q + 2 * 128 - 1) / (2 * 128) > 65535) return CY_ERR_INVALID_VALUE;
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
#ifdef CY_ATTN_EXPERIMENTS
  // Experiment build only (scripts/build_experiment.py ... CY_ATTN_EXPERIMENTS=1): the variants
  // below measured slower than the default and are not in the product library.  Read per call:
  // CY_ATTN_KERNEL: 1 (default) the two-tile single-CTA kernel, 2 the CTA-pair kernel;
  // CY_ATTN_SPLIT: softmax warps per row group in the pair kernel, 2 (default) or 4.
  const int kern = [] {
    const char* e = std::getenv("CY_ATTN_KERNEL");
    return (e && std::atoi(e) == 2) ? 2 : 1;
  }();
  const int split = [] {
    const char* e = std::getenv("CY_ATTN_SPLIT");
    const int v = e ? std::atoi(e) : 2;
    return v == 4 ? 4 : 2;
  }();
#else
  const int kern = 1, split = 2;  // product: the two-tile kernel, default layout
#endif
  CUtensorMap tQ, tK, tV, tO;
  std::memset(&tK, 0, sizeof(tK));
  tV = tK;
  const bool o32 = kern == 2 && split == 4;  // 32-column output boxes, unswizzled staging
  // the two-tile kernels (kern 1) load Q / K / V tiles as one 4-D box each; the pair kernel keeps 3-D maps
  const bool four = (kern == 1);
  const uint32_t kv_rows = CY_ATTN_DB ? 64 : 128;  // K / V box rows (keys per block)
  bool ok = (four ? make_map4(&tQ, dt, Q, seq_q, bh) : make_map(&tQ, dt, Q, seq_q, bh, 64, 128)) &&
            make_map(&tO, dt, O, seq_q, bh, o32 ? 32 : 64, 32, !o32);
  if (seq_k > 0)
    ok = ok && (four ? make_map4(&tK, dt, K, seq_k, bh, kv_rows) && make_map4(&tV, dt, V, seq_k, bh, kv_rows)
                     : make_map(&tK, dt, K, seq_k, bh, 64, kern == 2 ? 64 : 128) && make_map(&tV, dt, V, seq_k, bh, 64, 128));
  if (!ok) return CY_ERR_LAUNCH;
  Params p;
  p.sq = (int)seq_q;
  p.sk = (int)seq_k;
  p.bh = (int)bh;
  p.causal = causal ? 1 : 0;
  p.scale_log2 = scale * 1.4426950408889634f;
  p.lse = lse;
  p.lpt = (((causal && CY_ATTN_LPT) || bh > 65535) && !CY_ATTN_DB && !CY_ATTN_T1) ? 1 : 0;
#ifdef CY_ATTN_EXPERIMENTS
  // CY_ATTN_L2HINT: 1 = evict_last hint on the Q/K/V TMA loads, 0 = none (tuning knob)
  p.l2hint = [] {
    const char* e = std::getenv("CY_ATTN_L2HINT");
    return e ? std::atoi(e) : 1;
  }();
  // CY_ATTN_EMU: how many of every 8 exponential pairs run on the FMA pipe (tuning knob; default 0).
  // Measured on B200 (scripts/mufu_probe.cu): MUFU.EX2 16/clk/SM, FFMA2 ~56 pairs/clk/SM (half
  // rate), so a cubic exp2 costs about as much FMA-pipe time as MUFU time: at most +12% on the
  // isolated softmax step and 2-5% slower inside both kernels.
  const int emu = [] {
    const char* e = std::getenv("CY_ATTN_EMU");
    const int v = e ? std::atoi(e) : 0;
    return (v == 0 || v == 2 || v == 3 || v == 4) ? v : 0;
  }();
  const void* fns[6][2][4] = {
      {{(const void*)&attn_fwd_kernel<0, 0>, (const void*)&attn_fwd_kernel<0, 2>,
        (const void*)&attn_fwd_kernel<0, 3>, (const void*)&attn_fwd_kernel<0, 4>},
       {(const void*)&attn_fwd_kernel<1, 0>, (const void*)&attn_fwd_kernel<1, 2>,
        (const void*)&attn_fwd_kernel<1, 3>, (const void*)&attn_fwd_kernel<1, 4>}},
      {{(const void*)&attn_pair_kernel<0, 0, 2>, (const void*)&attn_pair_kernel<0, 2, 2>,
        (const void*)&attn_pair_kernel<0, 3, 2>, (const void*)&attn_pair_kernel<0, 4, 2>},
       {(const void*)&attn_pair_kernel<1, 0, 2>, (const void*)&attn_pair_kernel<1, 2, 2>,
        (const void*)&attn_pair_kernel<1, 3, 2>, (const void*)&attn_pair_kernel<1, 4, 2>}},
      {{(const void*)&attn_pair_kernel<0, 0, 4>, (const void*)&attn_pair_kernel<0, 2, 4>,
        (const void*)&attn_pair_kernel<0, 3, 4>, (const void*)&attn_pair_kernel<0, 4, 4>},
       {(const void*)&attn_pair_kernel<1, 0, 4>, (const void*)&attn_pair_kernel<1, 2, 4>,
        (const void*)&attn_pair_kernel<1, 3, 4>, (const void*)&attn_pair_kernel<1, 4, 4>}},
      {{(const void*)&attn_fwd_kernel<0, 0, 2>, (const void*)&attn_fwd_kernel<0, 2, 2>,
        (const void*)&attn_fwd_kernel<0, 3, 2>, (const void*)&attn_fwd_kernel<0, 4, 2>},
       {(const void*)&attn_fwd_kernel<1, 0, 2>, (const void*)&attn_fwd_kernel<1, 2, 2>,
        (const void*)&attn_fwd_kernel<1, 3, 2>, (const void*)&attn_fwd_kernel<1, 4, 2>}},
      {{(const void*)&attn_fwd_kernel<0, 0, 3>, (const void*)&attn_fwd_kernel<0, 2, 3>,
        (const void*)&attn_fwd_kernel<0, 3, 3>, (const void*)&attn_fwd_kernel<0, 4, 3>},
       {(const void*)&attn_fwd_kernel<1, 0, 3>, (const void*)&attn_fwd_kernel<1, 2, 3>,
        (const void*)&attn_fwd_kernel<1, 3, 3>, (const void*)&attn_fwd_kernel<1, 4, 3>}},
      {{(const void*)&attn_persist_kernel<0>, nullptr, nullptr, nullptr},
       {(const void*)&attn_persist_kernel<1>, nullptr, nullptr, nullptr}}};
  const int ei = emu == 0 ? 0 : emu - 1;
  // CY_ATTN_CS: two-tile kernel softmax layout: 3 (default) one warp per row, 12 warps with
  // setmaxnreg so each row stays in registers (one TMEM pass); 1 the same with 10 warps and two
  // TMEM passes; 2 two warps per row, both tiles in turn
  const int cs = [] {
    const char* e = std::getenv("CY_ATTN_CS");
    const int v = e ? std::atoi(e) : 3;
    return (v == 1 || v == 2) ? v : 3;
  }();
  // CY_ATTN_PERSIST=1: the default layout as a persistent kernel (one CTA per SM walking the work
  // items, static round-robin).  Measured -2 % non-causal at 8192, +2 % at 2048, -8..12 % causal
  // (static schedule, uneven items), so off by default.  Not used with EMU or seq_k == 0.
  const int persist = [] {
    const char* e = std::getenv("CY_ATTN_PERSIST");
    return e ? std::atoi(e) : 0;
  }();
  const bool ps = kern == 1 && cs == 3 && emu == 0 && persist && seq_k > 0;
  const int ki = ps ? 5 : kern == 1 ? (cs == 2 ? 3 : cs == 3 ? 4 : 0) : (split == 2 ? 1 : 2);
  const void* fn = fns[ki][dt][ps ? 0 : ei];
#else
  p.l2hint = 1;  // evict_last on Q/K/V (measured: without it causal 16384 loses 6 %)
  constexpr int ki = 4, ei = 0;
  const int cs = 3;
#if CY_ATTN_T1
  const void* fn = dt == CY_F16 ? (const void*)&attn_t1_kernel<0> : (const void*)&attn_t1_kernel<1>;
#elif CY_ATTN_DB
  const void* fn = dt == CY_F16 ? (const void*)&attn_db_kernel<0> : (const void*)&attn_db_kernel<1>;
#else
  const void* fn = dt == CY_F16 ? (const void*)&attn_fwd_kernel<0, 0, 3> : (const void*)&attn_fwd_kernel<1, 0, 3>;
#endif
#endif
#ifdef CY_ATTN_EXPERIMENTS
  const int smem = kern == 2 ? pr::SMEM_BYTES : ps ? PS_SMEM_BYTES : (kern == 1 && cs == 3) ? SMEM_BYTES3 : SMEM_BYTES;
#else
#if CY_ATTN_T1
  const int smem = t1::SMEM_BYTES;
#elif CY_ATTN_DB
  const int smem = db::SMEM_BYTES;
#else
  const int smem = SMEM_BYTES3;
#endif
#endif
  {
    std::lock_guard<std::mutex> lk(g_attr_mu);
    if (!g_attr_set[dev][ki][dt][ei]) {
      if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess) {
        cudaGetLastError();
        return CY_ERR_LAUNCH;
      }
      g_attr_set[dev][ki][dt][ei] = true;
    }
    if (g_sms[dev] == 0) cudaDeviceGetAttribute(&g_sms[dev], cudaDevAttrMultiProcessorCount, dev);
  }
  cudaLaunchConfig_t cfg;
  std::memset(&cfg, 0, sizeof(cfg));
  cudaLaunchAttribute attrs[2];
  attrs[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attrs[0].val.programmaticStreamSerializationAllowed = 1;
#ifdef CY_ATTN_EXPERIMENTS
  if (kern == 2) {
    cfg.gridDim = dim3((unsigned)(2 * ((seq_q + 2 * BQ - 1) / (2 * BQ))), (unsigned)bh, 1);
    cfg.blockDim = dim3(split == 2 ? pr::threads<2>() : pr::threads<4>(), 1, 1);
    attrs[1].id = cudaLaunchAttributeClusterDimension;
    attrs[1].val.clusterDim.x = 2;
    attrs[1].val.clusterDim.y = 1;
    attrs[1].val.clusterDim.z = 1;
    cfg.numAttrs = 2;
  } else if (ps) {
    const int64_t items = ((seq_q + BQ * NT - 1) / (BQ * NT)) * bh;
    cfg.gridDim = dim3((unsigned)std::min<int64_t>(items, std::max(1, g_sms[dev])), 1, 1);
    cfg.blockDim = dim3(384, 1, 1);
    cfg.numAttrs = 1;
  } else
#endif
  {
    const unsigned nq = (unsigned)((seq_q + BQ * (CY_ATTN_T1 ? 1 : NT) - 1) / (BQ * (CY_ATTN_T1 ? 1 : NT)));
    cfg.gridDim = p.lpt ? dim3((unsigned)bh, nq, 1) : dim3(nq, (unsigned)bh, 1);
    cfg.blockDim = dim3(cs == 3 ? 384 : THREADS, 1, 1);
    cfg.numAttrs = 1;
  }
  cfg.dynamicSmemBytes = smem;
  cfg.stream = static_cast<cudaStream_t>(stream);
  cfg.attrs = attrs;
  void* args[] = {&tQ, &tK, &tV, &tO, &p};
  if (cudaLaunchKernelExC(&cfg, fn, args) != cudaSuccess) {
    cudaGetLastError();
    return CY_ERR_LAUNCH;
  }
  cy_internal::note_launch();
  return CY_OK;
}
