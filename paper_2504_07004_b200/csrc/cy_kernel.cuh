// cy_kernel.cuh -- the sm_100a GEMM-family kernel: persistent, warp-specialised, TMA-fed,
// tcgen05.mma into TMEM, optional CTA pairs (cta_group::2), fused epilogue.
//
// One template covers the four entry points of include/cypress_b200.h:
//   V_GEMM       D  = alpha*A.B + beta*C                 (batched P:1520-1521)
//   V_DUAL_PAIR  D0 = alpha*A.B0 + beta*C0, D1 = alpha*A.B1 + beta*C1   (GLU core)
//   V_DUAL_SUM   D  = alpha*(A.B0 + A.B1) + beta*C
//   V_ROWREDUCE  D  = alpha*A.B + beta*C and y(i) = sum_k A(i,k)
//   V_DUAL_GLU   D  = act(alpha*A.B0) * (alpha*A.B1), act = SiLU | GELU-tanh   (GLU)
//
// Structure (the B200 re-derivation of the paper's warp-specialised, pipelined Hopper kernel,
// Fig. 3b, and of the passes' end state):
//   warp 0      producer: one lane drives TMA into an S-stage shared-memory ring (full/empty
//               mbarriers with phase bits = the paper's modulo-indexed buffers + backwards WAR
//               events).
//   warp 1      MMA issuer: one lane issues tcgen05.mma (M = 128*CG, N = BN, K = 16) into a TMEM
//               accumulator (never materialised whole elsewhere -- the paper's NONE memory,
//               P:675-683), commits stage releases and "accumulator full" to mbarriers.
//   warps 2-5   epilogue: TMEM -> registers (tcgen05.ld 32x32b) -> alpha/beta/cast in fp32 ->
//               swizzled shared staging -> per-warp TMA store; double-buffered accumulators let
//               tile i's epilogue overlap tile i+1's main loop.
//   warps 6-9   (V_ROWREDUCE only) SIMT row-sum of the A stages while the tensor core runs
//               (P:1580-1581); the fp32 accumulator lives in registers.
// Tiles (prange(cdiv(M,U), cdiv(N,V))) are scheduled persistently, one CTA (pair)
// per SM (pair), statically strided, grouped along M for L2 reuse.  CG == 2 pairs two SMs on
// one 256-row tile: each CTA loads its half of A and half of B, the leader issues
// tcgen05.mma.cta_group::2 (the "larger tensor core shared by pairs of SMs").
#pragma once
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "cy_ptx.cuh"

// CY_DEBUG_MODE: timing experiments only (results INVALID): 1 = no TMA refill, 2 = no epilogue,
// 4 = no D stores, 8 = TMEM loads only.  Compile-time only: the product library is always built
// with 0 (nothing at run time can switch it on); scripts/build_experiment.py builds a separate
// library with it set.
#ifndef CY_DEBUG_MODE
#define CY_DEBUG_MODE 0
#endif
// CY_MUTANT (scripts/mutants.sh only, never the product): one deliberate bug per value, to check
// that the parity tests catch it -- 1 the epilogue drops beta*C on each warp's last chunk, 2 split-K
// reduces one split too few, 3 the row reducers skip the last k-block, 4 (attention) the speculative
// softmax keeps its P when a row's max grows, 5 the epilogue writes (and reads C) at the next
// n-block's columns.
#ifndef CY_MUTANT
#define CY_MUTANT 0
#endif
// CY_C_FIRST: beta != 0 with one staging slot per epilogue warp: fetch the tile's first C chunk while
// the main loop runs
#ifndef CY_C_FIRST
#define CY_C_FIRST 1
#endif

// CY_GEMM_TRACE (timing experiments only, never in the product build): clock64() stamps of one
// CTA's per-tile events (scripts/gemm_trace.py reads them with cy_gemm_trace_read()).
#ifdef CY_GEMM_TRACE
#ifndef CY_GEMM_TRACE_CTA
#define CY_GEMM_TRACE_CTA 0
#endif
__device__ unsigned long long g_gemm_trace[64 * 16];
#define CY_TR(it, ev)                                                                      \
  do {                                                                                     \
    if (blockIdx.x == CY_GEMM_TRACE_CTA && (it) < 64) g_gemm_trace[(it) * 16 + (ev)] = clock64(); \
  } while (0)
#define CY_TR_ADD(it, ev, v)                                                               \
  do {                                                                                     \
    if (blockIdx.x == CY_GEMM_TRACE_CTA && (it) < 64 && (threadIdx.x & 31) == 0) g_gemm_trace[(it) * 16 + (ev)] += (v); \
  } while (0)
// kernel-level events of every CTA (< 1024): clock64 per event, globaltimer at entry
__device__ unsigned long long g_gemm_ktrace[1024 * 8];
__device__ unsigned long long g_gemm_gtime[1024];
#define CY_KT(ev)                                                            \
  do {                                                                       \
    if (blockIdx.x < 1024) g_gemm_ktrace[blockIdx.x * 8 + (ev)] = clock64(); \
  } while (0)
// MMA issuer of CTA CY_GEMM_TRACE_CTA, first tile: [k-block][0 = stage full seen, 1 = its MMAs issued]
__device__ unsigned long long g_gemm_mtrace[64 * 4];
#define CY_MT(it, kb, ev)                                                                      \
  do {                                                                                         \
    if (blockIdx.x == CY_GEMM_TRACE_CTA && (it) == 0 && (kb) < 64) g_gemm_mtrace[(kb) * 4 + (ev)] = clock64(); \
  } while (0)
// epilogue chunk timeline of CTA CY_GEMM_TRACE_CTA, first tile: [warp][chunk][event]
__device__ unsigned long long g_gemm_etrace[8 * 8 * 8];
#define CY_ET(it, ew, q, ev)                                                                  \
  do {                                                                                        \
    if (blockIdx.x == CY_GEMM_TRACE_CTA && (it) == 0 && (q) < 8 && lane == 0)                 \
      g_gemm_etrace[((ew) * 8 + (q)) * 8 + (ev)] = clock64();                                 \
  } while (0)
#else
#define CY_ET(it, ew, q, ev) \
  do {                       \
  } while (0)
#define CY_MT(it, kb, ev) \
  do {                    \
  } while (0)
#define CY_KT(ev) \
  do {            \
  } while (0)
#define CY_TR(it, ev) \
  do {                \
  } while (0)
#define CY_TR_ADD(it, ev, v) \
  do {                       \
  } while (0)
#endif

namespace cy {

constexpr int kDebug = CY_DEBUG_MODE;
// Experiment paths switched by Params fields the host sets only in CY_TUNING_KNOBS builds (L2
// prefetch of later batches, C-tile L2 prefetch, D-store L2 policy): compiled out of the product.
#ifdef CY_TUNING_KNOBS
constexpr bool kTuning = true;
#else
constexpr bool kTuning = false;
#endif

enum Variant : int { V_GEMM = 0, V_DUAL_PAIR = 1, V_DUAL_SUM = 2, V_ROWREDUCE = 3, V_DUAL_GLU = 4 };

struct Params {
  int M, N, K, L;        // problem (L = batch count)
  float alpha, beta;
  int has_c;             // beta != 0: C is read
  int m_blocks, n_blocks, k_blocks;
  int tiles;             // L * m_blocks * n_blocks
  int group_m;           // grouped rasterisation width (in m-blocks)
  int l2_policy;         // TMA L2 hints for A/B: 0 normal/normal, 1 last/last, 2 first/first, 3 first/last,
                         // 4 last/first, 5 none/none, 6 none/last, 7 last/none
  int raster;            // 0: groups of group_m m-blocks, m fastest (A panels resident, B streams);
                         // 1: groups of group_m n-blocks, n fastest (B panels resident, A streams)
  float* y;              // V_ROWREDUCE: y[M]
  int act;               // V_DUAL_GLU: 0 = SiLU, 1 = GELU (tanh form)
  int n_extra;           // number of extra D destinations in DstMaps (0 = D only)
  int a_reuse;           // 1: two-slot k-blocks interleave MMAs with the A collector buffer
  int sleep_ns;          // >0: epilogue waits for the accumulator with nanosleep backoff (cap, ns)
  int splits;            // split-K (V_GEMM, one accumulator): CTA (pair) s of a cluster of `splits`
                         // CTAs (pairs) takes k-blocks [s*kb_split, (s+1)*kb_split) of the cluster's tile
  int kb_split;          // k-blocks per split (the last split may hold fewer; every split holds >= 1)
  float* ws;             // split-K: fp32 partial slices (cy_gemm_splitk workspace)
  int dyn;               // 1: dynamic tile schedule (one cluster launched per tile, running clusters steal
                         //    pending ones with clusterlaunchcontrol.try_cancel); 0: static stride;
                         // 2: one cluster per tile, no stealing (non-persistent)
  int a4d;               // 1 (BK = 128): A is a 4-D map {64, rows, K / 64, batch} (K % 64 == 0): one op per stage
  int b4d;               // 1: B (and B1) tensor maps are 4-D {64 cols, K, N/64 atoms, batch} (N % 64 == 0):
                         //    one TMA op per B slot instead of one per 64-column atom
  int serp;              // 1: odd raster groups sweep the n-blocks in reverse (boustrophedon), so a
                         //    group starts on the B panels its predecessor just read
  // Batched L2 prefetch (pf_dist > 0): the CTA (pair leader) running tile r of problem b prefetches
  // slice r (of m_blocks * n_blocks) of problem b + pf_dist's A and B spans into L2, so the tiles
  // of that problem find their operands in L2 instead of waiting on HBM.
  int pf_dist;
  int d_policy;          // L2 policy of the D stores: 0 none, 1 evict_first, 2 evict_last
  int c_pf;              // beta != 0: each epilogue warp prefetches its chunks' C tiles into L2 when it
                         // learns its next tile (during that tile's main loop)
  const char* pf_a;      // A of problem 0 (span: pf_a_bytes from pf_a + b * pf_a_stride)
  const char* pf_b;
  long long pf_a_stride, pf_b_stride;
  long long pf_a_bytes, pf_b_bytes;
};

// Extra destinations of every D tile (fused replication): tensor maps over this
// shard's row block of the replicated D on other GPUs (peer memory mapped into this process).
constexpr int kMaxExtraDst = 7;
struct DstMaps {
  CUtensorMap m[kMaxExtraDst];
};

constexpr int pow2_cols(int c) { return c <= 32 ? 32 : c <= 64 ? 64 : c <= 128 ? 128 : c <= 256 ? 256 : 512; }

template <int DT_, int CG_, int BN_, int STAGES_, int VAR_, int NSUB_ = 1, int MC_ = 1, int BK_ = 64, int MX_ = 0>
struct Cfg {
  static constexpr int DT = DT_;  // 0 = fp16, 1 = bf16
  static constexpr int CG = CG_;  // CTAs per MMA (tcgen05 cta_group)
  static constexpr int BN = BN_;  // MMA N (one accumulator's width)
  static constexpr int STAGES = STAGES_;
  static constexpr int VAR = VAR_;
  static constexpr int NSUB = NSUB_;          // GEMM: N sub-tiles per tile sharing each A stage
  // MC = 2: a cluster of two CTA pairs stacked along M shares every B stage: each CTA loads half
  // of its B atoms and multicasts them to the CTA at the same position in the other pair, so a
  // 512 x TILE_N cluster tile reads B from L2 once (SURVEY a4 "cluster TMA multicast").
  static constexpr int MC = MC_;
  // MX = 1: a 2 x 2 cluster of single CTAs (cta_group::1, K = 128 per stage) whose cluster tile is
  // 256 x 2*BN: the two CTAs on the same rows each load one K-atom of the A stage and multicast it to
  // both, the two CTAs on the same columns each load one 64-row K half of the B stage and multicast
  // it to both, so every CTA issues half of its operand bytes (the per-SM TMA feed, not the tensor
  // core, bounds the narrow tiles of few-tile problems)
  static constexpr int MX = MX_;
  static constexpr int CL = MX ? 4 : CG * MC;  // cluster size
  static constexpr bool DUAL = (VAR == V_DUAL_PAIR || VAR == V_DUAL_SUM || VAR == V_DUAL_GLU);
  static constexpr bool GLU = (VAR == V_DUAL_GLU);
  static constexpr int BM_CTA = 128;          // accumulator rows per CTA = TMEM lanes
  static constexpr int BM = BM_CTA * CG;      // MMA M = output tile height
  static constexpr int TILE_N = DUAL ? BN : NSUB * BN;  // output tile width
  // K per stage: 64 (one 128-byte swizzle atom) or 128 (two K-atoms, 16 KB apart for A, one box
  // each for A and every B slot: half the TMA ops per byte, which sets the per-SM TMA rate)
  static constexpr int BK = BK_;
  static constexpr int KAT = BK / 64;         // K-atoms per stage
  static constexpr int A_ATOM = BM_CTA * 128;  // one 64-element K-atom of the CTA's A rows (16 KB)
  static constexpr int UMMA_K = 16;
  static constexpr int NUM_B = DUAL ? 2 : NSUB;  // B slots per stage
  static constexpr int NUM_ACC = (VAR == V_DUAL_PAIR || GLU) ? 2 : (VAR == V_DUAL_SUM ? 1 : NSUB);
  static constexpr int NUM_OUT = GLU ? 1 : NUM_ACC;  // output tiles the epilogue writes per tile
  static constexpr int BN_CTA = BN / CG;      // B columns held per CTA
  static constexpr int A_BYTES = BM_CTA * BK * 2;
  static constexpr int B_BYTES = BN_CTA * BK * 2;
  static constexpr int B_ATOM_BYTES = BK * 128;  // 64 K-rows x 64 N-columns (128 B) per TMA box
  static constexpr int STAGE_BYTES = A_BYTES + NUM_B * B_BYTES;
  static constexpr int ACC_COLS = NUM_ACC * BN;
  static constexpr int NUM_ACC_BUF = (2 * ACC_COLS <= 512) ? 2 : 1;
  static constexpr int TMEM_COLS = pow2_cols(NUM_ACC_BUF * ACC_COLS);
  // Single-buffered accumulators (TMEM full) leave the epilogue exposed: give it two warps per
  // TMEM lane quarter (each takes every other 64-column chunk) and one staging buffer each.
  // (Measured and not kept: the same split for double-buffered 256 x 256 tiles, which shortens the
  // last tile's epilogue -- 2048^3 -1.6 % time, batched 64 x 1024^3 on 256 x 256 +3 %, 1-CTA
  // 128 x 256 tiles +5..10 %: the 320-thread build caps registers at 168 and spills.)
  static constexpr int EPI_SPLIT = (NUM_ACC_BUF == 1) ? 2 : 1;
  static constexpr int EPI_WARPS = 4 * EPI_SPLIT;
  static constexpr int EPI_BUFS = (EPI_SPLIT == 2) ? 1 : 2;
  static constexpr int RED_WARPS = (VAR == V_ROWREDUCE) ? 4 : 0;
  static constexpr int THREADS = 32 * (2 + EPI_WARPS + RED_WARPS);
  static constexpr int EPI_BUF_BYTES = 32 * 128;  // 32 rows x 64 columns x 2 B
  static constexpr int EPI_BYTES = EPI_WARPS * EPI_BUFS * EPI_BUF_BYTES;
  static constexpr int BAR_BYTES = 512;
  static constexpr int SCHED_SLOTS = 4;       // tile-ID ring depth (dynamic schedule)
  static constexpr int NUM_WARPS = THREADS / 32;
  static constexpr int SMEM_BYTES = 1024 + STAGES * STAGE_BYTES + EPI_BYTES + BAR_BYTES;
  // split-K across the CTAs (pairs) of a cluster: plain GEMM tiles with one accumulator
  static constexpr bool SPLITTABLE = (VAR == V_GEMM && MC == 1 && NSUB == 1 && MX == 0);
  static_assert(24 * STAGES + 232 + 8 * EPI_WARPS <= BAR_BYTES, "barrier region");
  // Row-reduce: the reducer warps learn that their CTA's A stage is in shared memory from a
  // second tcgen05.commit (bMDone, multicast to both CTAs of a pair) issued after the MMAs that
  // read the stage; the stage is released only when the MMAs and the reducers are both done.
  static constexpr bool REDUCE = (VAR == V_ROWREDUCE);
  // Single-buffered TMEM with two accumulators: the epilogue releases them one at a time and the
  // MMA issuer starts the next tile on accumulator 0 while accumulator 1 drains.
  static constexpr bool SPLIT = (NUM_ACC_BUF == 1 && NUM_ACC == 2 && !GLU);

  static_assert(BN % 64 == 0 && BN_CTA % 64 == 0, "B is loaded in 64-column swizzle atoms");
  static_assert(BK == 64 || (BK == 128 && MC == 1), "K per stage: 64, or 128 without B multicast");
  static_assert(MX == 0 || (CG == 1 && MC == 1 && BK == 128 && NSUB == 1 && VAR == V_GEMM && BN == 64),
                "2 x 2 multicast cluster: single-CTA GEMM tiles of 128 x 64 with K = 128 stages");
  // cluster tile (rows x columns) and the scheduler's block sizes
  static constexpr int CT_M = MX ? 2 * BM : BM * MC;
  static constexpr int CT_N = MX ? 2 * TILE_N : TILE_N;
  static_assert(BN >= 64 && BN <= 256, "tcgen05 kind::f16 N range");
  static_assert(SMEM_BYTES <= 232448, "exceeds 227 KB of dynamic shared memory");
  static_assert(NUM_ACC_BUF * ACC_COLS <= 512, "TMEM has 512 columns");
  static_assert(!DUAL || NSUB == 1, "dual GEMM uses its two B slots for B0/B1");
  static_assert(MC == 1 || (MC == 2 && CG == 2 && VAR == V_GEMM && (NUM_B * BN_CTA / 64) % 2 == 0),
                "B multicast: GEMM on CTA pairs with an even number of B atoms per stage");

  // Instruction descriptor, kind::f16: c_format F32 [4,6) | a_format [7,10) | b_format [10,13) |
  // a_major K (bit 15 = 0) | b_major MN (bit 16 = 1) | N>>3 [17,23) | M>>4 [24,29).
  static constexpr uint32_t IDESC = (1u << 4) | (uint32_t(DT) << 7) | (uint32_t(DT) << 10) | (1u << 16) |
                                    (uint32_t(BN >> 3) << 17) | (uint32_t(BM >> 4) << 24);
};

__device__ __forceinline__ void tile_coords(const Params& p, int t, int& b, int& mb, int& nb) {
  const int per_b = p.m_blocks * p.n_blocks;
  b = t / per_b;
  const int r = t - b * per_b;
  if (p.raster == 1) {
    const int group = p.group_m * p.m_blocks;
    const int g = r / group;
    const int first_n = g * p.group_m;
    const int gn = min(p.n_blocks - first_n, p.group_m);
    const int rg = r - g * group;
    nb = first_n + rg % gn;
    mb = rg / gn;
    if (p.serp && (g & 1)) mb = p.m_blocks - 1 - mb;
    return;
  }
  const int group = p.group_m * p.n_blocks;
  const int g = r / group;
  const int first_m = g * p.group_m;
  const int gm = min(p.m_blocks - first_m, p.group_m);
  const int rg = r - g * group;
  mb = first_m + rg % gm;
  nb = rg / gm;
  if (p.serp && (g & 1)) nb = p.n_blocks - 1 - nb;
}

// Tile t and the k-block range [kb0, kb1) of split `sidx` (0 when not split).
__device__ __forceinline__ void unit_coords(const Params& p, int t, int sidx, int& b, int& mb, int& nb, int& kb0,
                                            int& kb1) {
  tile_coords(p, t, b, mb, nb);
  kb0 = sidx * p.kb_split;
  kb1 = min(p.k_blocks, kb0 + p.kb_split);
}

// GLU activations in fp32 (reading R14): SiLU x / (1 + e^-x); GELU tanh form
// 0.5 x (1 + tanh(sqrt(2/pi) (x + 0.044715 x^3))).
__device__ __forceinline__ float act_f32(int act, float x) {
  if (act == 0) return x / (1.0f + __expf(-x));
  const float c = 0.7978845608028654f;
  return 0.5f * x * (1.0f + tanhf(c * fmaf(0.044715f * x, x * x, x)));
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
__device__ __forceinline__ float2 unpack2(uint32_t v) {
  if constexpr (DT == 0) {
    __half2 h = *reinterpret_cast<__half2*>(&v);
    return __half22float2(h);
  } else {
    __nv_bfloat162 h = *reinterpret_cast<__nv_bfloat162*>(&v);
    return __bfloat1622float2(h);
  }
}

template <class C>
__global__ void __launch_bounds__(C::THREADS, 1)
    cy_sm100_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB0,
                    const __grid_constant__ CUtensorMap tmB1, const __grid_constant__ CUtensorMap tmC0,
                    const __grid_constant__ CUtensorMap tmC1, const __grid_constant__ CUtensorMap tmD0,
                    const __grid_constant__ CUtensorMap tmD1, const Params p,
                    const __grid_constant__ DstMaps extra) {
  extern __shared__ uint8_t smem_raw[];
#ifdef CY_GEMM_TRACE
  if (threadIdx.x == 0) {
    CY_KT(0);
    unsigned long long gt;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
    if (blockIdx.x < 1024) g_gemm_gtime[blockIdx.x] = gt;
  }
#endif
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;  // SWIZZLE_128B atoms need 1024-B alignment
  const uint32_t sStage0 = base;
  const uint32_t sEpi = base + C::STAGES * C::STAGE_BYTES;
  const uint32_t sBar = sEpi + C::EPI_BYTES;
  const uint32_t bFull = sBar;                               // [STAGES]
  const uint32_t bEmpty = sBar + 8 * C::STAGES;              // [STAGES]
  const uint32_t bMDone = sBar + 16 * C::STAGES;             // [STAGES] (REDUCE only): MMAs read it
  const uint32_t bTFull = sBar + 24 * C::STAGES;             // [2]
  const uint32_t bTEmpty = bTFull + 16;                      // [2]
  const uint32_t bCBar = bTFull + 32;                        // [8]: per-epilogue-warp C-tile loads
  const uint32_t sTmemSlot = bTFull + 96;
  const uint32_t bSFull = bTFull + 104;                      // [SCHED_SLOTS] tile-ID ring: response landed
  const uint32_t bSEmpty = bSFull + 8 * C::SCHED_SLOTS;      // [SCHED_SLOTS] all warps of the cluster read it
  const uint32_t sResp = (bSEmpty + 8 * C::SCHED_SLOTS + 15u) & ~15u;  // [SCHED_SLOTS] x 16-B responses
  const uint32_t bRed = sResp + 16 * C::SCHED_SLOTS;         // [EPI_WARPS] split-K: partials of every split written
  volatile uint32_t* tmem_slot = reinterpret_cast<volatile uint32_t*>(smem_raw + (sTmemSlot - raw));

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  // split-K: the cluster is `splits` CTAs (pairs) stacked along K, all on the same output tile
  const int SPL = C::SPLITTABLE ? p.splits : 1;
  const int CLr = C::CL * SPL;                                  // cluster size (run time)
  const uint32_t crank = (CLr > 1) ? cluster_ctarank() : 0u;    // rank in the cluster
  const uint32_t rank = crank & (C::CG - 1);                    // rank in the CTA pair
  const uint32_t pp = (C::MC == 2) ? crank / C::CG : 0u;        // pair index in the cluster (MC == 2)
  const int sidx = (SPL > 1) ? int(crank / C::CG) : 0;          // split index (split-K)
  const uint32_t leader = crank & ~uint32_t(C::CG - 1);         // this pair's MMA leader
  // MX: position in the 2 x 2 cluster (rm along M, rn along N); offsets of this CTA's tile in the
  // cluster tile
  const int rm = C::MX ? int(crank & 1u) : 0, rn = C::MX ? int(crank >> 1) : 0;
  const int row_off = C::MX ? rm * C::BM : int(pp) * C::BM + int(rank) * C::BM_CTA;
  const int col_off = C::MX ? rn * C::TILE_N : 0;
  const int cid = blockIdx.x / CLr;
  const int ncl = gridDim.x / CLr;

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmA);
    prefetch_tmap(&tmB0);
    if (C::DUAL) prefetch_tmap(&tmB1);
    prefetch_tmap(&tmD0);
    if (C::VAR == V_DUAL_PAIR) prefetch_tmap(&tmD1);
  }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(bFull + 8 * s, 1);
      mbar_init(bEmpty + 8 * s, (C::MX ? 4 : C::MC) + C::RED_WARPS);  // MMA commit of every pair reading it
      if (C::REDUCE) mbar_init(bMDone + 8 * s, 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(bTFull + 8 * b, 1);
      mbar_init(bTEmpty + 8 * b, C::CG * C::EPI_WARPS);
    }
    for (int w = 0; w < C::EPI_WARPS; ++w) mbar_init(bCBar + 8 * w, 1);
    for (int j = 0; j < C::SCHED_SLOTS; ++j) {
      mbar_init(bSFull + 8 * j, 1);
      mbar_init(bSEmpty + 8 * j, CLr * C::NUM_WARPS);
    }
    if (SPL > 1)
      for (int w = 0; w < C::EPI_WARPS; ++w) mbar_init(bRed + 8 * w, SPL);
    fence_mbar_init();
  }
  if (warp == 1) {
    tmem_alloc<C::CG>(sTmemSlot, C::TMEM_COLS);
    tmem_relinquish<C::CG>();
  }
  tc_fence_before();
  if (CLr > 1) cluster_sync(); else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  if (threadIdx.x == 0) CY_KT(1);
  // Everything above (barrier init, TMEM allocation, descriptor prefetch) overlapped the tail of
  // the previous kernel on this stream; global memory is touched only after it has completed.
  pdl_wait();
  pdl_launch_dependents();  // (every thread: a lane-0 branch here would leave the warps' convergence
                            //  unprovable for ptxas, which then wraps each elected MMA / TMA in a loop)

  // ---------------------------------------------------------------- tile schedule
  // Tile i of this cluster: static -> cid + i*ncl; dynamic -> i == 0: own cluster's tile, i > 0:
  // the tile of the cluster that try_cancel stole for us (ring slot (i-1) % SCHED_SLOTS).
  // Every warp of both CTAs reads every slot and releases it on the leader's bSEmpty.
  auto sched_next = [&](int i, int& t, bool warp_wide) -> bool {
    if (!p.dyn) {
      t = cid + i * ncl;
      return t < p.tiles;
    }
    if (i == 0) {
      t = cid;
      return t < p.tiles;
    }
    if (p.dyn == 2) return false;  // one tile per launched cluster, no stealing
    const int j = (i - 1) % C::SCHED_SLOTS;
    const uint32_t ph = ((i - 1) / C::SCHED_SLOTS) & 1;
    uint32_t ok, cx;
    if (warp_wide) {  // converged warp: one elected lane releases the slot (no lane-0 branch)
      mbar_wait_w(bSFull + 8 * j, ph);
      clc_decode(sResp + 16 * j, ok, cx);
      __syncwarp();
      if (CLr > 1) mbar_arrive_cluster_e(mapa(bSEmpty + 8 * j, 0));
      else mbar_arrive_e(bSEmpty + 8 * j);
    } else {
      mbar_wait(bSFull + 8 * j, ph);
      clc_decode(sResp + 16 * j, ok, cx);
      if (CLr > 1) mbar_arrive_cluster(mapa(bSEmpty + 8 * j, 0));
      else mbar_arrive(bSEmpty + 8 * j);
    }
    t = static_cast<int>(cx) / CLr;
    return ok != 0;
  };
  // Producer warp, at the start of its tile i: arm this CTA's slot for tile i+1 and (leader)
  // ask the hardware for the next pending cluster.
  auto sched_request = [&](int i) {
    if (p.dyn != 1) return;
    const int j = i % C::SCHED_SLOTS;
    mbar_arrive_expect_tx_e(bSFull + 8 * j, 16);
    if (crank == 0) {
      mbar_wait_w(bSEmpty + 8 * j, ((i / C::SCHED_SLOTS) & 1) ^ 1);
      if (CLr > 1) clc_try_cancel_multicast_e(sResp + 16 * j, bSFull + 8 * j);
      else clc_try_cancel_e(sResp + 16 * j, bSFull + 8 * j);
    }
  };

  if (warp == 0) {
    // ------------------------------------------------------------------ producer (TMA)
    {  // all 32 lanes, converged; single-thread instructions are elect.sync-predicated (cy_ptx.cuh)
      uint64_t pol_a, pol_b;
      switch (p.l2_policy) {
        case 1: pol_a = pol_b = policy_evict_last(); break;
        case 2: pol_a = pol_b = policy_evict_first(); break;
        case 3: pol_a = policy_evict_first(); pol_b = policy_evict_last(); break;
        case 4: pol_a = policy_evict_last(); pol_b = policy_evict_first(); break;
        case 6: pol_a = policy_evict_normal(); pol_b = policy_evict_last(); break;
        case 7: pol_a = policy_evict_last(); pol_b = policy_evict_normal(); break;
        default: pol_a = pol_b = policy_evict_normal(); break;
      }
      // no cache hint at all on an operand: measured, hint-free requests for the same lines from
      // different SMs merge in L2
      const bool hint_a = p.l2_policy != 5 && p.l2_policy != 6;
      const bool hint_b = p.l2_policy != 5 && p.l2_policy != 7;
      uint32_t stage = 0, phase = 0;
      constexpr bool PAIR_TMA = (C::CG == 2);
      int t;
      for (int i = 0; sched_next(i, t, true); ++i) {
        CY_TR(i, 0);
        sched_request(i);
        int b, mb, nb, kb0, kb1;
        unit_coords(p, t, sidx, b, mb, nb, kb0, kb1);
        // (timing experiments only: measured slower at every distance)
        if (kTuning && p.pf_dist > 0 && crank == 0 && b + p.pf_dist < p.L) {
          // this tile's slice of problem b + pf_dist's operands (16-B granules)
          const int per_b = p.m_blocks * p.n_blocks;
          const int r = t - b * per_b;
          const int bb = b + p.pf_dist;
          auto pf = [&](const char* base, long long stride, long long bytes) {
            const long long gran = bytes >> 4;
            const long long g0 = gran * r / per_b, g1 = gran * (r + 1) / per_b;
            const char* a = base + bb * stride + (g0 << 4);
            for (long long g = g0; g < g1; g += (1ll << 20)) {  // <= 16 MB per op
              const long long n16 = min(g1 - g, 1ll << 20);
              bulk_prefetch_l2_e(a + ((g - g0) << 4), uint32_t(n16 << 4));
            }
          };
          pf(p.pf_a, p.pf_a_stride, p.pf_a_bytes);
          pf(p.pf_b, p.pf_b_stride, p.pf_b_bytes);
        }
        const int am = mb * C::CT_M + row_off;
        const int bn = nb * C::CT_N + col_off + rank * C::BN_CTA;
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait_w(bEmpty + 8 * stage, phase ^ 1);
          if (kb == kb0) CY_TR(i, 1);
          if (kb == kb1 - 1) CY_TR(i, 2);
          const uint32_t sA = sStage0 + stage * C::STAGE_BYTES;
          uint32_t fb = bFull + 8 * stage;
          if ((kDebug & 1) && (phase || i != 0)) {  // timing experiment: reuse stale stages
            if (PAIR_TMA ? rank == 0 : true) mbar_arrive_e(fb);  // (MC == 1 only)
            if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
            continue;
          }
          if constexpr (PAIR_TMA) {
            if (rank == 0) mbar_arrive_expect_tx_e(fb, C::STAGE_BYTES * 2);
            fb = mapa(fb, leader);  // both CTAs of the pair count bytes on the leader's barrier
          } else {
            mbar_arrive_expect_tx_e(fb, C::STAGE_BYTES);
          }
          const int k0 = kb * C::BK;
          if constexpr (C::MX) {
            // A: K-atom rn of the stage, to both CTAs on these rows; B: K rows [64 rm, 64 rm + 64) of
            // the stage, to both CTAs on these columns (every CTA's expect_tx above counts all
            // STAGE_BYTES landing in it)
            tma_load_3d_mc_e(sA + rn * C::A_ATOM, &tmA, fb, k0 + 64 * rn, am, b, uint16_t(0x5u << rm), pol_a, hint_a);
            tma_load_3d_mc_e(sA + C::A_BYTES + rm * (64 * 128), &tmB0, fb, bn, k0 + 64 * rm, b, uint16_t(0x3u << (2 * rn)),
                             pol_b, hint_b);
            if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
            continue;
          }
          auto load = [&](uint32_t dst, const CUtensorMap* tm, int c0, int c1, uint64_t pol, bool hint) {
            if constexpr (PAIR_TMA) {
              if (hint) tma_load_3d_pair_e(dst, tm, fb, c0, c1, b, pol);
              else tma_load_3d_pair_nohint_e(dst, tm, fb, c0, c1, b);
            } else {
              if (hint) tma_load_3d_e(dst, tm, fb, c0, c1, b, pol);
              else tma_load_3d_nohint_e(dst, tm, fb, c0, c1, b);
            }
          };
          if constexpr (C::KAT == 1) {
            load(sA, &tmA, k0, am, pol_a, hint_a);
          } else if (p.a4d) {  // both K-atoms of A in one 4-D box {64, 128 rows, KAT, 1}
            if constexpr (PAIR_TMA) tma_load_4d_pair_e(sA, &tmA, fb, 0, am, k0 / 64, b, pol_a, hint_a);
            else tma_load_4d_e(sA, &tmA, fb, 0, am, k0 / 64, b, pol_a, hint_a);
          } else {
#pragma unroll
            for (int a = 0; a < C::KAT; ++a) load(sA + a * C::A_ATOM, &tmA, k0 + 64 * a, am, pol_a, hint_a);
          }
#pragma unroll
          for (int sl = 0; sl < C::NUM_B; ++sl) {
            // slot sl: dual -> B0 / B1 at the same columns; GEMM -> N sub-tile sl of B
            const CUtensorMap* tmB = (C::DUAL && sl == 1) ? &tmB1 : &tmB0;
            const int cb = bn + (C::DUAL ? 0 : sl * C::BN);
            if (C::MC == 1 && p.b4d) {  // all of the slot's 64-column atoms in one 4-D box (one TMA op)
              const uint32_t dst = sA + C::A_BYTES + sl * C::B_BYTES;
              if constexpr (PAIR_TMA) tma_load_4d_pair_e(dst, tmB, fb, 0, k0, cb / 64, b, pol_b, hint_b);
              else tma_load_4d_e(dst, tmB, fb, 0, k0, cb / 64, b, pol_b, hint_b);
              continue;
            }
#pragma unroll
            for (int j = 0; j < C::BN_CTA / 64; ++j) {
              const uint32_t dst = sA + C::A_BYTES + sl * C::B_BYTES + j * C::B_ATOM_BYTES;
              if constexpr (C::MC == 2) {
                // every other atom: ours, multicast to us and our counterpart in the other pair
                if (((sl * (C::BN_CTA / 64) + j) & 1) == int(pp))
                  tma_load_3d_pair_mc_e(dst, tmB, fb, cb + 64 * j, k0, b, uint16_t((1u << crank) | (1u << (crank ^ 2u))),
                                        pol_b);
              } else {
                load(dst, tmB, cb + 64 * j, k0, pol_b, hint_b);
              }
            }
          }
          if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------------ MMA issuer
    if (rank == 0) {  // all 32 lanes, converged; the MMAs and commits are elect.sync-predicated
      uint32_t stage = 0, phase = 0;
      constexpr uint16_t kAllMask = uint16_t((1u << C::CL) - 1u);  // stage release: every CTA of the cluster
      const uint16_t pair_mask = uint16_t(0x3u << leader);          // this pair's two CTAs
      int kfirst = 0;  // first k-block of the current work unit (accumulate = 0 there)
      // all 4 k16 MMAs of one k-block for B slot `sl` of ring stage `st` into accumulator base `d`
      auto issue = [&](uint32_t d, int st, int sl, int kb) {
        const uint32_t sA = sStage0 + st * C::STAGE_BYTES;
        const uint32_t sB = sA + C::A_BYTES + sl * C::B_BYTES;
#pragma unroll
        for (int kk = 0; kk < C::BK / C::UMMA_K; ++kk) {
          // A: K-major SW128, 8-row groups 1024 B apart; K advances 32 B inside the atom, K-atoms
          // (BK = 128) A_ATOM apart.
          const uint64_t ad = sdesc_sw128(sA + (kk >> 2) * C::A_ATOM + (kk & 3) * 32, 16, 1024);
          // B: MN-major SW128, 64-column atoms B_ATOM_BYTES apart (LBO), 8-K-row groups 1024 B
          // apart (SBO); K advances 16 rows = 2048 B.
          const uint64_t bd = sdesc_sw128(sB + kk * 2048, C::B_ATOM_BYTES, 1024);
          const uint32_t acc = (kb != kfirst || kk != 0);
          if constexpr (C::VAR == V_DUAL_SUM) mma_f16_e<C::CG>(d, ad, bd, C::IDESC, sl ? 1u : acc);
          else mma_f16_e<C::CG>(d + sl * C::BN, ad, bd, C::IDESC, acc);
        }
      };
      // both B slots of one k-block, interleaved per k16 step so the second MMA reuses the A
      // operand the first one loaded (collector::a fill / lastuse) instead of re-reading smem
      auto issue_both = [&](uint32_t d, int st, int kb) {
        const uint32_t sA = sStage0 + st * C::STAGE_BYTES;
        const uint32_t sB = sA + C::A_BYTES;
#pragma unroll
        for (int kk = 0; kk < C::BK / C::UMMA_K; ++kk) {
          const uint64_t ad = sdesc_sw128(sA + (kk >> 2) * C::A_ATOM + (kk & 3) * 32, 16, 1024);
          const uint64_t bd0 = sdesc_sw128(sB + kk * 2048, C::B_ATOM_BYTES, 1024);
          const uint64_t bd1 = sdesc_sw128(sB + C::B_BYTES + kk * 2048, C::B_ATOM_BYTES, 1024);
          const uint32_t acc = (kb != kfirst || kk != 0);
          if constexpr (C::VAR == V_DUAL_SUM) {
            mma_f16_col_e<C::CG, 1>(d, ad, bd0, C::IDESC, acc);
            mma_f16_col_e<C::CG, 2>(d, ad, bd1, C::IDESC, 1u);
          } else {
            mma_f16_col_e<C::CG, 1>(d, ad, bd0, C::IDESC, acc);
            mma_f16_col_e<C::CG, 2>(d + C::BN, ad, bd1, C::IDESC, acc);
          }
        }
      };
      auto release = [&](int st) {
        // frees the stage: in both CTAs of the pair (B multicast, MC == 2: in both pairs)
        if constexpr (C::MX) mma_commit_mc_e(bEmpty + 8 * st, kAllMask);  // all four CTAs feed every stage
        else mma_commit_e<C::CG>(bEmpty + 8 * st, C::MC == 2 ? kAllMask : pair_mask);
        if constexpr (C::REDUCE) mma_commit_e<C::CG>(bMDone + 8 * st, pair_mask);  // reducers may read it
      };
      int t;
      for (int it = 0; sched_next(it, t, true); ++it) {
        const int buf = (C::NUM_ACC_BUF == 2) ? (it & 1) : 0;
        const uint32_t bph = (C::NUM_ACC_BUF == 2) ? ((it >> 1) & 1) : (it & 1);
        const uint32_t d = tmem_base + buf * C::ACC_COLS;
        int ub, umb, unb, kb0, kb1;
        unit_coords(p, t, sidx, ub, umb, unb, kb0, kb1);
        kfirst = kb0;
        CY_TR(it, 3);
#ifdef CY_GEMM_TRACE
        long long tr_mw = 0;  // full-barrier wait cycles of this tile (kept in a register: a global
                              // read-modify-write per k-block would slow the traced CTA itself)
        auto wait_full = [&](int kb) {
          const long long w0 = clock64();
          mbar_wait_w(bFull + 8 * stage, phase);
          tr_mw += clock64() - w0;
          if (kb == kb0) CY_TR(it, 5);
          if (it == 0 && kb == kb0) CY_KT(2);
        };
#else
        auto wait_full = [&](int) { mbar_wait_w(bFull + 8 * stage, phase); };
#endif
        if constexpr (!C::SPLIT) {
          mbar_wait_w(bTEmpty + 8 * buf, bph ^ 1);
          CY_TR(it, 4);
          tc_fence_after();
          for (int kb = kb0; kb < kb1; ++kb) {
            CY_MT(it, kb - kb0, 2);
            wait_full(kb);
            CY_MT(it, kb - kb0, 0);
            tc_fence_after();
            if constexpr (C::NUM_B == 2) {
              if (p.a_reuse) issue_both(d, stage, kb);
              else { issue(d, stage, 0, kb); issue(d, stage, 1, kb); }
            } else {
              issue(d, stage, 0, kb);
            }
            CY_MT(it, kb - kb0, 1);
            release(stage);
            CY_MT(it, kb - kb0, 3);
            if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
          }
        } else {
          // bTEmpty[a] = accumulator a drained by both CTAs' epilogues
          mbar_wait_w(bTEmpty, bph ^ 1);
          CY_TR(it, 4);
          tc_fence_after();
          bool acc1 = false;
          int held = 0, held0 = 0, held_kb0 = 0;
          auto flush = [&]() {  // accumulator-1 MMAs of the held stages, in k order, then release
            for (int h = 0; h < held; ++h) {
              const int st = (held0 + h) % C::STAGES;
              issue(d, st, 1, held_kb0 + h);
              release(st);
            }
            held = 0;
          };
          for (int kb = kb0; kb < kb1; ++kb) {
            wait_full(kb);
            tc_fence_after();
            if (acc1 && held == 0 && p.a_reuse) {  // steady state: both accumulators, A reused
              issue_both(d, stage, kb);
              release(stage);
              if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
              continue;
            }
            issue(d, stage, 0, kb);
            if (!acc1 && __any_sync(0xffffffffu, mbar_test_wait(bTEmpty + 8, bph ^ 1))) {
              acc1 = true;
              tc_fence_after();
            }
            if (held == 0) { held0 = stage; held_kb0 = kb; }
            ++held;
            if (acc1) {
              flush();
            } else if (held == C::STAGES) {  // every stage is held: wait for accumulator 1
#ifdef CY_GEMM_TRACE
              const long long w1 = clock64();
              mbar_wait_w(bTEmpty + 8, bph ^ 1);
              CY_TR_ADD(it, 14, clock64() - w1);
#else
              mbar_wait_w(bTEmpty + 8, bph ^ 1);
#endif
              acc1 = true;
              tc_fence_after();
              flush();
            }
            if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
          }
          if (held) {
            mbar_wait_w(bTEmpty + 8, bph ^ 1);
            tc_fence_after();
            flush();
          }
        }
        mma_commit_e<C::CG>(bTFull + 8 * buf, pair_mask);  // accumulator ready, both CTAs of the pair
        CY_TR(it, 6);
#ifdef CY_GEMM_TRACE
        CY_TR_ADD(it, 7, tr_mw);
#endif
        CY_KT(3);
      }
    } else if (lane == 0) {
      // peer CTA: the leader issues all MMAs; follow the tile schedule only
      int t;
      for (int it = 0; sched_next(it, t, false); ++it) {
      }
    }
  } else if (warp < 2 + C::EPI_WARPS) {
    // ------------------------------------------------------------------ epilogue
    // Per warp and tile, a fixed list of 32-row x 64-column chunks: q -> (accumulator a, chunk c).
    // The warp's chunks of one accumulator are loaded from TMEM in groups of G before the
    // accumulator is handed back (G = 2 when TMEM is single-buffered, so the MMA issuer waits only
    // for the loads, not for the conversions and stores); with two staging slots the C tile of the
    // next chunk is fetched while the current one is converted and stored.
    constexpr int NCH = C::BN / 64;                 // 64-column chunks per accumulator
    constexpr int CPW = NCH / C::EPI_SPLIT;         // chunks per warp per accumulator
    constexpr int G = (C::EPI_SPLIT == 2 && !C::GLU && !C::REDUCE && CPW == 2) ? 2 : 1;
    constexpr int NQ = C::NUM_OUT * CPW;            // chunks per warp per tile
    constexpr bool CPF = (C::EPI_BUFS == 2);        // C prefetch one chunk ahead
    const int ew = warp - 2;
    const int q4 = warp & 3;  // TMEM lane quarter this warp may access
    const int half = ew / 4;  // EPI_SPLIT == 2: this warp takes chunks c with c % 2 == half
    const uint32_t sE = sEpi + ew * C::EPI_BUFS * C::EPI_BUF_BYTES;
    const uint32_t cbar = bCBar + 8 * ew;
    const uint64_t pol = policy_evict_normal();
    const uint64_t dpol = p.d_policy == 1 ? policy_evict_first() : policy_evict_last();
    uint32_t slot = 0, cphase = 0;
    auto chunk_col = [&](int q) { return (C::EPI_SPLIT == 2 ? half : 0) + (q % CPW) * C::EPI_SPLIT; };
    // column of chunk q in the output; C/D maps of chunk q
    auto chunk_n0 = [&](int nb, int q) {
      if (CY_MUTANT == 5 && p.n_blocks > 1) nb = (nb + 1) % p.n_blocks;  // (mutant: D to the wrong columns)
      return nb * C::CT_N + col_off + (C::DUAL ? 0 : (q / CPW) * C::BN) + 64 * chunk_col(q);
    };
    auto chunk_c = [&](int q) { return (C::VAR == V_DUAL_PAIR && q / CPW == 1) ? &tmC1 : &tmC0; };
    auto chunk_d = [&](int q) { return (C::VAR == V_DUAL_PAIR && q / CPW == 1) ? &tmD1 : &tmD0; };
    // lane 0: wait until slot `s` may be overwritten (the store that last used it has read it) and
    // fetch chunk q's C tile into it
    auto fetch_c = [&](int nb, int row0, int b, int q, uint32_t s) {
      if (lane == 0) {
        bulk_wait_read<C::EPI_BUFS - 1>();
        mbar_arrive_expect_tx(cbar, C::EPI_BUF_BYTES);
        tma_load_3d(sE + s * C::EPI_BUF_BYTES, chunk_c(q), cbar, chunk_n0(nb, q), row0, b, pol);
      }
    };
    int t;
    // C prefetch: not with split-K (each split stores only some of its chunks)
    const bool cpf = CPF && p.has_c && SPL == 1;
    // single staging slot (EPI_BUFS == 1): only the tile's first C chunk is fetched ahead (during the
    // main loop); the others follow one at a time as the slot frees
    const bool cpf0 = !CPF && p.has_c && SPL == 1 && CY_C_FIRST;
    uint32_t red_phase = 0;  // split-K: parity of this warp's bRed barrier
    for (int it = 0; sched_next(it, t, true); ++it) {
      int b, mb, nb, kb0, kb1;
      unit_coords(p, t, sidx, b, mb, nb, kb0, kb1);
      const bool has_k = kb1 > kb0;
      const int buf = (C::NUM_ACC_BUF == 2) ? (it & 1) : 0;
      const uint32_t bph = (C::NUM_ACC_BUF == 2) ? ((it >> 1) & 1) : (it & 1);
      const int row0 = mb * C::CT_M + row_off + 32 * q4;
      if (kTuning && p.has_c && p.c_pf && lane == 0) {  // C of every chunk this warp will read, into L2 (neutral)
#pragma unroll 1
        for (int q = cpf ? 1 : 0; q < NQ; ++q) tma_prefetch_3d(chunk_c(q), chunk_n0(nb, q), row0, b);
      }
      if (cpf || cpf0) fetch_c(nb, row0, b, 0, slot);  // overlaps the tile's main loop
      if (ew == 0 && lane == 0) CY_TR(it, 8);
      if (p.sleep_ns) mbar_wait_sleep(bTFull + 8 * buf, bph, p.sleep_ns);
      else mbar_wait(bTFull + 8 * buf, bph);
      if (ew == 0 && lane == 0) CY_TR(it, 9);
      tc_fence_after();
      if constexpr ((kDebug & 2) != 0) {  // timing experiment: drop the epilogue
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          for (int a = 0; a < (C::SPLIT ? 2 : 1); ++a) {
            const uint32_t bar = bTEmpty + 8 * (C::SPLIT ? a : buf);
            if constexpr (C::CG == 2) mbar_arrive_cluster(mapa(bar, leader));
            else mbar_arrive(bar);
          }
        }
        continue;
      }
      // TMEM lane quarter q4, accumulator a, 64 columns of chunk q (two x32 loads)
      auto tmem_chunk = [&](int a, int q) {
        return tmem_base + (uint32_t(32 * q4) << 16) + buf * C::ACC_COLS + a * C::BN + 64 * chunk_col(q);
      };
      auto release = [&](int a) {  // accumulator a (buffer `buf`) is in registers: hand TMEM back
        if (C::SPLIT || a == C::NUM_OUT - 1) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            const uint32_t bar = bTEmpty + 8 * (C::SPLIT ? a : buf);
            if constexpr (C::CG == 2) mbar_arrive_cluster(mapa(bar, leader));
            else mbar_arrive(bar);
            if (ew == 0) CY_TR(it, a == 0 ? 10 : 11);
          }
        }
      };
      // wait until the current slot may be written (no C) / holds chunk q's C tile
      auto slot_ready = [&](int q) {
#ifdef CY_GEMM_TRACE
        const long long w0 = clock64();
        struct Add {
          long long w0; int it, ew, lane;
          __device__ ~Add() { if (ew == 0 && lane == 0) CY_TR_ADD(it, 13, clock64() - w0); }
        } add{w0, it, ew, lane};
#endif
        if (p.has_c) {
          if (!cpf && !(cpf0 && q == 0)) fetch_c(nb, row0, b, q, slot);
          mbar_wait(cbar, cphase);
          cphase ^= 1;
        } else {
          if (lane == 0) bulk_wait_read<C::EPI_BUFS - 1>();  // the store that last used this slot has read it
          __syncwarp();
        }
      };
      auto store_chunk = [&](int q) {  // staging slot -> D (and the replicas), next slot, next C
        CY_ET(it, ew, q, 3);
        fence_proxy_async_smem();
        __syncwarp();
        CY_ET(it, ew, q, 4);
        if (lane == 0 && !(kDebug & 4)) {  // (debug 4: timing experiment without the D stores)
          const int n0 = chunk_n0(nb, q);
          const uint32_t sb = sE + slot * C::EPI_BUF_BYTES;
          if (kTuning && p.d_policy) tma_store_3d_hint(chunk_d(q), sb, n0, row0, b, dpol);  // (neutral)
          else tma_store_3d(chunk_d(q), sb, n0, row0, b);
          for (int j = 0; j < p.n_extra; ++j) tma_store_3d(&extra.m[j], sb, n0, row0, b);  // replicas
          bulk_commit();
          if (ew == 0 && q == NQ - 1) CY_TR(it, 12);
          if (ew == 0 && q == NQ - 1) CY_KT(4);
        }
        if constexpr (C::EPI_BUFS == 2) slot ^= 1;
        if (cpf && q + 1 < NQ) fetch_c(nb, row0, b, q + 1, slot);  // next chunk's C
      };
      const bool unit_alpha = (p.alpha == 1.0f);
      // chunk q from fp32 registers (r: the accumulator, gt: GLU gate) -> alpha/act/beta*C in fp32
      // -> one RN cast -> swizzled staging -> TMA store
      auto emit = [&](int q, const uint32_t (&r)[64], const uint32_t (&gt)[C::GLU ? 64 : 1]) {
        slot_ready(q);
        CY_ET(it, ew, q, 2);
        const uint32_t row_addr = sE + slot * C::EPI_BUF_BYTES + lane * 128;
#pragma unroll
        for (int v = 0; v < 8; ++v) {
          const uint32_t addr = row_addr + ((v ^ (lane & 7)) << 4);  // SWIZZLE_128B chunk
          float f[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const int col = 8 * v + e;
            const float x = __uint_as_float(r[col]);
            f[e] = unit_alpha ? x : x * p.alpha;
            if constexpr (C::GLU) {
              const float gx = __uint_as_float(gt[col]);
              const float u = unit_alpha ? gx : gx * p.alpha;
              f[e] = act_f32(p.act, f[e]) * u;
            }
          }
          if (p.has_c) {
            uint32_t cv[4];
            ld_shared_v4(addr, cv[0], cv[1], cv[2], cv[3]);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float2 cf = unpack2<C::DT>(cv[e]);
              if (CY_MUTANT == 1 && q == NQ - 1) continue;
              f[2 * e] = fmaf(p.beta, cf.x, f[2 * e]);
              f[2 * e + 1] = fmaf(p.beta, cf.y, f[2 * e + 1]);
            }
          }
          st_shared_v4(addr, pack2<C::DT>(f[0], f[1]), pack2<C::DT>(f[2], f[3]), pack2<C::DT>(f[4], f[5]),
                       pack2<C::DT>(f[6], f[7]));
        }
        store_chunk(q);
        CY_ET(it, ew, q, 5);
      };
      auto load_chunk = [&](int q, uint32_t (&r)[64], uint32_t (&gt)[C::GLU ? 64 : 1]) {
        const int a = q / CPW;
        if (has_k) {
          const uint32_t ta = tmem_chunk(a, q);
          tmem_ld_32x32b_x32(ta, *reinterpret_cast<uint32_t(*)[32]>(&r[0]));
          tmem_ld_32x32b_x32(ta + 32, *reinterpret_cast<uint32_t(*)[32]>(&r[32]));
          if constexpr (C::GLU) {
            tmem_ld_32x32b_x32(ta + C::BN, *reinterpret_cast<uint32_t(*)[32]>(&gt[0]));
            tmem_ld_32x32b_x32(ta + C::BN + 32, *reinterpret_cast<uint32_t(*)[32]>(&gt[32]));
          }
          tmem_ld_wait();
        } else {
#pragma unroll
          for (int i = 0; i < 64; ++i) r[i] = 0u;
          if constexpr (C::GLU) {
#pragma unroll
            for (int i = 0; i < 64; ++i) gt[i] = 0u;
          }
        }
      };
      if constexpr (C::VAR == V_GEMM && C::MC == 1 && C::NSUB == 1) {  // (the host splits only these)
        if (SPL > 1) {
          // ---- split-K: the cluster's SPL CTAs (pairs) each hold the partial sum of
          // their k-range.  Every epilogue warp writes its slice (32 rows x NQ chunks, fp32) to the
          // workspace and arrives on the same warp's barrier in every split CTA of its pair half;
          // then warp `ew` of split s reduces the chunks q = s (mod SPL) over all splits, in split
          // order (deterministic), and stores them.  The splits share the reduction; the cluster
          // guarantees they are co-resident.  Slice layout: float4 j of lane l of chunk q at
          // ((q*16 + j)*32 + l) -- every warp-wide access is 512 contiguous bytes.
          const int wslot = (t * C::CG + int(rank)) * C::EPI_WARPS + ew;
          constexpr int SLICE4 = NQ * 16 * 32;  // float4 per slice
          float4* wsl = reinterpret_cast<float4*>(p.ws) + size_t(wslot) * SPL * SLICE4;
          uint32_t gt[C::GLU ? 64 : 1];
#pragma unroll 1
          for (int q = 0; q < NQ; ++q) {
            uint32_t r[64];
            load_chunk(q, r, gt);
            if ((q + 1) % CPW == 0) release(q / CPW);
            float4* dst = wsl + size_t(sidx) * SLICE4 + q * 16 * 32 + lane;
#pragma unroll
            for (int j = 0; j < 16; ++j)
              __stcg(dst + 32 * j, make_float4(__uint_as_float(r[4 * j]), __uint_as_float(r[4 * j + 1]),
                                               __uint_as_float(r[4 * j + 2]), __uint_as_float(r[4 * j + 3])));
          }
          __threadfence();
          __syncwarp();
          if (lane < SPL)  // lane s: our slice is written -> split s's barrier for this warp
            mbar_arrive_release_cluster(mapa(bRed + 8 * ew, uint32_t(lane * C::CG) + rank));
          mbar_wait_acquire_cluster(bRed + 8 * ew, red_phase);
          red_phase ^= 1;
#pragma unroll 1
          for (int q = sidx; q < NQ; q += SPL) {
            uint32_t r[64];
#pragma unroll 1
            for (int s2 = 0; s2 < SPL - (CY_MUTANT == 2 ? 1 : 0); ++s2) {
              const float4* src = wsl + size_t(s2) * SLICE4 + q * 16 * 32 + lane;
#pragma unroll
              for (int j = 0; j < 16; ++j) {
                const float4 v = __ldcg(src + 32 * j);
                if (s2 == 0) {
                  r[4 * j] = __float_as_uint(v.x), r[4 * j + 1] = __float_as_uint(v.y);
                  r[4 * j + 2] = __float_as_uint(v.z), r[4 * j + 3] = __float_as_uint(v.w);
                } else {
                  r[4 * j] = __float_as_uint(__uint_as_float(r[4 * j]) + v.x);
                  r[4 * j + 1] = __float_as_uint(__uint_as_float(r[4 * j + 1]) + v.y);
                  r[4 * j + 2] = __float_as_uint(__uint_as_float(r[4 * j + 2]) + v.z);
                  r[4 * j + 3] = __float_as_uint(__uint_as_float(r[4 * j + 3]) + v.w);
                }
              }
            }
            emit(q, r, gt);
          }
          continue;
        }
      }
      if (G == 2 && !p.has_c) {
        // beta == 0, single-buffered TMEM: both of this warp's chunks of an accumulator are loaded
        // and rounded (alpha*acc, one RN cast) into 16-bit pairs before the accumulator is handed
        // back, so the MMA issuer waits only for the TMEM loads.
        auto load_pack = [&](int a, int g, uint32_t (&pk)[32]) {
          uint32_t r[64];
          if (has_k) {
            const uint32_t ta = tmem_chunk(a, a * CPW + g);
            tmem_ld_32x32b_x32(ta, *reinterpret_cast<uint32_t(*)[32]>(&r[0]));
            tmem_ld_32x32b_x32(ta + 32, *reinterpret_cast<uint32_t(*)[32]>(&r[32]));
            tmem_ld_wait();
          } else {
#pragma unroll
            for (int i = 0; i < 64; ++i) r[i] = 0u;
          }
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            const float x0 = __uint_as_float(r[2 * i]), x1 = __uint_as_float(r[2 * i + 1]);
            pk[i] = unit_alpha ? pack2<C::DT>(x0, x1) : pack2<C::DT>(x0 * p.alpha, x1 * p.alpha);
          }
        };
        auto put = [&](int q, const uint32_t (&pk)[32]) {  // packed chunk -> staging -> TMA store
          slot_ready(q);
          const uint32_t row_addr = sE + slot * C::EPI_BUF_BYTES + lane * 128;
#pragma unroll
          for (int v = 0; v < 8; ++v)
            st_shared_v4(row_addr + ((v ^ (lane & 7)) << 4), pk[4 * v], pk[4 * v + 1], pk[4 * v + 2], pk[4 * v + 3]);
          store_chunk(q);
        };
        if constexpr (C::NUM_OUT == 2 && (kDebug & 8) == 0) {
          // Two accumulators (tile N = 512 or a dual pair): accumulator 1 is handed back after only
          // one store, not two -- chunk 0 of accumulator 0 goes out first, then accumulator 1 is
          // loaded while its other chunk waits in registers (3 chunks held, 96 registers).
          uint32_t pa[32], pb[32], pc[32];
          load_pack(0, 0, pa);
          load_pack(0, 1, pb);
          release(0);
          put(0, pa);
          load_pack(1, 0, pa);
          load_pack(1, 1, pc);
          release(1);
          put(1, pb);
          put(CPW, pa);
          put(CPW + 1, pc);
        } else {
#pragma unroll 1
          for (int a = 0; a < C::NUM_OUT; ++a) {
            uint32_t pk[2][32];
            load_pack(a, 0, pk[0]);
            load_pack(a, 1, pk[1]);
            release(a);
            if constexpr ((kDebug & 8) != 0) continue;  // timing experiment: TMEM loads only
            put(a * CPW, pk[0]);
            put(a * CPW + 1, pk[1]);
          }
        }
        continue;
      }
#pragma unroll 1
      for (int q = 0; q < NQ; ++q) {
        uint32_t r[64];
        uint32_t gt[C::GLU ? 64 : 1];  // GLU: the gate operand (accumulator 1)
        CY_ET(it, ew, q, 0);
        load_chunk(q, r, gt);
        CY_ET(it, ew, q, 1);
        // The accumulator's last chunk is in registers: hand its TMEM columns back to the MMA
        // issuer before converting and storing it.
        if ((q + 1) % CPW == 0) release(q / CPW);
        if constexpr ((kDebug & 8) != 0) continue;  // timing experiment: TMEM loads only
        emit(q, r, gt);
      }
    }
    if (lane == 0) bulk_wait_read<0>();  // shared staging must outlive the stores' reads
#ifdef CY_GEMM_TRACE
    if (ew == 0 && lane == 0) {
      bulk_wait<0>();
      CY_KT(5);
    }
#endif
  } else {
    // ------------------------------------------------------------------ row reduction (SIMT)
    const int q = warp & 3;
    const int r = 32 * q + lane;  // row of this CTA's 128-row A stage
    uint32_t stage = 0, phase = 0;
    int t;
    for (int it = 0; sched_next(it, t, true); ++it) {
      int b, mb, nb;
      tile_coords(p, t, b, mb, nb);
      const bool do_red = (nb == 0);  // one n-tile per row block reduces: no atomics, deterministic
      float acc = 0.f;
      for (int kb = 0; kb < p.k_blocks; ++kb) {
        mbar_wait(bMDone + 8 * stage, phase);  // the tensor core has read this stage; it is still resident
        if (do_red && !(CY_MUTANT == 3 && kb == p.k_blocks - 1)) {
#pragma unroll
          for (int a = 0; a < C::KAT; ++a) {  // K-atoms in k order
            const uint32_t row_addr = sStage0 + stage * C::STAGE_BYTES + a * C::A_ATOM + r * 128;
#pragma unroll
            for (int v = 0; v < 8; ++v) {  // logical 16-B chunk v = K elements 8v..8v+7, in k order
              uint32_t x[4];
              ld_shared_v4(row_addr + ((v ^ (r & 7)) << 4), x[0], x[1], x[2], x[3]);
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const float2 f = unpack2<C::DT>(x[e]);
                acc += f.x;
                acc += f.y;
              }
            }
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(bEmpty + 8 * stage);
        if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
      }
      if (do_red) {
        const int row = mb * C::BM + rank * C::BM_CTA + r;
        if (row < p.M) p.y[(size_t)b * p.M + row] = acc;
      }
    }
  }

  __syncwarp();
  if (threadIdx.x == 0) CY_KT(6);
  tc_fence_before();
  if (CLr > 1) cluster_sync(); else __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<C::CG>(tmem_base, C::TMEM_COLS);
    if (lane == 0) CY_KT(7);
  }
}

}  // namespace cy
