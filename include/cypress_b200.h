/*
 * cypress_b200.h -- C ABI of the B200-native (sm_100a) GEMM family that
 * Cypress (arXiv 2504.07004) compiles: D = alpha*A*B + beta*C with fp32
 * accumulation, batched, dual-GEMM and GEMM + row-reduction.
 *
 * Citations: P:n = PAPER.md line n (the paper's LaTeX source).
 *
 * General contract (all entry points):
 *  - extern "C", never throw, never allocate device memory, never
 *    synchronize.  Work is enqueued on `stream` (a cudaStream_t passed as
 *    void*; NULL = legacy default stream) of the CURRENT device, which must
 *    own every pointer.  Return is immediate; asynchronous faults surface on
 *    the stream like any CUDA kernel.
 *  - Storage is row-major; every leading dimension (ld*) and batch stride
 *    (stride*) is in ELEMENTS.  A is m x k, B is k x n, C and D are m x n.
 *    This matches the paper's logical shapes A[M,K], B[K,N], C[M,N]
 *    (Fig. 6a); the paper fixes no majorness (R5).
 *  - A, B, B0, B1, C, C0, C1 are read-only (the paper's read privileges,
 *    P:495).  If beta == 0, C is NOT read and may be NULL (BLAS rule, R4).
 *    C == D with ldc == ldd (exact alias) is allowed; any other overlap of
 *    an output with an input or with another output is CY_ERR_INVALID_VALUE.
 *  - dtype: A, B, C, D share one 16-bit type (cy_dtype_t); accumulation is
 *    fp32 in tensor memory; the epilogue computes alpha*acc + beta*C in fp32
 *    and rounds ONCE to the output type with IEEE round-to-nearest-even
 *    (R3, R7).  Boundary tiles are handled in-kernel (zero-filled loads,
 *    clipped stores, R8): no element outside [0,m) x [0,n) is written.
 *  - m == 0 or n == 0 (or batch == 0): CY_OK, nothing launched (except cy_gemm_rowreduce with
 *    n == 0, which still computes y).
 *    k == 0: D = beta*C (y = 0), computed by the same kernel.
 *  - Hardware rules (TMA): every base pointer 16-byte aligned; every ld and
 *    stride a multiple of 8 elements (16 bytes), else CY_ERR_MISALIGNED.
 *    There is no fallback path (no CPU, no library GEMM).
 *  - Requires compute capability 10.0 (B200, sm_100a); otherwise
 *    CY_ERR_UNSUPPORTED_DEVICE.
 *  - Thread safety: calls from several host threads on different streams
 *    are safe; the library keeps only lazily built, mutex-guarded caches
 *    (kernel attributes, SM count, driver entry point, TMA descriptors).
 */
#ifndef CYPRESS_B200_H_
#define CYPRESS_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  CY_OK = 0,
  CY_ERR_INVALID_VALUE = 1,      /* bad size, ld, NULL, overlap, mode/pointer mismatch */
  CY_ERR_MISALIGNED = 2,         /* pointer not 16-B aligned or ld/stride not a multiple of 8 */
  CY_ERR_UNSUPPORTED_DEVICE = 3, /* current device is not compute capability 10.0 */
  CY_ERR_LAUNCH = 4,             /* cudaGetLastError() after the launch, or descriptor encode failure */
  CY_ERR_INTERNAL = 5
} cy_status_t;

typedef enum { CY_F16 = 0, CY_BF16 = 1 } cy_dtype_t;

/* Dual-GEMM output mode (R1):
 *  CY_DUAL_PAIR: D0 = alpha*A*B0 + beta*C0 and D1 = alpha*A*B1 + beta*C1
 *                (BASELINE configs[3], the GLU core P:1532)
 *  CY_DUAL_SUM:  D0 = alpha*(A*B0 + A*B1) + beta*C0  ("A.B1 + A.B2");
 *                C1 and D1 must be NULL. */
typedef enum { CY_DUAL_PAIR = 0, CY_DUAL_SUM = 1 } cy_dual_mode_t;

/* GEMM, "C = A x B", tile program clear -> accumulate over
 * K tiles -> copy out (Fig. 6a), with BLAS alpha/beta (R4). */
cy_status_t cy_gemm(cy_dtype_t dt, int64_t m, int64_t n, int64_t k, float alpha,
                    const void* A, int64_t lda, const void* B, int64_t ldb, float beta,
                    const void* C, int64_t ldc, void* D, int64_t ldd, void* stream);

/* Strided batched GEMM: "L independent GEMMs in a single pass".
 * X_b = X + b*strideX (elements), b < batch; one launch covers all b.  With batch > 1 every
 * stride must be positive (no broadcast operands) and strideD >= m*ldd (outputs do not overlap). */
cy_status_t cy_gemm_batched(cy_dtype_t dt, int64_t m, int64_t n, int64_t k, int64_t batch,
                            float alpha, const void* A, int64_t lda, int64_t strideA,
                            const void* B, int64_t ldb, int64_t strideB, float beta,
                            const void* C, int64_t ldc, int64_t strideC, void* D, int64_t ldd,
                            int64_t strideD, void* stream);

/* Split-K GEMM: the strided-batched GEMM of cy_gemm_batched with the K dimension of
 * every output tile divided among `splits` CTAs (or CTA pairs) that form one thread-block cluster,
 * so that shapes with few output tiles and a long K (wave-quantised: the paper's small-size
 * overheads) occupy every SM.  Each split accumulates its k-range in TMEM and writes an
 * fp32 partial slice to `workspace`; after a cluster barrier every split reduces a share of the
 * tile's chunks over all splits, in split order (deterministic, independent of timing;
 * integer-valued inputs stay exact), and runs the usual epilogue on them (alpha, beta*C, one RN
 * cast).  splits = 0: the library's cost model picks the count (1 = no split, the cy_gemm_batched
 * kernel); splits = S >= 1: S, capped at 8 CTAs per cluster and reduced to the largest count that
 * leaves no split empty.  workspace: device memory of at least cy_gemm_splitk_workspace_size()
 * bytes for the same arguments, 16-byte aligned, any contents; it may be reused by later calls on
 * the same stream, with any shape, but not by concurrent calls.  It must not overlap A, B, C or D.
 * Errors as cy_gemm_batched, plus CY_ERR_INVALID_VALUE for splits outside 0..64 or a workspace
 * smaller than a requested split needs, CY_ERR_MISALIGNED for a misaligned workspace. */
cy_status_t cy_gemm_splitk(cy_dtype_t dt, int64_t m, int64_t n, int64_t k, int64_t batch, float alpha,
                           const void* A, int64_t lda, int64_t strideA, const void* B, int64_t ldb,
                           int64_t strideB, float beta, const void* C, int64_t ldc, int64_t strideC, void* D,
                           int64_t ldd, int64_t strideD, int splits, void* workspace, size_t workspace_bytes,
                           void* stream);
/* Workspace bytes cy_gemm_splitk needs for these arguments on the current device (0 when the
 * choice is not to split, or the arguments are invalid). */
size_t cy_gemm_splitk_workspace_size(cy_dtype_t dt, int64_t m, int64_t n, int64_t k, int64_t batch, int splits);

/* Dual GEMM: A*B0 and A*B1 in one kernel sharing the A tiles, B0/B1 copies
 * overlapped in the main loop.  See cy_dual_mode_t. */
cy_status_t cy_dual_gemm(cy_dtype_t dt, cy_dual_mode_t mode, int64_t m, int64_t n, int64_t k,
                         float alpha, const void* A, int64_t lda, const void* B0, int64_t ldb0,
                         const void* B1, int64_t ldb1, float beta, const void* C0, int64_t ldc0,
                         const void* C1, int64_t ldc1, void* D0, int64_t ldd0, void* D1,
                         int64_t ldd1, void* stream);

/* Replicated GEMM -- the compute step fused with its collective (BASELINE
 * configs[4] "M-sharded ... + all-gather"): computes this rank's M-row shard
 * D_shard = alpha*A*B + beta*C (A: m x k, C: m x n) and the epilogue stores every output tile
 * directly into each of the `ndst` (1..8) destination matrices at rows [row_offset, row_offset + m).
 * D_dst[j] is the base of a rows_total x n row-major matrix with leading dimension ldd, in device
 * memory addressable by the current device -- typically the replicated D of every GPU of the job
 * mapped into this process (CUDA IPC / symmetric memory over NVLink), so no separate all-gather
 * runs.  Stores never leave the shard's row block of a destination.  Completion follows stream
 * order on this device; the caller synchronizes with the peers before they read (e.g. a device
 * barrier after the kernel).  Destinations must not overlap each other, A, B or C. */
cy_status_t cy_gemm_replicated(cy_dtype_t dt, int64_t m, int64_t n, int64_t k, float alpha,
                               const void* A, int64_t lda, const void* B, int64_t ldb, float beta,
                               const void* C, int64_t ldc, void* const* D_dst, int ndst, int64_t ldd,
                               int64_t row_offset, int64_t rows_total, void* stream);

/* Device-side barrier between the ranks of a job that share memory through peer mappings (CUDA IPC
 * over NVLink / NVSwitch): the synchronisation step of the fused replicated GEMM (SURVEY NEXT-2 and
 * 8(e); BASELINE configs[4] "+ all-gather").  dist.py runs, on every rank's stream,
 *   cy_peer_barrier -> cy_gemm_replicated -> cy_peer_barrier
 * (peers are done reading the previous result; then every peer's tile stores have landed).
 * flags[j] (j < world): rank j's array of at least `world` uint32 flags, zero before first use,
 * 4-byte aligned, mapped into this process (flags[rank] is this rank's own).  `epoch` is 1 on the
 * first call and grows by one per call, identically on every rank.  One 32-thread kernel on
 * `stream`: thread j fences system-wide, stores epoch into flags[j][rank] (release, system scope)
 * and waits until flags[rank][j] >= epoch (acquire).  Launched without programmatic serialisation,
 * so it starts only after the preceding work on `stream` has completed.  A peer that never
 * arrives makes the kernel trap after ~60 s (the fault surfaces on the stream) instead of hanging.
 * world in 1..8, 0 <= rank < world, epoch != 0, no NULL flag pointer, else CY_ERR_INVALID_VALUE;
 * a flag pointer that is not 4-byte aligned: CY_ERR_MISALIGNED. */
cy_status_t cy_peer_barrier(uint32_t* const* flags, int world, int rank, uint32_t epoch, void* stream);

/* GLU activation for cy_dual_gemm_glu. */
typedef enum { CY_ACT_SILU = 0, CY_ACT_GELU_TANH = 1 } cy_act_t;

/* Dual GEMM with a gated-linear-unit epilogue (the use the paper gives for dual-GEMM,
 * P:1532-1533):  D = act(alpha*A*B0) (elementwise *) (alpha*A*B1),
 * act = SiLU (x / (1 + e^-x)) or GELU in its tanh form; both products accumulate in fp32 TMEM and
 * the activation and product are applied in fp32 before one RN cast (R14).  The two
 * products are never written to memory.  D is m x n; D must not overlap A, B0 or B1. */
cy_status_t cy_dual_gemm_glu(cy_dtype_t dt, cy_act_t act, int64_t m, int64_t n, int64_t k, float alpha,
                             const void* A, int64_t lda, const void* B0, int64_t ldb0, const void* B1,
                             int64_t ldb1, void* D, int64_t ldd, void* stream);

/* GEMM + row reduction: "C = A.B and y(i) = sum_k A(i,k)" in a single kernel,
 * the reduction done on SIMT warps from the shared-memory A tiles while the
 * tensor core computes A.B.  y: m floats (fp32, device),
 * unscaled and independent of B/alpha/beta/C (R2); must not overlap D.
 * y(i) is summed in fp32 in k order.  n == 0 (no D): y alone is computed by a row-sum kernel with
 * the same order (B, C, D are not touched and may be NULL); k == 0: y = 0. */
cy_status_t cy_gemm_rowreduce(cy_dtype_t dt, int64_t m, int64_t n, int64_t k, float alpha,
                              const void* A, int64_t lda, const void* B, int64_t ldb, float beta,
                              const void* C, int64_t ldc, void* D, int64_t ldd, float* y,
                              void* stream);

/* Forward attention (the Flash Attention 2/3 forward of the paper's Sec. 5.3,
 * P:1594-1664, FP16/BF16, HeadDim 128 -- P:1636):
 *   O = softmax(scale * Q K^T) V  per (batch, head), rows masked to key <= query when causal
 *   (top-left aligned);  lse[b*heads+h][i] = log sum_j exp(scale * q_i.k_j)  (natural log, fp32).
 * Layout: Q [batch, heads, seq_q, 128], K and V [batch, heads, seq_k, 128], O like Q, all
 * contiguous (row stride 128 elements).  Scores and O accumulate in fp32 (TMEM); the softmax runs
 * in fp32 in the exp2 domain; P is rounded to the input type for the P.V product (as FA2/FA3 do).
 * lse may be NULL.  head_dim must be 128; batch*heads < 2^31 (above 65535 with ceil(seq_q / 256)
 * <= 65535).  O must not overlap Q, K, V. */
cy_status_t cy_attention_fwd(cy_dtype_t dt, int64_t batch, int64_t heads, int64_t seq_q, int64_t seq_k,
                             int64_t head_dim, float scale, int causal, const void* Q, const void* K,
                             const void* V, void* O, float* lse, void* stream);

/* Human-readable status. */
const char* cy_status_string(cy_status_t s);

/* ---- tuning / introspection (tests, bench) ---------------------------- */

/* Number of compiled kernel configurations (tile shape x CTA-pairing x stages). */
int cy_num_configs(void);
/* Describe config `id`: writes cta_group (1|2), tile_m (rows per cluster tile: 128 x cta_group x
 * CTA pairs sharing B; the last config is two pairs with B multicast, tile_m = 512), tile_n,
 * stages. Returns CY_OK or CY_ERR_INVALID_VALUE. */
cy_status_t cy_config_info(int id, int* cta_group, int* tile_m, int* tile_n, int* stages);
/* Force config `id` for subsequent GEMM / batched / rowreduce calls of this process
 * (-1 restores the shape heuristic).  Used by config-invariance tests. */
cy_status_t cy_force_config(int id);
/* Config id chosen by the most recent successful launch in this process (-1 if none). */
int cy_last_config(void);
/* Exact kernel of the most recent successful launch: variant (0 GEMM/batched, 1 dual pair, 2 dual
 * sum, 3 row-reduce, 4 dual GLU), cta_group, tile_m, tile_n, stages, threads per CTA, dynamic smem
 * bytes, dtype.  Any pointer may be NULL.  CY_ERR_INVALID_VALUE if nothing was launched yet. */
cy_status_t cy_last_kernel_info(int* variant, int* cta_group, int* tile_m, int* tile_n, int* stages,
                                int* threads, int* smem_bytes, int* dtype);
/* Split count of the most recent successful GEMM-family launch (1 = not split). */
int cy_last_splits(void);
/* Number of kernel launches this library issued in this process (monotone counter). */
int64_t cy_launch_count(void);

#ifdef __cplusplus
}
#endif

#endif /* CYPRESS_B200_H_ */
