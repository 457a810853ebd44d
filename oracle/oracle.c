/*
 * oracle/oracle.c -- plain, slow, obviously-correct fp64 CPU oracle for the
 * Cypress GEMM family (arXiv 2504.07004).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py (cpu_baseline / --impl reference legs) may load this library.
 * The product path (paper_2504_07004_b200/, include/) never links, imports or
 * executes anything under oracle/, and this file shares no code, header,
 * table or constant generator with the CUDA path.
 *
 * Citations: P:n = /root/reference/PAPER.md line n.
 *
 * What it computes (each a plain definition, written out; no blocking, no
 * fusion, no reordering beyond the stated loop order):
 *   GEMM            D = alpha * A.B + beta * C      "C = A x B" P:125 (Sec. 2),
 *                                                   P:1513 (Sec. 5.2); tile
 *                                                   program P:520-525 (Fig. 6a);
 *                                                   alpha/beta: DESIGN.md R4
 *   Batched GEMM    L independent GEMMs             P:1520-1521 (Sec. 5.2)
 *   Dual GEMM SUM   D = alpha*(A.B0 + A.B1)+beta*C  P:1529 (Sec. 5.2)
 *   Dual GEMM PAIR  D0 = alpha*A.B0+beta*C0,
 *                   D1 = alpha*A.B1+beta*C1         BASELINE.json configs[3]; GLU use P:1532
 *   Row reduction   y(i) = sum_k A(i,k)              P:1579 (Sec. 5.2)
 *
 * Precision: all arithmetic in IEEE fp64.  fp16 x fp16 (and bf16 x bf16)
 * products are exact in fp64 (11+11 <= 53 significand bits); the only fp64
 * error is summation, <= K * 2^-53 * sum|a||b|.  For integer-valued inputs
 * with |partial sums| < 2^53 the result is exact.
 *
 * Storage: every matrix is row-major with a leading dimension in elements;
 * inputs are raw 16-bit patterns (fp16 = IEEE binary16, bf16 = top half of
 * binary32).  Outputs are unrounded fp64 (D_ref); the separate encoder
 * cyo_encode() rounds fp64 to the 16-bit format with IEEE round-to-nearest-
 * even (overflow -> +-inf, NaN -> quiet NaN) -- DESIGN.md reading R7.
 *
 * Loop order: i (rows, OpenMP-parallel) -> k -> j with an fp64 row
 * accumulator; this is the textbook triple loop with the j loop innermost so
 * rows of B stream.  beta == 0 means C is not read (BLAS rule, R4).
 */
#define _DEFAULT_SOURCE
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define CYO_F16 0
#define CYO_BF16 1

/* ---- 16-bit codecs ------------------------------------------------------ */

/* IEEE binary16: 1 sign, 5 exponent (bias 15), 10 fraction bits. */
double cyo_half_to_double(uint16_t h) {
  int sign = (h >> 15) & 1;
  int e = (h >> 10) & 0x1f;
  int f = h & 0x3ff;
  double v;
  if (e == 0) {
    v = ldexp((double)f, -24); /* subnormal: f * 2^-24 */
  } else if (e == 31) {
    v = f ? NAN : INFINITY;
  } else {
    v = ldexp((double)(1024 + f), e - 25); /* (1 + f/1024) * 2^(e-15) */
  }
  return sign ? -v : v;
}

/* bfloat16: 1 sign, 8 exponent (bias 127), 7 fraction bits. */
double cyo_bf16_to_double(uint16_t h) {
  int sign = (h >> 15) & 1;
  int e = (h >> 7) & 0xff;
  int f = h & 0x7f;
  double v;
  if (e == 0) {
    v = ldexp((double)f, -133); /* subnormal: f * 2^-133 */
  } else if (e == 255) {
    v = f ? NAN : INFINITY;
  } else {
    v = ldexp((double)(128 + f), e - 134); /* (1 + f/128) * 2^(e-127) */
  }
  return sign ? -v : v;
}

/*
 * Round x to a binary format with `mbits` fraction bits, exponent bias
 * `bias`, max biased exponent `emax_b` (all-ones = inf/NaN) using IEEE
 * round-to-nearest, ties-to-even.  rint() runs in the default FE_TONEAREST
 * mode, which is ties-to-even; every operand passed to it is an exact
 * scaling of x, so there is exactly one rounding.
 */
static uint16_t round_to_bits(double x, int mbits, int ebits, int bias) {
  const int emax_b = (1 << ebits) - 1;
  uint16_t sign = signbit(x) ? (uint16_t)(1u << (mbits + ebits)) : 0;
  if (isnan(x)) return (uint16_t)(sign | (emax_b << mbits) | (1u << (mbits - 1)));
  double ax = fabs(x);
  if (isinf(ax)) return (uint16_t)(sign | (emax_b << mbits));
  const int emin = 1 - bias; /* exponent of the smallest normal */
  if (ax < ldexp(1.0, emin)) {
    /* subnormal range: quantum 2^(emin - mbits) */
    double q = rint(ldexp(ax, mbits - emin)); /* in [0, 2^mbits] */
    /* q == 2^mbits encodes the smallest normal, which the bit layout gives */
    return (uint16_t)(sign | (uint16_t)q);
  }
  int e2;
  double fr = frexp(ax, &e2); /* ax = fr * 2^e2, fr in [0.5, 1) */
  int E = e2 - 1;             /* ax = (2 fr) * 2^E, 2fr in [1, 2) */
  double q = rint(ldexp(2.0 * fr - 1.0, mbits)); /* fraction, in [0, 2^mbits] */
  if (q == ldexp(1.0, mbits)) { q = 0; E += 1; }
  int eb = E + bias;
  if (eb >= emax_b) return (uint16_t)(sign | (emax_b << mbits)); /* overflow */
  return (uint16_t)(sign | (uint16_t)(eb << mbits) | (uint16_t)q);
}

uint16_t cyo_double_to_half_rn(double x) { return round_to_bits(x, 10, 5, 15); }
uint16_t cyo_double_to_bf16_rn(double x) { return round_to_bits(x, 7, 8, 127); }

static double decode1(int dt, uint16_t h) {
  return dt == CYO_BF16 ? cyo_bf16_to_double(h) : cyo_half_to_double(h);
}

void cyo_decode(int dt, const uint16_t* in, double* out, int64_t n) {
  for (int64_t i = 0; i < n; ++i) out[i] = decode1(dt, in[i]);
}

void cyo_encode(int dt, const double* in, uint16_t* out, int64_t n) {
  for (int64_t i = 0; i < n; ++i)
    out[i] = dt == CYO_BF16 ? cyo_double_to_bf16_rn(in[i]) : cyo_double_to_half_rn(in[i]);
}

/* ---- GEMM -------------------------------------------------------------- */

/*
 * D_ref[r][j] = alpha * sum_{k<K} A[i][k] * B[k][j] + (beta != 0 ? beta*C[i][j] : 0)
 * for i = rows[r] (or i = r when rows == NULL, nrows = m), 0 <= j < n.
 * Dref is nrows x n with leading dimension lddref (doubles).
 * Returns 0, or -1 on invalid arguments / allocation failure.
 */
int cyo_gemm(int dt, int64_t m, int64_t n, int64_t k, double alpha,
             const uint16_t* A, int64_t lda, const uint16_t* B, int64_t ldb,
             double beta, const uint16_t* C, int64_t ldc,
             double* Dref, int64_t lddref, const int64_t* rows, int64_t nrows) {
  if (m < 0 || n < 0 || k < 0 || nrows < 0) return -1;
  if (!rows) nrows = m;
  if (nrows == 0 || n == 0) return 0;
  /* decode B once: K x N doubles (row-major, ld = n) */
  double* Bd = (double*)malloc(sizeof(double) * (size_t)(k > 0 ? k : 1) * (size_t)n);
  if (!Bd) return -1;
  for (int64_t kk = 0; kk < k; ++kk)
    for (int64_t j = 0; j < n; ++j) Bd[kk * n + j] = decode1(dt, B[kk * ldb + j]);
  int err = 0;
#pragma omp parallel
  {
    double* acc = (double*)malloc(sizeof(double) * (size_t)n);
    if (!acc) {
#pragma omp atomic write
      err = 1;
    }
#pragma omp for schedule(dynamic, 1)
    for (int64_t r = 0; r < nrows; ++r) {
      if (!acc) continue;
      int64_t i = rows ? rows[r] : r;
      for (int64_t j = 0; j < n; ++j) acc[j] = 0.0;
      for (int64_t kk = 0; kk < k; ++kk) {
        double a = decode1(dt, A[i * lda + kk]);
        const double* brow = Bd + kk * n;
        for (int64_t j = 0; j < n; ++j) acc[j] += a * brow[j];
      }
      double* drow = Dref + r * lddref;
      for (int64_t j = 0; j < n; ++j) {
        double d = alpha * acc[j];
        if (beta != 0.0) d += beta * decode1(dt, C[i * ldc + j]);
        drow[j] = d;
      }
    }
    free(acc);
  }
  free(Bd);
  return err ? -1 : 0;
}

/*
 * Batched: for b < batch, X_b = X + b * strideX (elements); D_ref_b at
 * Dref + b * strideDref.  Each batch is an independent cyo_gemm
 * ("L independent GEMMs").
 */
int cyo_gemm_batched(int dt, int64_t m, int64_t n, int64_t k, int64_t batch, double alpha,
                     const uint16_t* A, int64_t lda, int64_t strideA,
                     const uint16_t* B, int64_t ldb, int64_t strideB, double beta,
                     const uint16_t* C, int64_t ldc, int64_t strideC,
                     double* Dref, int64_t lddref, int64_t strideDref) {
  if (batch < 0) return -1;
  for (int64_t b = 0; b < batch; ++b) {
    int rc = cyo_gemm(dt, m, n, k, alpha, A + b * strideA, lda, B + b * strideB, ldb, beta,
                      beta != 0.0 ? C + b * strideC : NULL, ldc, Dref + b * strideDref, lddref,
                      NULL, m);
    if (rc) return rc;
  }
  return 0;
}

/*
 * Dual GEMM.
 *   mode 0 (PAIR): D0 = alpha*A.B0 + beta*C0 ; D1 = alpha*A.B1 + beta*C1
 *   mode 1 (SUM):  D0 = alpha*(A.B0 + A.B1) + beta*C0   ("A.B1 + A.B2")
 * The SUM definition accumulates both products into one fp64 row accumulator
 * in k order (A.B0 terms then A.B1 terms per k).
 */
int cyo_dual_gemm(int dt, int mode, int64_t m, int64_t n, int64_t k, double alpha,
                  const uint16_t* A, int64_t lda, const uint16_t* B0, int64_t ldb0,
                  const uint16_t* B1, int64_t ldb1, double beta,
                  const uint16_t* C0, int64_t ldc0, const uint16_t* C1, int64_t ldc1,
                  double* D0ref, int64_t ldd0ref, double* D1ref, int64_t ldd1ref,
                  const int64_t* rows, int64_t nrows) {
  if (mode == 0) {
    int rc = cyo_gemm(dt, m, n, k, alpha, A, lda, B0, ldb0, beta, C0, ldc0, D0ref, ldd0ref, rows, nrows);
    if (rc) return rc;
    return cyo_gemm(dt, m, n, k, alpha, A, lda, B1, ldb1, beta, C1, ldc1, D1ref, ldd1ref, rows, nrows);
  }
  if (mode != 1) return -1;
  if (m < 0 || n < 0 || k < 0 || nrows < 0) return -1;
  if (!rows) nrows = m;
  if (nrows == 0 || n == 0) return 0;
  double* B0d = (double*)malloc(sizeof(double) * (size_t)(k > 0 ? k : 1) * (size_t)n);
  double* B1d = (double*)malloc(sizeof(double) * (size_t)(k > 0 ? k : 1) * (size_t)n);
  if (!B0d || !B1d) { free(B0d); free(B1d); return -1; }
  for (int64_t kk = 0; kk < k; ++kk)
    for (int64_t j = 0; j < n; ++j) {
      B0d[kk * n + j] = decode1(dt, B0[kk * ldb0 + j]);
      B1d[kk * n + j] = decode1(dt, B1[kk * ldb1 + j]);
    }
  int err = 0;
#pragma omp parallel
  {
    double* acc = (double*)malloc(sizeof(double) * (size_t)n);
    if (!acc) {
#pragma omp atomic write
      err = 1;
    }
#pragma omp for schedule(dynamic, 1)
    for (int64_t r = 0; r < nrows; ++r) {
      if (!acc) continue;
      int64_t i = rows ? rows[r] : r;
      for (int64_t j = 0; j < n; ++j) acc[j] = 0.0;
      for (int64_t kk = 0; kk < k; ++kk) {
        double a = decode1(dt, A[i * lda + kk]);
        for (int64_t j = 0; j < n; ++j) acc[j] += a * B0d[kk * n + j] + a * B1d[kk * n + j];
      }
      double* drow = D0ref + r * ldd0ref;
      for (int64_t j = 0; j < n; ++j) {
        double d = alpha * acc[j];
        if (beta != 0.0) d += beta * decode1(dt, C0[i * ldc0 + j]);
        drow[j] = d;
      }
    }
    free(acc);
  }
  free(B0d);
  free(B1d);
  return err ? -1 : 0;
}

/*
 * GLU dual GEMM (R14; "Dual-GEMM is a core computation in Gated Linear Units",
 * P:1532-1533):  D = act(alpha * A.B0) (elementwise *) (alpha * A.B1)
 *   act 0 = SiLU:      x / (1 + exp(-x))
 *   act 1 = GELU-tanh: 0.5 x (1 + tanh(sqrt(2/pi) (x + 0.044715 x^3)))
 * Both products are the plain fp64 triple loop of cyo_gemm; the activation and the product are
 * applied to the fp64 results.
 */
static double act_eval(int act, double x) {
  if (act == 0) return x / (1.0 + exp(-x));
  const double c = sqrt(2.0 / M_PI);
  return 0.5 * x * (1.0 + tanh(c * (x + 0.044715 * x * x * x)));
}

double cyo_act(int act, double x) { return act_eval(act, x); }

int cyo_dual_glu(int dt, int act, int64_t m, int64_t n, int64_t k, double alpha,
                 const uint16_t* A, int64_t lda, const uint16_t* B0, int64_t ldb0,
                 const uint16_t* B1, int64_t ldb1, double* Dref, int64_t lddref,
                 const int64_t* rows, int64_t nrows) {
  if (act != 0 && act != 1) return -1;
  if (!rows) nrows = m;
  if (nrows == 0 || n == 0) return 0;
  double* X0 = (double*)malloc(sizeof(double) * (size_t)nrows * (size_t)n);
  double* X1 = (double*)malloc(sizeof(double) * (size_t)nrows * (size_t)n);
  if (!X0 || !X1) { free(X0); free(X1); return -1; }
  int rc = cyo_gemm(dt, m, n, k, alpha, A, lda, B0, ldb0, 0.0, NULL, n, X0, n, rows, nrows);
  if (!rc) rc = cyo_gemm(dt, m, n, k, alpha, A, lda, B1, ldb1, 0.0, NULL, n, X1, n, rows, nrows);
  if (!rc)
    for (int64_t r = 0; r < nrows; ++r)
      for (int64_t j = 0; j < n; ++j) Dref[r * lddref + j] = act_eval(act, X0[r * n + j]) * X1[r * n + j];
  free(X0);
  free(X1);
  return rc;
}

/*
 * Row reduction over the INPUT A ("y(i) = sum_k A(i,k)"), fp64,
 * unscaled and independent of B, alpha, beta, C.  y has nrows entries.
 */
int cyo_rowsum(int dt, int64_t m, int64_t k, const uint16_t* A, int64_t lda, double* y,
               const int64_t* rows, int64_t nrows) {
  if (m < 0 || k < 0 || nrows < 0) return -1;
  if (!rows) nrows = m;
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < nrows; ++r) {
    int64_t i = rows ? rows[r] : r;
    double s = 0.0;
    for (int64_t kk = 0; kk < k; ++kk) s += decode1(dt, A[i * lda + kk]);
    y[r] = s;
  }
  return 0;
}

/*
 * Forward attention (paper Sec. 5.3, P:1594-1611 -- Flash Attention 2/3 compute
 * exactly this; HeadDim 128, FP16):
 *   S = scale * Q.K^T,  P = softmax_rows(S) (keys j > i masked when causal),  O = P.V,
 *   lse_i = log(sum_j exp(S_ij)).
 * Layout: Q [BH, sq, d], K and V [BH, sk, d], O [BH, sq, d] contiguous (BH = batch * heads).
 * Plain definition in fp64: per row, the max-shifted exponentials, their sum, the weighted sum of
 * V rows.  Causal masking keeps key j <= query i (top-left aligned).
 */
int cyo_attention(int dt, int64_t bh, int64_t sq, int64_t sk, int64_t d, double scale, int causal,
                  const uint16_t* Q, const uint16_t* K, const uint16_t* V, double* O, double* lse) {
  if (bh < 0 || sq < 0 || sk < 0 || d <= 0) return -1;
  int err = 0;
#pragma omp parallel for schedule(dynamic, 1) collapse(2)
  for (int64_t h = 0; h < bh; ++h)
    for (int64_t i = 0; i < sq; ++i) {
      double* s = (double*)malloc(sizeof(double) * (size_t)(sk > 0 ? sk : 1));
      if (!s) {
#pragma omp atomic write
        err = 1;
        continue;
      }
      const uint16_t* q = Q + (h * sq + i) * d;
      const int64_t nk = causal ? (i + 1 < sk ? i + 1 : sk) : sk;
      double mx = -INFINITY;
      for (int64_t j = 0; j < nk; ++j) {
        const uint16_t* kr = K + (h * sk + j) * d;
        double acc = 0.0;
        for (int64_t t = 0; t < d; ++t) acc += decode1(dt, q[t]) * decode1(dt, kr[t]);
        s[j] = scale * acc;
        if (s[j] > mx) mx = s[j];
      }
      double l = 0.0;
      for (int64_t j = 0; j < nk; ++j) {
        s[j] = exp(s[j] - mx);
        l += s[j];
      }
      double* o = O + (h * sq + i) * d;
      for (int64_t t = 0; t < d; ++t) o[t] = 0.0;
      for (int64_t j = 0; j < nk; ++j) {
        const uint16_t* vr = V + (h * sk + j) * d;
        for (int64_t t = 0; t < d; ++t) o[t] += s[j] * decode1(dt, vr[t]);
      }
      for (int64_t t = 0; t < d; ++t) o[t] = nk > 0 ? o[t] / l : 0.0;
      if (lse) lse[h * sq + i] = nk > 0 ? mx + log(l) : -INFINITY;
      free(s);
    }
  return err ? -1 : 0;
}

/* Threads the OpenMP runtime will use (for the cpu_baseline "cores" field). */
#ifdef _OPENMP
#include <omp.h>
int cyo_num_threads(void) { return omp_get_max_threads(); }
void cyo_set_threads(int n) { if (n > 0) omp_set_num_threads(n); }
#else
int cyo_num_threads(void) { return 1; }
void cyo_set_threads(int n) { (void)n; }
#endif
