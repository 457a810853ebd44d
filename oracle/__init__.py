"""fp64 CPU oracle for the Cypress GEMM family (arXiv 2504.07004).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  The product path (``paper_2504_07004_b200``) never imports it and
shares no code with it; the only module both sides use is ``synth`` (seeded
input generators, no method arithmetic).

This is a thin ctypes marshalling layer over ``oracle/oracle.c`` (plain C,
fp64, OpenMP over rows); every computation happens in that file, whose
header cites the PAPER.md passage each function follows:

* ``gemm``          D = alpha*A.B + beta*C
* ``gemm_batched``  L independent GEMMs
* ``dual_gemm``     SUM: alpha*(A.B0 + A.B1)+beta*C P:1529; PAIR: BASELINE configs[3]
* ``rowsum``        y(i) = sum_k A(i,k)
* ``dual_glu``      act(alpha*A.B0) * (alpha*A.B1)    GLU, P:1532 (R14)
* ``attention``     softmax(scale Q K^T) V, lse       Sec. 5.3, P:1594-1611 (FA2/FA3 forward)
* ``encode``/``decode``  IEEE RN-even 16-bit codecs (R7)

Inputs are numpy ``uint16`` arrays of raw fp16/bf16 bit patterns, row-major;
2-D views with a row stride (leading dimension) are accepted as-is.
Outputs are unrounded float64 (``D_ref``); ``encode`` rounds to 16-bit.

Parity pins: ``tests/test_oracle.py`` (codec vs numpy/torch over all 65536
patterns, brute force with exact rationals, numpy.matmul special case,
closed forms).  No function here is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

F16 = 0
BF16 = 1

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile oracle.c -> liboracle.so with gcc (IEEE fp64, no FP contraction)."""
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC):
        tmp = _LIB_PATH + f".tmp{os.getpid()}"
        subprocess.check_call([
            "gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-fopenmp", "-ffp-contract=off",
            "-fno-fast-math", _SRC, "-o", tmp, "-lm"])
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


def _load():
    global _lib
    if _lib is not None:
        return _lib
    build()
    lib = ctypes.CDLL(_LIB_PATH)
    i64, dbl, vp, ci = ctypes.c_int64, ctypes.c_double, ctypes.c_void_p, ctypes.c_int
    lib.cyo_half_to_double.argtypes = [ctypes.c_uint16]
    lib.cyo_half_to_double.restype = dbl
    lib.cyo_bf16_to_double.argtypes = [ctypes.c_uint16]
    lib.cyo_bf16_to_double.restype = dbl
    lib.cyo_double_to_half_rn.argtypes = [dbl]
    lib.cyo_double_to_half_rn.restype = ctypes.c_uint16
    lib.cyo_double_to_bf16_rn.argtypes = [dbl]
    lib.cyo_double_to_bf16_rn.restype = ctypes.c_uint16
    lib.cyo_decode.argtypes = [ci, vp, vp, i64]
    lib.cyo_encode.argtypes = [ci, vp, vp, i64]
    lib.cyo_gemm.argtypes = [ci, i64, i64, i64, dbl, vp, i64, vp, i64, dbl, vp, i64, vp, i64, vp, i64]
    lib.cyo_gemm.restype = ci
    lib.cyo_gemm_batched.argtypes = [ci, i64, i64, i64, i64, dbl, vp, i64, i64, vp, i64, i64, dbl,
                                     vp, i64, i64, vp, i64, i64]
    lib.cyo_gemm_batched.restype = ci
    lib.cyo_dual_gemm.argtypes = [ci, ci, i64, i64, i64, dbl, vp, i64, vp, i64, vp, i64, dbl,
                                  vp, i64, vp, i64, vp, i64, vp, i64, vp, i64]
    lib.cyo_dual_gemm.restype = ci
    lib.cyo_rowsum.argtypes = [ci, i64, i64, vp, i64, vp, vp, i64]
    lib.cyo_rowsum.restype = ci
    lib.cyo_dual_glu.argtypes = [ci, ci, i64, i64, i64, dbl, vp, i64, vp, i64, vp, i64, vp, i64, vp, i64]
    lib.cyo_dual_glu.restype = ci
    lib.cyo_act.argtypes = [ci, dbl]
    lib.cyo_act.restype = dbl
    lib.cyo_attention.argtypes = [ci, i64, i64, i64, i64, dbl, ci, vp, vp, vp, vp, vp]
    lib.cyo_attention.restype = ci
    lib.cyo_num_threads.restype = ci
    lib.cyo_set_threads.argtypes = [ci]
    _lib = lib
    return lib


def _dt(dtype) -> int:
    if dtype in (F16, "f16", "fp16", "float16"):
        return F16
    if dtype in (BF16, "bf16", "bfloat16"):
        return BF16
    raise ValueError(f"unknown 16-bit dtype {dtype!r}")


def _mat(x, name):
    """Return (pointer, ld) for a 2-D uint16 array whose rows may be strided."""
    if x is None:
        return None, 0
    if x.dtype != np.uint16 or x.ndim != 2:
        raise TypeError(f"{name}: expected 2-D uint16 bit patterns, got {x.dtype} {x.ndim}-D")
    if x.size == 0:
        return x.ctypes.data, max(x.shape[1], 1)
    if x.strides[1] != 2 and x.shape[1] > 1:
        raise ValueError(f"{name}: columns must be contiguous")
    return x.ctypes.data, x.strides[0] // 2


def _rows(rows, m):
    if rows is None:
        return None, m, None
    r = np.ascontiguousarray(rows, dtype=np.int64)
    if r.size and (r.min() < 0 or r.max() >= m):
        raise IndexError("row index out of range")
    return r.ctypes.data, r.size, r


def num_threads() -> int:
    return int(_load().cyo_num_threads())


def set_threads(n: int) -> None:
    """OpenMP threads for the oracle (bench: all host cores, whatever OMP_NUM_THREADS says)."""
    _load().cyo_set_threads(int(n))


def decode(dtype, bits) -> np.ndarray:
    bits = np.ascontiguousarray(bits, dtype=np.uint16)
    out = np.empty(bits.shape, dtype=np.float64)
    _load().cyo_decode(_dt(dtype), bits.ctypes.data, out.ctypes.data, bits.size)
    return out


def encode(dtype, x) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.float64)
    out = np.empty(x.shape, dtype=np.uint16)
    _load().cyo_encode(_dt(dtype), x.ctypes.data, out.ctypes.data, x.size)
    return out


def gemm(dtype, A, B, C=None, alpha=1.0, beta=0.0, rows=None) -> np.ndarray:
    """fp64 D_ref = alpha*A.B + beta*C (rows ``rows`` of it, if given)."""
    m, k = A.shape
    k2, n = B.shape
    if k2 != k:
        raise ValueError("inner dimensions differ")
    pa, lda = _mat(A, "A")
    pb, ldb = _mat(B, "B")
    if beta != 0.0:
        if C is None or C.shape != (m, n):
            raise ValueError("C must be m x n when beta != 0")
        pc, ldc = _mat(C, "C")
    else:
        pc, ldc = None, n
    pr, nr, _keep = _rows(rows, m)
    D = np.empty((nr, n), dtype=np.float64)
    rc = _load().cyo_gemm(_dt(dtype), m, n, k, float(alpha), pa, lda, pb, ldb, float(beta), pc, ldc,
                          D.ctypes.data, n, pr, nr)
    if rc:
        raise RuntimeError("cyo_gemm failed")
    return D


def gemm_batched(dtype, A, B, C=None, alpha=1.0, beta=0.0) -> np.ndarray:
    """A: (L, m, k), B: (L, k, n), C: (L, m, n) contiguous uint16 -> (L, m, n) fp64."""
    L, m, k = A.shape
    _, _, n = B.shape
    A = np.ascontiguousarray(A)
    B = np.ascontiguousarray(B)
    D = np.empty((L, m, n), dtype=np.float64)
    if beta != 0.0:
        C = np.ascontiguousarray(C)
        pc = C.ctypes.data
    else:
        pc = None
    rc = _load().cyo_gemm_batched(_dt(dtype), m, n, k, L, float(alpha), A.ctypes.data, k, m * k,
                                  B.ctypes.data, n, k * n, float(beta), pc, n, m * n,
                                  D.ctypes.data, n, m * n)
    if rc:
        raise RuntimeError("cyo_gemm_batched failed")
    return D


def dual_gemm(dtype, mode, A, B0, B1, C0=None, C1=None, alpha=1.0, beta=0.0, rows=None):
    """mode 'pair' -> (D0_ref, D1_ref); mode 'sum' -> D_ref (fp64)."""
    mode_i = {"pair": 0, "sum": 1}[mode]
    m, k = A.shape
    n = B0.shape[1]
    pa, lda = _mat(A, "A")
    pb0, ldb0 = _mat(B0, "B0")
    pb1, ldb1 = _mat(B1, "B1")
    pc0, ldc0 = _mat(C0, "C0") if beta != 0.0 else (None, n)
    pc1, ldc1 = _mat(C1, "C1") if (beta != 0.0 and mode_i == 0) else (None, n)
    pr, nr, _keep = _rows(rows, m)
    D0 = np.empty((nr, n), dtype=np.float64)
    D1 = np.empty((nr, n), dtype=np.float64) if mode_i == 0 else None
    rc = _load().cyo_dual_gemm(_dt(dtype), mode_i, m, n, k, float(alpha), pa, lda, pb0, ldb0, pb1, ldb1,
                               float(beta), pc0, ldc0, pc1, ldc1, D0.ctypes.data, n,
                               D1.ctypes.data if D1 is not None else None, n, pr, nr)
    if rc:
        raise RuntimeError("cyo_dual_gemm failed")
    return (D0, D1) if mode_i == 0 else D0


ACTS = {"silu": 0, "gelu_tanh": 1}


def act(name, x) -> np.ndarray:
    """The oracle's activation (fp64), elementwise."""
    f = _load().cyo_act
    a = ACTS[name]
    return np.vectorize(lambda v: f(a, float(v)), otypes=[np.float64])(np.asarray(x, dtype=np.float64))


def dual_glu(dtype, act_name, A, B0, B1, alpha=1.0, rows=None) -> np.ndarray:
    """fp64 D_ref = act(alpha*A.B0) * (alpha*A.B1)  (GLU)."""
    m, k = A.shape
    n = B0.shape[1]
    pa, lda = _mat(A, "A")
    pb0, ldb0 = _mat(B0, "B0")
    pb1, ldb1 = _mat(B1, "B1")
    pr, nr, _keep = _rows(rows, m)
    D = np.empty((nr, n), dtype=np.float64)
    rc = _load().cyo_dual_glu(_dt(dtype), ACTS[act_name], m, n, k, float(alpha), pa, lda, pb0, ldb0, pb1, ldb1,
                              D.ctypes.data, n, pr, nr)
    if rc:
        raise RuntimeError("cyo_dual_glu failed")
    return D


def attention(dtype, Q, K, V, scale=None, causal=False):
    """fp64 (O, lse) of softmax(scale * Q K^T) V per (batch*head); Q: (BH, sq, d), K/V: (BH, sk, d)."""
    Q, K, V = (np.ascontiguousarray(x, dtype=np.uint16) for x in (Q, K, V))
    bh, sq, d = Q.shape
    sk = K.shape[1]
    if scale is None:
        scale = 1.0 / np.sqrt(d)
    O = np.empty((bh, sq, d), dtype=np.float64)
    lse = np.empty((bh, sq), dtype=np.float64)
    rc = _load().cyo_attention(_dt(dtype), bh, sq, sk, d, float(scale), int(bool(causal)), Q.ctypes.data,
                               K.ctypes.data, V.ctypes.data, O.ctypes.data, lse.ctypes.data)
    if rc:
        raise RuntimeError("cyo_attention failed")
    return O, lse


def rowsum(dtype, A, rows=None) -> np.ndarray:
    """y(i) = sum_k A(i,k) in fp64."""
    m, k = A.shape
    pa, lda = _mat(A, "A")
    pr, nr, _keep = _rows(rows, m)
    y = np.empty(nr, dtype=np.float64)
    rc = _load().cyo_rowsum(_dt(dtype), m, k, pa, lda, y.ctypes.data, pr, nr)
    if rc:
        raise RuntimeError("cyo_rowsum failed")
    return y


def tolerance(D_ref, k, sum_terms: int = 1):
    """Per-element bound from BASELINE.json north_star:
    |D - D_ref| <= 2^-8 |D_ref| + 1e-3 sqrt(K)   (sqrt(2K) for dual SUM)."""
    return 2.0 ** -8 * np.abs(D_ref) + 1e-3 * np.sqrt(sum_terms * k)
