"""paper_2504_07004_b200 -- B200-native (sm_100a) implementation of the GEMM family that
Cypress (arXiv 2504.07004) compiles: D = alpha*A*B + beta*C with fp32 accumulation, batched,
dual-GEMM and GEMM + row reduction.

Thin Python binding over the C ABI in ``include/cypress_b200.h`` (``libcypress_b200.so``):
argument marshalling only -- every arithmetic step runs in the sm_100a kernels.  PyTorch is
used for device memory and streams.  There is no CPU / library fallback: a missing extension
raises.

Entry points (same names as the C ABI, plus torch conveniences):
  gemm(A, B, C=None, alpha=1, beta=0, out=None)            -> D            cy_gemm
  gemm_batched(A, B, C=None, alpha=1, beta=0, out=None)    -> D (L,m,n)    cy_gemm_batched
  dual_gemm(A, B0, B1, C0=None, C1=None, mode="pair", ...) -> (D0, D1) | D cy_dual_gemm
  gemm_rowreduce(A, B, C=None, alpha=1, beta=0, ...)       -> (D, y)       cy_gemm_rowreduce
  dual_gemm_glu(A, B0, B1, act="silu", alpha=1, out=None)  -> D            cy_dual_gemm_glu
Raw pointer calls: ``paper_2504_07004_b200.cy_gemm(...)`` etc. (ctypes signatures of the header).
"""
from __future__ import annotations

from . import _lib
from ._lib import CY_BF16, CY_DUAL_PAIR, CY_DUAL_SUM, CY_F16, CyError, check

__all__ = [
    "gemm", "gemm_batched", "dual_gemm", "dual_gemm_glu", "gemm_rowreduce", "gemm_replicated", "attention", "CyError", "force_config", "last_config",
    "num_configs", "config_info", "launch_count", "last_kernel_info", "last_splits", "cy_gemm", "cy_gemm_batched", "cy_dual_gemm",
    "cy_gemm_rowreduce", "CY_F16", "CY_BF16", "CY_DUAL_PAIR", "CY_DUAL_SUM",
]


def __getattr__(name):
    # raw C-ABI entry points: paper_2504_07004_b200.cy_gemm(...) -> status
    if name.startswith("cy_") and name in _lib.EXPORTS:
        return getattr(_lib.load(), name)
    raise AttributeError(name)


def _torch():
    import torch

    return torch


def _dt(t):
    torch = _torch()
    if t.dtype == torch.float16:
        return CY_F16
    if t.dtype == torch.bfloat16:
        return CY_BF16
    raise TypeError(f"cypress_b200: unsupported dtype {t.dtype} (fp16 / bf16 only)")


def _ld(t, name):
    st, sh = t.stride(), t.shape  # (two attribute reads: this runs for every operand of every call)
    if len(st) != 2:
        raise ValueError(f"{name}: expected a 2-D tensor")
    if st[1] != 1 and sh[1] > 1:
        raise ValueError(f"{name}: rows must be contiguous (row-major, stride(1) == 1)")
    return st[0] if sh[0] > 1 else max(st[0], sh[1])


def _empty2d(m, n, like):
    """Row-major m x n output whose row stride is padded to a multiple of 8 elements."""
    torch = _torch()
    ld = (n + 7) // 8 * 8
    return torch.empty((m, ld), dtype=like.dtype, device=like.device)[:, :n]


def _ptr(t):
    return None if t is None else t.data_ptr()


def _stream(stream, dev):
    if stream is None:
        torch = _torch()
        return torch._C._cuda_getCurrentRawStream(dev if dev >= 0 else torch.cuda.current_device())
    return getattr(stream, "cuda_stream", stream)


def _check_dev(*ts):
    """All tensors must live on one CUDA device; returns its index.  Uses get_device() (an int)
    rather than .device objects: this runs on every call."""
    dev = -2
    for t in ts:
        if t is None:
            continue
        g = t.get_device()
        if g < 0:
            raise ValueError("cypress_b200: all tensors must be CUDA tensors (no CPU fallback)")
        if dev == -2:
            dev = g
        elif g != dev:
            raise ValueError(f"cypress_b200: tensors on different devices (cuda:{dev} vs cuda:{g})")
    return dev


class _on_device:
    """The C ABI works on the CURRENT device: make ``dev`` current for the call and restore the
    caller's device afterwards (torch semantics; a no-op when it is already current)."""

    __slots__ = ("dev", "prev")

    def __init__(self, dev):
        self.dev = dev
        self.prev = -1

    def __enter__(self):
        if self.dev >= 0:
            torch = _torch()
            cur = torch.cuda.current_device()
            if cur != self.dev:
                self.prev = cur
                torch.cuda.set_device(self.dev)
        return self

    def __exit__(self, *exc):
        if self.prev >= 0:
            _torch().cuda.set_device(self.prev)
        return False


def _same_dtype(ref, *named):
    for t, name in named:
        if t is not None and t.dtype != ref.dtype:
            raise ValueError(f"cypress_b200: {name} is {t.dtype}, A is {ref.dtype} (one 16-bit type for all operands)")


def _shape(t, want, name):
    if t is not None and tuple(t.shape) != tuple(want):
        raise ValueError(f"cypress_b200: {name} has shape {tuple(t.shape)}, expected {tuple(want)}")


def _mat2(A, B):
    if A.dim() != 2 or B.dim() != 2:
        raise ValueError("cypress_b200: A and B must be 2-D")
    m, k = A.shape
    if B.shape[0] != k:
        raise ValueError(f"cypress_b200: inner dimensions differ (A is {tuple(A.shape)}, B is {tuple(B.shape)})")
    return m, B.shape[1], k


_WS = {}        # (device, stream) -> split-K workspace (uint8 tensor)
_WS_NEED = {}   # (dtype, m, n, k, batch, splits, device, forced config) -> workspace bytes (0: not split)


_FORCED = [-1]  # the config forced through force_config() (part of the workspace-size cache key)


def _splitk_need(dt, m, n, k, L, splits, dev):
    key = (dt, m, n, k, L, splits, dev, _FORCED[0])
    need = _WS_NEED.get(key)
    if need is None:
        with _on_device(dev):
            need = int(_lib.load().cy_gemm_splitk_workspace_size(dt, m, n, k, L, splits))
        _WS_NEED[key] = need
    return need


def _workspace(dev, stream_handle, nbytes):
    """Split-K workspace for (device, stream): calls on one stream reuse it (stream order; the
    kernel's arrival counters are tagged per launch, so no zero fill); other streams get their own."""
    torch = _torch()
    key = (dev, int(stream_handle or 0))
    ws = _WS.get(key)
    if ws is None or ws.numel() < nbytes:
        ws = torch.empty((max(nbytes, 1 << 20),), dtype=torch.uint8, device=torch.device("cuda", dev))
        _WS[key] = ws
    return ws


def _gemm_call(dt, m, n, k, L, alpha, A, lda, sa, B, ldb, sb, beta, C, ldc, sc, D, ldd, sd, stream, dev, splits,
               what):
    """cy_gemm_batched, or cy_gemm_splitk when split-K is requested (splits > 1) or chosen by the
    library's cost model (splits=None: auto; the choice per shape is cached)."""
    lib = _lib.load()
    sk = 0 if splits is None else int(splits)
    need = 0 if sk == 1 else _splitk_need(dt, m, n, k, L, sk, dev)
    if need == 0 and sk <= 1 and L == 1 and sa == sb == sc == sd == 0:
        st = lib.cy_gemm(dt, m, n, k, float(alpha), A, lda, B, ldb, float(beta), C, ldc, D, ldd, stream)
    elif need == 0 and sk <= 1:
        st = lib.cy_gemm_batched(dt, m, n, k, L, float(alpha), A, lda, sa, B, ldb, sb, float(beta), C, ldc, sc, D,
                                 ldd, sd, stream)
    else:
        ws = _workspace(dev, stream, need)
        st = lib.cy_gemm_splitk(dt, m, n, k, L, float(alpha), A, lda, sa, B, ldb, sb, float(beta), C, ldc, sc, D, ldd,
                                sd, sk, ws.data_ptr(), ws.numel(), stream)
    check(st, what)


def gemm(A, B, C=None, alpha: float = 1.0, beta: float = 0.0, out=None, stream=None, splits=None):
    """D = alpha*A@B + beta*C  (A: m x k, B: k x n, row-major).  cy_gemm / cy_gemm_splitk.
    splits: None = the library's choice (split-K only where its cost model predicts a gain),
    1 = never split, S > 1 = split K into S parts."""
    dev = _check_dev(A, B, C, out)
    m, n, k = _mat2(A, B)
    use_c = beta != 0
    if use_c and C is None:
        raise ValueError("cypress_b200: beta != 0 needs C")
    _same_dtype(A, (B, "B"), (C if use_c else None, "C"), (out, "out"))
    _shape(C if use_c else None, (m, n), "C")
    _shape(out, (m, n), "out")
    if out is None:
        out = _empty2d(m, n, A)
    with _on_device(dev):
        _gemm_call(_dt(A), m, n, k, 1, alpha, _ptr(A), _ld(A, "A"), 0, _ptr(B), _ld(B, "B"), 0, beta,
                   _ptr(C) if use_c else None, _ld(C, "C") if use_c else n, 0, _ptr(out), _ld(out, "out"), 0,
                   _stream(stream, dev), dev, splits, "cy_gemm")
    return out


def gemm_batched(A, B, C=None, alpha: float = 1.0, beta: float = 0.0, out=None, stream=None, splits=None):
    """D[b] = alpha*A[b]@B[b] + beta*C[b] for b < L (3-D tensors, rows contiguous)."""
    torch = _torch()
    dev = _check_dev(A, B, C, out)
    if A.dim() != 3 or B.dim() != 3:
        raise ValueError("cypress_b200: batched A and B must be 3-D (L, rows, cols)")
    L, m, k = A.shape
    if B.shape[0] != L or B.shape[1] != k:
        raise ValueError(f"cypress_b200: B has shape {tuple(B.shape)}, expected ({L}, {k}, n)")
    n = B.shape[2]
    use_c = beta != 0
    if use_c and C is None:
        raise ValueError("cypress_b200: beta != 0 needs C")
    _same_dtype(A, (B, "B"), (C if use_c else None, "C"), (out, "out"))
    _shape(C if use_c else None, (L, m, n), "C")
    _shape(out, (L, m, n), "out")
    if out is None:
        out = torch.empty((L, m, n), dtype=A.dtype, device=A.device)

    def lds(t):
        if t is None:
            return n, 0
        if t.stride(2) != 1 and t.size(2) > 1:
            raise ValueError("cypress_b200: rows must be contiguous")
        return t.stride(1), t.stride(0)

    lda, sa = lds(A)
    ldb, sb = lds(B)
    ldc, sc = lds(C if use_c else None)
    ldd, sd = lds(out)
    with _on_device(dev):
        _gemm_call(_dt(A), m, n, k, L, alpha, _ptr(A), lda, sa, _ptr(B), ldb, sb, beta, _ptr(C) if use_c else None,
                   ldc, sc, _ptr(out), ldd, sd, _stream(stream, dev), dev, splits, "cy_gemm_batched")
    return out


def dual_gemm(A, B0, B1, C0=None, C1=None, alpha: float = 1.0, beta: float = 0.0, mode: str = "pair",
              out0=None, out1=None, stream=None):
    """mode "pair": (D0, D1) = (alpha*A@B0 + beta*C0, alpha*A@B1 + beta*C1);
    mode "sum": D = alpha*(A@B0 + A@B1) + beta*C0.  cy_dual_gemm."""
    dev = _check_dev(A, B0, B1, C0, C1, out0, out1)
    if mode not in ("pair", "sum"):
        raise ValueError("mode must be 'pair' or 'sum'")
    pair = mode == "pair"
    m, n, k = _mat2(A, B0)
    _shape(B1, (k, n), "B1")
    use_c = beta != 0
    if use_c and (C0 is None or (pair and C1 is None)):
        raise ValueError("cypress_b200: beta != 0 needs C0 (and C1 in pair mode)")
    if not pair and (C1 is not None or out1 is not None):
        raise ValueError("cypress_b200: sum mode takes no C1 / out1")
    _same_dtype(A, (B0, "B0"), (B1, "B1"), (C0 if use_c else None, "C0"), (C1 if use_c else None, "C1"),
                (out0, "out0"), (out1, "out1"))
    for t, name in ((C0 if use_c else None, "C0"), (C1 if use_c else None, "C1"), (out0, "out0"), (out1, "out1")):
        _shape(t, (m, n), name)
    if out0 is None:
        out0 = _empty2d(m, n, A)
    if pair and out1 is None:
        out1 = _empty2d(m, n, A)
    with _on_device(dev):
        st = _lib.load().cy_dual_gemm(
            _dt(A), CY_DUAL_PAIR if pair else CY_DUAL_SUM, m, n, k, float(alpha), _ptr(A), _ld(A, "A"), _ptr(B0),
            _ld(B0, "B0"), _ptr(B1), _ld(B1, "B1"), float(beta), _ptr(C0) if use_c else None,
            _ld(C0, "C0") if use_c else n, _ptr(C1) if (use_c and pair) else None,
            _ld(C1, "C1") if (use_c and pair) else n, _ptr(out0), _ld(out0, "out0"),
            _ptr(out1) if pair else None, _ld(out1, "out1") if pair else n, _stream(stream, dev))
    check(st, "cy_dual_gemm")
    return (out0, out1) if pair else out0


def attention(Q, K, V, scale=None, causal: bool = False, out=None, lse=None, stream=None):
    """Forward attention O = softmax(scale Q K^T) V (FA2/FA3 forward, HeadDim 128).
    Q: (batch, heads, seq_q, 128), K/V: (batch, heads, seq_k, 128), contiguous fp16/bf16.
    Returns (O, lse) with lse (batch, heads, seq_q) fp32 natural log-sum-exp.  cy_attention_fwd."""
    torch = _torch()
    dev = _check_dev(Q, K, V, out, lse)
    if Q.dim() != 4 or K.dim() != 4 or V.dim() != 4:
        raise ValueError("cypress_b200: Q, K, V must be 4-D (batch, heads, seq, head_dim)")
    b, h, sq, d = Q.shape
    sk = K.shape[2]
    if tuple(K.shape) != (b, h, sk, d):
        raise ValueError(f"cypress_b200: K has shape {tuple(K.shape)}, expected ({b}, {h}, seq_k, {d}) "
                         "(same batch, heads and head_dim as Q; no GQA/MQA broadcast)")
    if tuple(V.shape) != tuple(K.shape):
        raise ValueError(f"cypress_b200: V has shape {tuple(V.shape)}, expected K's {tuple(K.shape)}")
    _same_dtype(Q, (K, "K"), (V, "V"), (out, "out"))
    for t, name in ((Q, "Q"), (K, "K"), (V, "V"), (out, "out"), (lse, "lse")):
        if t is not None and not t.is_contiguous():
            raise ValueError(f"cypress_b200: {name} must be contiguous")
    _shape(out, (b, h, sq, d), "out")
    _shape(lse, (b, h, sq), "lse")
    if lse is not None and lse.dtype != torch.float32:
        raise ValueError("cypress_b200: lse must be float32")
    if scale is None:
        scale = d ** -0.5
    if out is None:
        out = torch.empty_like(Q)
    if lse is None:
        lse = torch.empty((b, h, sq), dtype=torch.float32, device=Q.device)
    with _on_device(dev):
        st = _lib.load().cy_attention_fwd(_dt(Q), b, h, sq, sk, d, float(scale), int(bool(causal)), _ptr(Q),
                                          _ptr(K), _ptr(V), _ptr(out), _ptr(lse), _stream(stream, dev))
    check(st, "cy_attention_fwd")
    return out, lse


def gemm_replicated(A, B, dsts, row_offset: int, rows_total: int, C=None, alpha: float = 1.0, beta: float = 0.0,
                    ldd=None, stream=None):
    """Compute D_shard = alpha*A@B + beta*C and store it at rows [row_offset, row_offset + m) of every
    destination in ``dsts`` (2-D tensors or raw device addresses of rows_total x n matrices with
    leading dimension ``ldd``; taken from the first tensor if not given, required for raw addresses).
    cy_gemm_replicated (fused replication; the destinations are usually peers' buffers)."""
    import ctypes

    dev = _check_dev(A, B, C)
    m, n, k = _mat2(A, B)
    use_c = beta != 0
    if use_c and C is None:
        raise ValueError("cypress_b200: beta != 0 needs C")
    _same_dtype(A, (B, "B"), (C if use_c else None, "C"))
    _shape(C if use_c else None, (m, n), "C")
    ptrs = []
    for d in dsts:
        if isinstance(d, int):
            ptrs.append(d)
            continue
        _same_dtype(A, (d, "dst"))
        _shape(d, (rows_total, n), "dst")
        if ldd is None:
            ldd = _ld(d, "dst")
        elif _ld(d, "dst") != ldd:
            raise ValueError("cypress_b200: every destination must have leading dimension ldd")
        ptrs.append(d.data_ptr())
    if ldd is None:
        raise ValueError("cypress_b200: raw destination addresses need ldd")
    arr = (ctypes.c_void_p * len(ptrs))(*ptrs)
    with _on_device(dev):
        st = _lib.load().cy_gemm_replicated(_dt(A), m, n, k, float(alpha), _ptr(A), _ld(A, "A"), _ptr(B),
                                            _ld(B, "B"), float(beta), _ptr(C) if use_c else None,
                                            _ld(C, "C") if use_c else n, arr, len(ptrs), int(ldd), int(row_offset),
                                            int(rows_total), _stream(stream, dev))
    check(st, "cy_gemm_replicated")


def dual_gemm_glu(A, B0, B1, act: str = "silu", alpha: float = 1.0, out=None, stream=None):
    """D = act(alpha*A@B0) * (alpha*A@B1), act in {"silu", "gelu_tanh"} (GLU).  cy_dual_gemm_glu."""
    dev = _check_dev(A, B0, B1, out)
    m, n, k = _mat2(A, B0)
    _shape(B1, (k, n), "B1")
    _same_dtype(A, (B0, "B0"), (B1, "B1"), (out, "out"))
    _shape(out, (m, n), "out")
    if act not in ("silu", "gelu_tanh"):
        raise ValueError("act must be 'silu' or 'gelu_tanh'")
    a = {"silu": _lib.CY_ACT_SILU, "gelu_tanh": _lib.CY_ACT_GELU_TANH}[act]
    if out is None:
        out = _empty2d(m, n, A)
    with _on_device(dev):
        st = _lib.load().cy_dual_gemm_glu(_dt(A), a, m, n, k, float(alpha), _ptr(A), _ld(A, "A"), _ptr(B0),
                                          _ld(B0, "B0"), _ptr(B1), _ld(B1, "B1"), _ptr(out), _ld(out, "out"),
                                          _stream(stream, dev))
    check(st, "cy_dual_gemm_glu")
    return out


def gemm_rowreduce(A, B, C=None, alpha: float = 1.0, beta: float = 0.0, out=None, y=None, stream=None):
    """D = alpha*A@B + beta*C and y[i] = sum_k A[i,k] (fp32), one kernel.  cy_gemm_rowreduce."""
    torch = _torch()
    dev = _check_dev(A, B, C, out, y)
    m, n, k = _mat2(A, B)
    use_c = beta != 0
    if use_c and C is None:
        raise ValueError("cypress_b200: beta != 0 needs C")
    _same_dtype(A, (B, "B"), (C if use_c else None, "C"), (out, "out"))
    _shape(C if use_c else None, (m, n), "C")
    _shape(out, (m, n), "out")
    _shape(y, (m,), "y")
    if y is not None and (y.dtype != torch.float32 or (m > 1 and y.stride(0) != 1)):
        raise ValueError("cypress_b200: y must be a contiguous float32 vector")
    if out is None:
        out = _empty2d(m, n, A)
    if y is None:
        y = torch.empty((m,), dtype=torch.float32, device=A.device)
    with _on_device(dev):
        st = _lib.load().cy_gemm_rowreduce(
            _dt(A), m, n, k, float(alpha), _ptr(A), _ld(A, "A"), _ptr(B), _ld(B, "B"), float(beta),
            _ptr(C) if use_c else None, _ld(C, "C") if use_c else n, _ptr(out),
            _ld(out, "out") if n > 0 else max(8, out.stride(0)), _ptr(y), _stream(stream, dev))
    check(st, "cy_gemm_rowreduce")
    return out, y


def force_config(cfg_id: int):
    check(_lib.load().cy_force_config(int(cfg_id)), "cy_force_config")
    _FORCED[0] = int(cfg_id)


def last_config() -> int:
    return int(_lib.load().cy_last_config())


def num_configs() -> int:
    return int(_lib.load().cy_num_configs())


def config_info(cfg_id: int) -> dict:
    import ctypes

    v = [ctypes.c_int() for _ in range(4)]
    check(_lib.load().cy_config_info(int(cfg_id), *[ctypes.byref(x) for x in v]), "cy_config_info")
    return {"cta_group": v[0].value, "tile_m": v[1].value, "tile_n": v[2].value, "stages": v[3].value}


VARIANTS = {0: "gemm", 1: "dual_pair", 2: "dual_sum", 3: "rowreduce", 4: "dual_glu"}


def last_kernel_info() -> dict:
    """Exact kernel (variant, tile, stages, threads, smem) of the most recent launch."""
    import ctypes

    v = [ctypes.c_int() for _ in range(8)]
    check(_lib.load().cy_last_kernel_info(*[ctypes.byref(x) for x in v]), "cy_last_kernel_info")
    keys = ("variant", "cta_group", "tile_m", "tile_n", "stages", "threads", "smem_bytes", "dtype")
    d = dict(zip(keys, (x.value for x in v)))
    d["variant"] = VARIANTS.get(d["variant"], d["variant"])
    d["dtype"] = "f16" if d["dtype"] == 0 else "bf16"
    return d


def last_splits() -> int:
    """Split count of the most recent GEMM-family launch (1 = not split)."""
    return int(_lib.load().cy_last_splits())


def launch_count() -> int:
    return int(_lib.load().cy_launch_count())
