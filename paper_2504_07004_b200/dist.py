"""Multi-GPU partitioning of the GEMM family.

One process per GPU (torchrun), ``torch.distributed`` for the plumbing.  The path shards
naturally -- independent output row blocks (GEMM, dual, row-reduce) or batch indices
(batched) -- so no collective sits on the data path: every rank computes its own shard with
the sm_100a kernels and B is replicated.  Only when the caller asks for a replicated result
(``replicate=True``) is D (and y) all-gathered over NCCL (NVLink / NVSwitch); row-major D makes
each rank's shard a contiguous row block, so the gather needs no packing.

Fused replication: ``replicate="fused"`` skips the all-gather; the kernel's
epilogue stores each output tile into every rank's replicated D through peer mappings
(``cy_gemm_replicated``).  It needs CUDA peer access (NVLink) and NCCL-backed symmetric memory;
the kernel side is tested on one GPU with local destinations.

Shard geometry: ``rows_per = ceil(m / world)`` rounded up to ``align`` (256 = the CTA-pair tile
height, BASELINE configs[4]); rank r owns rows [r*rows_per, min(m, (r+1)*rows_per)).  Uneven
tails are gathered through a padded buffer and sliced.

``gemm_fn`` hooks exist so host-side logic (sharding, gathering, assembly) can be tested
on CPU with the gloo backend; the product default is the CUDA path, which has no fallback.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def _world(group):
    if not dist.is_available() or not dist.is_initialized():
        return 1, 0
    return dist.get_world_size(group), dist.get_rank(group)


def shard_rows(m: int, world: int, rank: int, align: int = 256):
    """Contiguous row block [start, end) of rank ``rank`` and the padded per-rank row count."""
    per = -(-m // max(world, 1))
    per = -(-per // align) * align if align > 1 else per
    start = min(m, rank * per)
    end = min(m, (rank + 1) * per)
    return start, end, per


def shard_batches(L: int, world: int, rank: int):
    per = -(-L // max(world, 1))
    start = min(L, rank * per)
    return start, min(L, start + per), per


def _default_gemm():
    from . import gemm

    return gemm


def _gather_rows(local_padded, m, per, world, group):
    """all_gather contiguous row blocks (each ``per`` rows, the last ones possibly short)."""
    full = torch.empty((per * world,) + tuple(local_padded.shape[1:]), dtype=local_padded.dtype,
                       device=local_padded.device)
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(full, local_padded.contiguous(), group=group)
    else:  # gloo (CPU tests of the host logic; CUDA tensors are staged through host memory)
        host = full.cpu() if full.is_cuda else full
        dist.all_gather(list(host.chunk(world)), local_padded.contiguous().cpu(), group=group)
        if host is not full:
            full.copy_(host)
    return full[:m]


_SYMM_CACHE = {}


def _symm_buffer(rows, n, dtype, device, group):
    """One symmetric-memory (NVLink-mapped) D buffer per (shape, dtype, group), reused across calls."""
    from torch.distributed import _symmetric_memory as symm

    key = (rows, n, dtype, device, id(group))
    if key not in _SYMM_CACHE:
        buf = symm.empty((rows, n), dtype=dtype, device=device)
        hdl = symm.rendezvous(buf, group if group is not None else dist.group.WORLD)
        _SYMM_CACHE[key] = (buf, hdl)
    return _SYMM_CACHE[key]


def sharded_gemm(A_local, B, C_local=None, alpha=1.0, beta=0.0, *, m_total=None, group=None,
                 replicate=False, align=256, gemm_fn=None):
    """Rank-local D = alpha*A_local@B + beta*C_local (A_local = this rank's row block).

    replicate=False:   returns the local D block (no communication).
    replicate=True:    returns the full (m_total x n) D on every rank via one NCCL all-gather.
    replicate="fused": the GEMM epilogue writes every tile straight into every rank's replicated D
                       (symmetric memory over NVLink, cy_gemm_replicated) -- no separate collective;
                       a device barrier then orders the peers.  Returns a view of a cached
                       symmetric buffer (overwritten by the next call with the same shape).
    """
    world, rank = _world(group)
    rows, n = A_local.shape[0], B.shape[1]
    if replicate == "fused" and world > 1:
        from . import gemm_replicated

        m = m_total if m_total is not None else rows * world
        start, _, per = shard_rows(m, world, rank, align)
        buf, hdl = _symm_buffer(per * world, n, A_local.dtype, A_local.device, group)
        ptrs = [int(hdl.buffer_ptrs[r]) for r in range(world)]
        gemm_replicated(A_local, B, ptrs, row_offset=start, rows_total=per * world, C=C_local, alpha=alpha,
                        beta=beta)
        hdl.barrier(channel=0)  # every rank's stores are visible before anyone reads
        return buf[:m]
    gemm_fn = gemm_fn or _default_gemm()
    if not replicate or world == 1:
        return gemm_fn(A_local, B, C_local, alpha, beta)
    m = m_total if m_total is not None else rows * world
    _, _, per = shard_rows(m, world, rank, align)
    if rows > per:
        raise ValueError(f"local block has {rows} rows > per-rank {per}")
    padded = torch.zeros((per, n), dtype=A_local.dtype, device=A_local.device)
    gemm_fn(A_local, B, C_local, alpha, beta, out=padded[:rows])  # computed in place, no copy
    return _gather_rows(padded, m, per, world, group)


def sharded_gemm_rowreduce(A_local, B, C_local=None, alpha=1.0, beta=0.0, *, m_total=None, group=None,
                           replicate=False, align=256, rowreduce_fn=None):
    """Rank-local (D, y) of the fused GEMM + row reduction; replicate=True all-gathers both
    (BASELINE configs[4]: M-sharded over 8 GPUs + NCCL all-gather)."""
    if rowreduce_fn is None:
        from . import gemm_rowreduce as rowreduce_fn
    world, rank = _world(group)
    rows, n = A_local.shape[0], B.shape[1]
    if not replicate or world == 1:
        return rowreduce_fn(A_local, B, C_local, alpha, beta)
    m = m_total if m_total is not None else rows * world
    _, _, per = shard_rows(m, world, rank, align)
    Dp = torch.zeros((per, n), dtype=A_local.dtype, device=A_local.device)
    yp = torch.zeros((per,), dtype=torch.float32, device=A_local.device)
    rowreduce_fn(A_local, B, C_local, alpha, beta, out=Dp[:rows], y=yp[:rows])  # in place
    return _gather_rows(Dp, m, per, world, group), _gather_rows(yp, m, per, world, group)


def sharded_gemm_batched(A_local, B_local, C_local=None, alpha=1.0, beta=0.0, *, L_total=None, group=None,
                         replicate=False, batched_fn=None):
    """Batch-index sharding: this rank holds batches [start, end) of A, B (and C)."""
    if batched_fn is None:
        from . import gemm_batched as batched_fn
    world, rank = _world(group)
    D = batched_fn(A_local, B_local, C_local, alpha, beta)
    if not replicate or world == 1:
        return D
    L = L_total if L_total is not None else A_local.shape[0] * world
    _, _, per = shard_batches(L, world, rank)
    Dp = torch.zeros((per,) + tuple(D.shape[1:]), dtype=D.dtype, device=D.device)
    Dp[: D.shape[0]].copy_(D)
    return _gather_rows(Dp, L, per, world, group)


def sharded_dual_gemm(A_local, B0, B1, alpha=1.0, mode="pair", *, m_total=None, group=None, replicate=False,
                      align=256, dual_fn=None):
    if dual_fn is None:
        from . import dual_gemm

        def dual_fn(A, X, Y, a):
            return dual_gemm(A, X, Y, alpha=a, mode=mode)
    world, rank = _world(group)
    out = dual_fn(A_local, B0, B1, alpha)
    if not replicate or world == 1:
        return out
    outs = out if isinstance(out, tuple) else (out,)
    rows = A_local.shape[0]
    m = m_total if m_total is not None else rows * world
    _, _, per = shard_rows(m, world, rank, align)
    res = []
    for D in outs:
        Dp = torch.zeros((per, D.shape[1]), dtype=D.dtype, device=D.device)
        Dp[:rows].copy_(D)
        res.append(_gather_rows(Dp, m, per, world, group))
    return tuple(res) if isinstance(out, tuple) else res[0]
