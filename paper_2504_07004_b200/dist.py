"""Multi-GPU partitioning of the GEMM family (NEXT-2).

One process per GPU (torchrun), ``torch.distributed`` for the plumbing.  The path shards
naturally -- independent output row blocks (GEMM, dual, row-reduce) or batch indices
(batched) -- so no collective sits on the data path: every rank computes its own shard with
the sm_100a kernels and B is replicated (BASELINE configs[2, 4]).  Only when the caller asks for
a replicated result is D (and y) exchanged:

``replicate=True``   the shard is computed in ``chunks`` row blocks straight into its place in
                     the full output; right after chunk j's kernel is queued, chunk j is sent to
                     every peer and every peer's chunk j received into place (NCCL point-to-point
                     in one group call).  ProcessGroupNCCL runs it on its own stream, which waits
                     only for the work queued so far, so chunk j's exchange overlaps chunk j+1's
                     GEMM ("separate comm stream, chunked by row-block").  Row-major D
                     makes each block contiguous: no packing, no copy.
``replicate="fused"`` no collective at all: the GEMM epilogue stores every tile into every
                     rank's replicated D through CUDA-IPC peer mappings (cy_gemm_replicated,
                     SURVEY NEXT-2), ordered by the device-side cy_peer_barrier before (peers done
                     reading the previous result) and after (all stores landed).

Shard geometry: ``per = ceil(m / world)`` rounded up to ``align`` (256 = the CTA-pair tile
height); rank r owns rows [r*per, min(m, (r+1)*per)).  The full result is a (per*world)-row
buffer sliced to m rows, so every rank's block sits at row r*per.

``*_fn`` hooks let the host logic (sharding, exchange, assembly) be tested on CPU with gloo and
reference-backed CPU compute injected by the tests; the product default is the CUDA path, which has no fallback.  With gloo
and CUDA tensors (one-GPU multi-rank tests) the exchange is staged through host memory.
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


def _ld8(n):
    return (n + 7) // 8 * 8


def _gather_buffer(rows, n, dtype, device):
    """(rows, ld8) contiguous gather target: the row stride is padded to the 16-byte TMA rule, so
    every row block is contiguous and any [r0:r1, :n] view is a valid kernel output."""
    return torch.empty((rows, _ld8(n)), dtype=dtype, device=device)


def _p2p_capable(t, group):
    backend = dist.get_backend(group)
    return backend == "nccl" or (backend == "gloo" and not t.is_cuda)


def _global(group, r):
    return r if group is None else dist.get_global_rank(group, r)


def _exchange(bufs_blocks, rank, world, group):
    """Point-to-point exchange of row blocks: for every (buf, blocks) pair, blocks[p] = (r0, r1)
    are the rows of ``buf`` that rank p owns in this exchange; each rank sends its own block to
    every peer and receives every peer's block into place.  Returns the async works."""
    ops = []
    for buf, blocks in bufs_blocks:
        r0, r1 = blocks[rank]
        for p in range(world):
            if p == rank:
                continue
            if r1 > r0:
                ops.append(dist.P2POp(dist.isend, buf[r0:r1], _global(group, p), group))
            q0, q1 = blocks[p]
            if q1 > q0:
                ops.append(dist.P2POp(dist.irecv, buf[q0:q1], _global(group, p), group))
    return dist.batch_isend_irecv(ops) if ops else []


def _gather_staged(buf, per, world, group):
    """all_gather of the per-rank row blocks of ``buf`` (shape (per*world, ...)) through host memory
    (gloo with CUDA tensors: the one-GPU multi-rank tests)."""
    host = buf.cpu()
    chunks = list(host.chunk(world))
    mine = chunks[dist.get_rank(group)].clone()
    dist.all_gather(chunks, mine, group=group)
    buf.copy_(host)


def _rows_of(p, m, per):
    return max(0, min(m, (p + 1) * per) - p * per)


def _row_sharded(rows, m, per, world, rank, group, bufs, compute, chunks, align):
    """Compute this rank's rows into their place in the full buffers and exchange them.

    bufs: full gather buffers, first dim per*world.  compute(r0, r1, views): local rows [r0, r1)
    into views[i] = bufs[i][rank*per + r0 : rank*per + r1].  Chunk j's exchange is queued right
    after chunk j's compute (overlap on the NCCL stream)."""
    if rows != _rows_of(rank, m, per):
        raise ValueError(f"rank {rank} holds {rows} rows; the shard geometry gives {_rows_of(rank, m, per)}")
    base = rank * per
    if not _p2p_capable(bufs[0], group):
        if rows:
            compute(0, rows, [b[base:base + rows] for b in bufs])
        for b in bufs:
            _gather_staged(b, per, world, group)
        return
    nch = max(1, int(chunks))
    cs = -(-per // nch)
    if align > 1 and per >= align:
        cs = -(-cs // align) * align
    works = []
    for j in range(-(-per // cs)):
        c0, c1 = j * cs, min(per, (j + 1) * cs)
        mine = (c0, min(c1, rows))
        if mine[1] > mine[0]:
            compute(mine[0], mine[1], [b[base + mine[0]:base + mine[1]] for b in bufs])
        blocks = []
        for p in range(world):
            rp = _rows_of(p, m, per)
            blocks.append((p * per + min(c0, rp), p * per + min(c1, rp)))
        works += _exchange([(b, blocks) for b in bufs], rank, world, group)
    for w in works:
        w.wait()


# ------------------------------------------------------------------ fused replication (NEXT-2)
class PeerBuffers:
    """A replicated-D buffer on every rank, mapped into every other rank's process through CUDA IPC
    (NVLink / NVSwitch peer memory across GPUs; plain IPC between processes sharing one GPU), plus
    the flag arrays of the device barrier.  Built once per (shape, dtype, group) and reused."""

    def __init__(self, rows, ld, dtype, device, group):
        from torch.multiprocessing.reductions import reduce_tensor

        self.world, self.rank = _world(group)
        self.group = group
        self.device = torch.device(device)
        self.local = torch.zeros((rows, ld), dtype=dtype, device=self.device)
        self.flags = torch.zeros((8,), dtype=torch.int32, device=self.device)
        torch.cuda.synchronize(self.device)
        uuid = str(torch.cuda.get_device_properties(self.device).uuid)
        mine = (reduce_tensor(self.local), reduce_tensor(self.flags), uuid)
        allh = [None] * self.world
        dist.all_gather_object(allh, mine, group=group)
        self._keep = []
        self.ptrs, self.flag_ptrs = [], []
        for p, (hl, hf, _) in enumerate(allh):
            if p == self.rank:
                t, f = self.local, self.flags
            else:
                t, f = hl[0](*hl[1]), hf[0](*hf[1])
                self._keep += [t, f]
            self.ptrs.append(t.data_ptr())
            self.flag_ptrs.append(f.data_ptr())
        uuids = [h[2] for h in allh]
        # ranks sharing one physical GPU (one-GPU multi-rank tests) cannot spin on each other in
        # kernels of different processes without time-slicing: they order through the host
        self.shared_gpu = len(set(uuids)) < len(uuids)
        self.epoch = 0
        dist.barrier(group=group)

    def barrier(self, stream, mode="auto"):
        if mode == "auto":
            mode = "host" if self.shared_gpu else "device"
        if mode == "host":
            stream.synchronize()
            dist.barrier(group=self.group)
            return
        import ctypes

        from . import _lib

        self.epoch += 1
        arr = (ctypes.c_void_p * self.world)(*self.flag_ptrs)
        _lib.check(_lib.load().cy_peer_barrier(arr, self.world, self.rank, self.epoch, stream.cuda_stream),
                   "cy_peer_barrier")


_PEER_CACHE = {}


def peer_buffers(rows, n, dtype, device, group) -> PeerBuffers:
    key = (rows, _ld8(n), dtype, str(device), id(group))
    if key not in _PEER_CACHE:
        _PEER_CACHE[key] = PeerBuffers(rows, _ld8(n), dtype, device, group)
    return _PEER_CACHE[key]


def _fused(A_local, B, C_local, alpha, beta, m, start, per, group, barrier):
    from . import gemm_replicated

    n = B.shape[1]
    world, _ = _world(group)
    pb = peer_buffers(per * world, n, A_local.dtype, A_local.device, group)
    stream = torch.cuda.current_stream(A_local.device)
    pb.barrier(stream, barrier)  # every peer is done reading the previous result (write-after-read)
    gemm_replicated(A_local, B, pb.ptrs, row_offset=start, rows_total=per * world, C=C_local, alpha=alpha,
                    beta=beta, ldd=pb.local.shape[1], stream=stream)
    pb.barrier(stream, barrier)  # every peer's tile stores have landed (read-after-write)
    return pb.local[:m, :n]


# ------------------------------------------------------------------ public entry points
def _default_gemm():
    from . import gemm

    return gemm


def sharded_gemm(A_local, B, C_local=None, alpha=1.0, beta=0.0, *, m_total=None, group=None,
                 replicate=False, align=256, gemm_fn=None, chunks=2, barrier="auto"):
    """Rank-local D = alpha*A_local@B + beta*C_local (A_local = this rank's row block).

    replicate=False:   returns the local D block (no communication).
    replicate=True:    returns the full (m_total x n) D on every rank (chunked, overlapped exchange).
    replicate="fused": the GEMM epilogue writes every tile straight into every rank's replicated D;
                       returns a view of a cached peer-mapped buffer (overwritten by the next call
                       with the same shape)."""
    world, rank = _world(group)
    rows, n = A_local.shape[0], B.shape[1]
    gemm_fn = gemm_fn or _default_gemm()
    if not replicate or world == 1:
        return gemm_fn(A_local, B, C_local, alpha, beta)
    m = m_total if m_total is not None else rows * world
    start, end, per = shard_rows(m, world, rank, align)
    if rows != end - start:
        raise ValueError(f"rank {rank} holds {rows} rows; the shard geometry gives {end - start}")
    if replicate == "fused":
        return _fused(A_local, B, C_local, alpha, beta, m, start, per, group, barrier)
    full = _gather_buffer(per * world, n, A_local.dtype, A_local.device)

    def compute(r0, r1, views):
        C = C_local[r0:r1] if (C_local is not None and beta != 0) else None
        gemm_fn(A_local[r0:r1], B, C, alpha, beta, out=views[0][:, :n])

    _row_sharded(rows, m, per, world, rank, group, [full], compute, chunks, align)
    return full[:m, :n]


def sharded_gemm_rowreduce(A_local, B, C_local=None, alpha=1.0, beta=0.0, *, m_total=None, group=None,
                           replicate=False, align=256, rowreduce_fn=None, chunks=2):
    """Rank-local (D, y) of the fused GEMM + row reduction; replicate=True exchanges both
    (BASELINE configs[4]: M-sharded over 8 GPUs + all-gather)."""
    if rowreduce_fn is None:
        from . import gemm_rowreduce as rowreduce_fn
    world, rank = _world(group)
    rows, n = A_local.shape[0], B.shape[1]
    if not replicate or world == 1:
        return rowreduce_fn(A_local, B, C_local, alpha, beta)
    m = m_total if m_total is not None else rows * world
    _, _, per = shard_rows(m, world, rank, align)
    Df = _gather_buffer(per * world, n, A_local.dtype, A_local.device)
    yf = torch.empty((per * world, 1), dtype=torch.float32, device=A_local.device)

    def compute(r0, r1, views):
        C = C_local[r0:r1] if (C_local is not None and beta != 0) else None
        rowreduce_fn(A_local[r0:r1], B, C, alpha, beta, out=views[0][:, :n], y=views[1][:, 0])

    _row_sharded(rows, m, per, world, rank, group, [Df, yf], compute, chunks, align)
    return Df[:m, :n], yf[:m, 0]


def sharded_gemm_batched(A_local, B_local, C_local=None, alpha=1.0, beta=0.0, *, L_total=None, group=None,
                         replicate=False, batched_fn=None):
    """Batch-index sharding: this rank holds batches [start, end) of A, B (and C)."""
    if batched_fn is None:
        from . import gemm_batched as batched_fn
    world, rank = _world(group)
    if not replicate or world == 1:
        return batched_fn(A_local, B_local, C_local, alpha, beta)
    Ll, m = A_local.shape[0], A_local.shape[1]
    n = B_local.shape[2]
    L = L_total if L_total is not None else Ll * world
    s, e, per = shard_batches(L, world, rank)
    if Ll != e - s:
        raise ValueError(f"rank {rank} holds {Ll} batches; the shard geometry gives {e - s}")
    full = torch.empty((per * world, m, _ld8(n)), dtype=A_local.dtype, device=A_local.device)
    if Ll:
        batched_fn(A_local, B_local, C_local, alpha, beta, out=full[rank * per:rank * per + Ll, :, :n])
    if _p2p_capable(full, group):
        blocks = [(p * per, p * per + max(0, min(L, (p + 1) * per) - p * per)) for p in range(world)]
        for w in _exchange([(full, blocks)], rank, world, group):
            w.wait()
    else:
        _gather_staged(full, per, world, group)
    return full[:L, :, :n]


def sharded_dual_gemm(A_local, B0, B1, alpha=1.0, mode="pair", *, m_total=None, group=None, replicate=False,
                      align=256, dual_fn=None, chunks=2):
    """Rank-local dual GEMM (pair: (D0, D1); sum: D); replicate=True exchanges the outputs."""
    if dual_fn is None:
        from . import dual_gemm

        def dual_fn(A, X, Y, a, out0=None, out1=None):
            return dual_gemm(A, X, Y, alpha=a, mode=mode, out0=out0, out1=out1)
    world, rank = _world(group)
    if not replicate or world == 1:
        return dual_fn(A_local, B0, B1, alpha)
    rows, n = A_local.shape[0], B0.shape[1]
    m = m_total if m_total is not None else rows * world
    _, _, per = shard_rows(m, world, rank, align)
    nout = 2 if mode == "pair" else 1
    bufs = [_gather_buffer(per * world, n, A_local.dtype, A_local.device) for _ in range(nout)]

    def compute(r0, r1, views):
        outs = [v[:, :n] for v in views]
        dual_fn(A_local[r0:r1], B0, B1, alpha, *outs)

    _row_sharded(rows, m, per, world, rank, group, bufs, compute, chunks, align)
    res = tuple(b[:m, :n] for b in bufs)
    return res if nout == 2 else res[0]
