"""World-size-2 gloo tests (CPU) of the multi-GPU host logic in paper_2504_07004_b200/dist.py:
row / batch shard geometry, replicated all-gather assembly, uneven tails.  The per-rank compute is
injected as an oracle-backed CPU function (tests may call the oracle; the product path may not),
so these tests check the partitioning and the gather, not the kernels (those are the -m gpu tests)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2504_07004_b200.dist import (shard_batches, shard_rows, sharded_dual_gemm, sharded_gemm,
                                        sharded_gemm_batched, sharded_gemm_rowreduce)


@pytest.mark.parametrize("m", [1, 255, 256, 600, 8192, 65536, 70001])
@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_shard_rows_cover_disjoint(m, world):
    seen = np.zeros(m, dtype=int)
    for r in range(world):
        s, e, per = shard_rows(m, world, r)
        assert per % 256 == 0 and 0 <= s <= e <= m and e - s <= per
        assert s == min(m, r * per)
        seen[s:e] += 1
    assert (seen == 1).all()


def test_shard_batches():
    for L, w in [(64, 8), (64, 3), (5, 2), (1, 4)]:
        got = [shard_batches(L, w, r)[:2] for r in range(w)]
        covered = sorted(i for s, e in got for i in range(s, e))
        assert covered == list(range(L))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _bits_to_t(bits):
    return torch.from_numpy(np.ascontiguousarray(bits).view(np.int16)).view(torch.float16)


def _t_to_bits(t):
    return t.contiguous().view(torch.int16).numpy().view(np.uint16)


def _worker(rank, world, port, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import oracle
        import synth

        def gemm_fn(A, B, C, alpha, beta, out=None):
            D = _bits_to_t(oracle.encode("f16", oracle.gemm("f16", _t_to_bits(A), _t_to_bits(B),
                                                                None if C is None else _t_to_bits(C), alpha, beta)))
            if out is not None:
                out.copy_(D)
                return out
            return D

        def rowreduce_fn(A, B, C, alpha, beta, out=None, y=None):
            D = gemm_fn(A, B, C, alpha, beta, out)
            yy = torch.from_numpy(oracle.rowsum("f16", _t_to_bits(A)).astype(np.float32))
            if y is not None:
                y.copy_(yy)
                return D, y
            return D, yy

        results = {}
        for m in (512, 600, 3):
            n, k = 64, 96
            A, B, C = synth.gemm_inputs(m, n, k, seed=500 + m, kind="int", with_c=True)
            s, e, _ = shard_rows(m, world, rank)
            D = sharded_gemm(_bits_to_t(A[s:e]), _bits_to_t(B), _bits_to_t(C[s:e]), 1.0, 2.0, m_total=m,
                             replicate=True, gemm_fn=gemm_fn)
            want = oracle.encode("f16", oracle.gemm("f16", A, B, C, 1.0, 2.0))
            results[f"gemm{m}"] = bool(np.array_equal(_t_to_bits(D), want))
            D2, y = sharded_gemm_rowreduce(_bits_to_t(A[s:e]), _bits_to_t(B), m_total=m, replicate=True,
                                           rowreduce_fn=rowreduce_fn)
            results[f"rr{m}"] = bool(np.array_equal(_t_to_bits(D2), oracle.encode("f16", oracle.gemm("f16", A, B)))
                                     and np.array_equal(y.numpy().astype(np.float64), oracle.rowsum("f16", A)))
            # local (non-replicated) result is exactly this rank's rows
            Dl = sharded_gemm(_bits_to_t(A[s:e]), _bits_to_t(B), None, 1.0, 0.0, m_total=m, gemm_fn=gemm_fn)
            results[f"local{m}"] = bool(np.array_equal(_t_to_bits(Dl), oracle.encode("f16", oracle.gemm("f16", A, B))[s:e]))
        # batched: batch-index shards
        L, m, n, k = 5, 16, 24, 32
        A, B, _ = synth.gemm_inputs(m, n, k, seed=77, batch=L, kind="int")
        s, e, _ = shard_batches(L, world, rank)

        def batched_fn(A_, B_, C_, alpha, beta, out=None):
            D = _bits_to_t(oracle.encode("f16", oracle.gemm_batched("f16", _t_to_bits(A_), _t_to_bits(B_))))
            if out is not None:
                out.copy_(D)
                return out
            return D

        Db = sharded_gemm_batched(_bits_to_t(A[s:e]), _bits_to_t(B[s:e]), L_total=L, replicate=True,
                                  batched_fn=batched_fn)
        results["batched"] = bool(np.array_equal(_t_to_bits(Db), oracle.encode("f16", oracle.gemm_batched("f16", A, B))))
        # dual pair
        A, B0, B1, _, _ = synth.dual_inputs(300, 40, 64, seed=88, kind="int")
        s, e, _ = shard_rows(300, world, rank)

        def dual_fn(A_, X, Y, a, out0=None, out1=None):
            r0, r1 = oracle.dual_gemm("f16", "pair", _t_to_bits(A_), _t_to_bits(X), _t_to_bits(Y), alpha=a)
            d0, d1 = _bits_to_t(oracle.encode("f16", r0)), _bits_to_t(oracle.encode("f16", r1))
            if out0 is not None:
                out0.copy_(d0)
                out1.copy_(d1)
                return out0, out1
            return d0, d1

        d0, d1 = sharded_dual_gemm(_bits_to_t(A[s:e]), _bits_to_t(B0), _bits_to_t(B1), m_total=300, replicate=True,
                                   dual_fn=dual_fn)
        r0, r1 = oracle.dual_gemm("f16", "pair", A, B0, B1)
        results["dual"] = bool(np.array_equal(_t_to_bits(d0), oracle.encode("f16", r0))
                               and np.array_equal(_t_to_bits(d1), oracle.encode("f16", r1)))
        q.put((rank, results))
        dist.destroy_process_group()
    except Exception as ex:  # pragma: no cover
        import traceback

        q.put((rank, {"error": traceback.format_exc()}))


@pytest.mark.timeout(300)
def test_gloo_world2_replicated_gather():
    import oracle

    oracle.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    for r in range(2):
        assert "error" not in out[r], out[r].get("error")
        bad = [k for k, v in out[r].items() if not v]
        assert not bad, (r, bad)
