"""Multi-rank parity tests of the CUDA path through paper_2504_07004_b200/dist.py (SURVEY 8(e), row
a10; NEXT-2): the real sm_100a kernels on every rank, compared bit for bit with the fp64 oracle on
integer-valued inputs (exactly one correct result, DESIGN R11).

* two gloo ranks sharing cuda:0 (runs on the one-GPU box): sharded_gemm / _rowreduce / _batched /
  _dual_gemm with replicate False, True (host-staged exchange) and "fused" (cy_gemm_replicated
  storing into both ranks' buffers through CUDA IPC; host-ordered barrier, the ranks share a GPU);
* the device barrier kernel cy_peer_barrier on one GPU, two streams playing two ranks;
* two NCCL ranks under torchrun on two GPUs (skipped with fewer): replicate True (chunked NCCL
  point-to-point overlapped with the compute) and "fused" with the device barrier;
* bench.py --gpus 2 re-launching itself (gloo, both ranks on cuda:0) prints n_gpus = 2.
"""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.timeout(900)]

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


# The worker body runs in a fresh interpreter per rank (spawned, or under torchrun).  It compares
# every sharded entry point with the oracle and prints one JSON line of failures.
WORKER = r'''
import json, os, sys, traceback
sys.path.insert(0, os.environ["CY_ROOT"]); sys.path.insert(0, os.path.join(os.environ["CY_ROOT"], "tests"))
import numpy as np, torch, torch.distributed as dist
import oracle, synth
from gpu_util import to_dev, to_bits
from paper_2504_07004_b200.dist import (shard_rows, shard_batches, sharded_gemm, sharded_gemm_rowreduce,
                                        sharded_gemm_batched, sharded_dual_gemm)
backend = os.environ["CY_BACKEND"]
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
dev = 0 if backend == "gloo" else int(os.environ.get("LOCAL_RANK", rank))
torch.cuda.set_device(dev)
if backend == "nccl":
    dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
else:
    dist.init_process_group("gloo")
fused_ok = backend == "nccl" or os.environ.get("CY_FUSED", "1") == "1"
bad = []
def check(name, got, want):
    if not np.array_equal(got, want):
        bad.append(name)
try:
    enc = lambda x: oracle.encode("f16", x)
    for (m, n, k) in [(1000, 264, 320), (600, 100, 96), (3, 72, 64), (2048, 512, 256)]:
        A, B, C = synth.gemm_inputs(m, n, k, seed=900 + m + n, kind="int", with_c=True)
        s, e, _ = shard_rows(m, world, rank)
        a, b, c = to_dev(np.ascontiguousarray(A[s:e]), "f16"), to_dev(B, "f16"), to_dev(np.ascontiguousarray(C[s:e]), "f16")
        want = enc(oracle.gemm("f16", A, B, C, 1.0, 2.0))
        want0 = enc(oracle.gemm("f16", A, B))
        for rep in (False, True, "fused"):
            if rep == "fused" and not fused_ok:
                continue
            for chunks in ((1, 2, 3) if rep is True else (2,)):
                D = sharded_gemm(a, b, c, 1.0, 2.0, m_total=m, replicate=rep, chunks=chunks)
                torch.cuda.synchronize()
                check(f"gemm{m}x{n}x{k} rep={rep} ch={chunks}", to_bits(D), want if rep else want[s:e])
        # the fused buffer is reused: a second call with other values must fully replace it
        if fused_ok:
            D = sharded_gemm(a, b, None, 1.0, 0.0, m_total=m, replicate="fused")
            torch.cuda.synchronize()
            check(f"gemm{m} fused again", to_bits(D), want0)
        for rep in (False, True):
            D, y = sharded_gemm_rowreduce(a, b, m_total=m, replicate=rep)
            torch.cuda.synchronize()
            check(f"rowreduce{m} rep={rep} D", to_bits(D), want0 if rep else want0[s:e])
            ys = oracle.rowsum("f16", A)
            check(f"rowreduce{m} rep={rep} y", y.cpu().numpy().astype(np.float64), ys if rep else ys[s:e])
        A3, B0, B1, _, _ = synth.dual_inputs(m, n, k, seed=950 + m, kind="int")
        r0, r1 = oracle.dual_gemm("f16", "pair", A3, B0, B1)
        rs = oracle.dual_gemm("f16", "sum", A3, B0, B1)
        a3 = to_dev(np.ascontiguousarray(A3[s:e]), "f16")
        for rep in (False, True):
            d0, d1 = sharded_dual_gemm(a3, to_dev(B0, "f16"), to_dev(B1, "f16"), m_total=m, replicate=rep)
            ds = sharded_dual_gemm(a3, to_dev(B0, "f16"), to_dev(B1, "f16"), mode="sum", m_total=m, replicate=rep)
            torch.cuda.synchronize()
            sl = slice(None) if rep else slice(s, e)
            check(f"dual{m} rep={rep} D0", to_bits(d0), enc(r0)[sl])
            check(f"dual{m} rep={rep} D1", to_bits(d1), enc(r1)[sl])
            check(f"dualsum{m} rep={rep}", to_bits(ds), enc(rs)[sl])
    for (L, m, n, k) in [(5, 128, 200, 64), (8, 256, 256, 256)]:
        A, B, _ = synth.gemm_inputs(m, n, k, seed=970 + L, batch=L, kind="int")
        s, e, _ = shard_batches(L, world, rank)
        want = enc(oracle.gemm_batched("f16", A, B))
        for rep in (False, True):
            D = sharded_gemm_batched(to_dev(np.ascontiguousarray(A[s:e]), "f16"), to_dev(np.ascontiguousarray(B[s:e]), "f16"),
                                     L_total=L, replicate=rep)
            torch.cuda.synchronize()
            check(f"batched{L} rep={rep}", to_bits(D), want if rep else want[s:e])
    out = {"rank": rank, "bad": bad}
except Exception:
    out = {"rank": rank, "error": traceback.format_exc()}
print("RESULT " + json.dumps(out), flush=True)
dist.barrier()
dist.destroy_process_group()
'''


def _run_ranks(world, backend, extra_env=None, timeout=600):
    port = _free_port()
    procs = []
    for r in range(world):
        env = dict(os.environ, CY_ROOT=ROOT, CY_BACKEND=backend, RANK=str(r), WORLD_SIZE=str(world),
                   LOCAL_RANK=str(r), MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), **(extra_env or {}))
        procs.append(subprocess.Popen([sys.executable, "-c", WORKER], env=env, cwd=ROOT, stdout=subprocess.PIPE,
                                      stderr=subprocess.PIPE, text=True))
    results = []
    for p in procs:
        out, err = p.communicate(timeout=timeout)
        lines = [ln[7:] for ln in out.splitlines() if ln.startswith("RESULT ")]
        assert p.returncode == 0 and lines, err[-3000:]
        results.append(json.loads(lines[-1]))
    for res in results:
        assert "error" not in res, res["error"]
        assert not res["bad"], (res["rank"], res["bad"])


def test_gloo_two_ranks_on_one_gpu_vs_oracle():
    """Two ranks on cuda:0 over gloo: every sharded entry point (replicate False / True / "fused")
    runs the real kernels and matches the oracle bit for bit on integer inputs, including uneven
    shards (m = 600, 1000, 3), n % 8 != 0 (n = 100: padded gather and peer buffers) and chunking."""
    _run_ranks(2, "gloo")


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs 2 GPUs (NCCL over NVLink)")
def test_nccl_two_gpus_vs_oracle():
    """Two ranks on two GPUs over NCCL: chunked point-to-point exchange and fused replication with
    the device barrier (peer memory over NVLink)."""
    _run_ranks(2, "nccl")


def test_peer_barrier_two_streams():
    """cy_peer_barrier protocol on one GPU: two streams play ranks 0 and 1 (one 32-thread CTA each,
    co-resident).  Each epoch, rank 0 writes a value and arrives; rank 1 arrives and then copies the
    value: after the barrier it must see this epoch's write (release/acquire at system scope)."""
    import ctypes

    from paper_2504_07004_b200 import _lib

    lib = _lib.load()
    flags = torch.zeros((2, 8), dtype=torch.int32, device="cuda")
    ptrs = (ctypes.c_void_p * 2)(flags[0].data_ptr(), flags[1].data_ptr())
    x = torch.zeros((1 << 20,), dtype=torch.float32, device="cuda")
    seen = torch.zeros((20,), dtype=torch.float32, device="cuda")
    s0, s1 = torch.cuda.Stream(), torch.cuda.Stream()
    torch.cuda.synchronize()
    for ep in range(1, 21):
        with torch.cuda.stream(s0):
            x.fill_(float(ep))
            assert lib.cy_peer_barrier(ptrs, 2, 0, ep, ctypes.c_void_p(s0.cuda_stream)) == 0
        with torch.cuda.stream(s1):
            assert lib.cy_peer_barrier(ptrs, 2, 1, ep, ctypes.c_void_p(s1.cuda_stream)) == 0
            seen[ep - 1].copy_(x[-1])
    torch.cuda.synchronize()
    assert seen.tolist() == [float(e) for e in range(1, 21)]
    assert flags[0, :2].tolist() == [20, 20] and flags[1, :2].tolist() == [20, 20]
    # argument checks
    assert lib.cy_peer_barrier(ptrs, 0, 0, 1, None) == 1
    assert lib.cy_peer_barrier(ptrs, 2, 2, 1, None) == 1
    assert lib.cy_peer_barrier(ptrs, 2, 0, 0, None) == 1
    bad = (ctypes.c_void_p * 2)(flags[0].data_ptr() + 2, flags[1].data_ptr())
    assert lib.cy_peer_barrier(bad, 2, 0, 1, None) == 2


def test_bench_gpus2_relaunches_itself():
    """bench.py --gpus 2 without torchrun re-launches itself with two ranks (here gloo, both on
    cuda:0) and rank 0 prints one line with n_gpus = 2."""
    env = dict(os.environ, BENCH_FORCE_DEVICE="0", BENCH_BACKEND="gloo")
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--workload", "sweep-2048", "--steps", "3",
                        "--warmup", "3", "--no-e2e"], cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [json.loads(ln) for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = lines[0]
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["gpu_launches"] == 3
    assert d["cpu_baseline"]["kind"] == "oracle"


def test_bench_allgather_workloads_two_ranks():
    """The replicated workloads run end to end with two ranks on cuda:0 (gloo: host-staged exchange;
    fused: CUDA-IPC peer stores) and report the exchange's NVLink bound."""
    env = dict(os.environ, BENCH_FORCE_DEVICE="0", BENCH_BACKEND="gloo")
    env.pop("WORLD_SIZE", None)
    for w in ("allgather", "allgather-fused"):
        r = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--workload", w, "--steps", "3", "--warmup",
                            "3", "--no-e2e", "--no-cpu-baseline"], cwd=ROOT, env=env, capture_output=True, text=True,
                           timeout=900)
        assert r.returncode == 0, r.stderr[-3000:]
        d = [json.loads(ln) for ln in r.stdout.splitlines() if ln.startswith("{")][0]
        assert d["n_gpus"] == 2 and d["exchange"]["nvlink_bound_ms"] > 0, d
