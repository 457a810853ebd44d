"""bench.py -- headline benchmark of the B200 Cypress GEMM family.

Default workload (BASELINE.json metric, configs[1] at its 8192^3 point, M-sharded to P GPUs
as in configs[4]): every rank computes an 8192 x 8192 x 8192 fp16 GEMM (its M-row shard of a
(8192*P) x 8192 x 8192 problem, B replicated) through the C ABI.  A step = one cy_gemm call
(host entry -> TMA descriptors -> one persistent tcgen05 kernel), i.e. every row a1-a6 of
SURVEY.md section 8(a).  No collective is on the data path (weak scaling).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload NAME] [--impl reference]

--gpus N > 1 without torchrun: the script re-launches itself under torch.distributed.run with N
processes (one per GPU, NCCL); under torchrun it checks that WORLD_SIZE == N.

Other workloads (--workload): sweep-<n> (n^3), batched (64 x 1024^3, batch-sharded; beta = 0),
batched-beta1 (the same with D = A*B + C: the HBM-bound case of SURVEY 8(d)), dual (dual-GEMM
pair 8192^3), glu (silu(A*B0)*(A*B1) 8192^3), rowreduce (65536/P x 8192 x 8192 + y), allgather
(rowreduce + chunked point-to-point exchange of D and y overlapped with the compute: replicated
result), allgather-fused (GEMM whose epilogue stores every tile into every rank's D over peer
mappings, device barriers around it), attention (FA forward fp16, HeadDim 128, 2 x 16 heads x
8192, non-causal; batch-sharded).

Prints ONE JSON line on rank 0.  Timing: CUDA events on the launching stream, W warm-up
steps, barrier + synchronize on both sides of exactly K timed steps, max over ranks.
L2: the JSON "l2" key states, per workload, how many input sets rotate and their total bytes
(> 126 MB L2 except where it says "L2-resident").
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "fp16 GEMM TFLOP/s per B200 and % of dense tensor peak; 8-GPU aggregate"
ATTN_METRIC = "fp16 flash-attention forward TFLOP/s (HeadDim 128, 4*b*h*s^2*d FLOP)"


def step_stats(per):
    """Mean / p10 / median / p90 of the per-step device times (ms); with a single region
    event pair (short steps) only the mean exists."""
    out = {"mean": round(statistics.mean(per), 5), "n": len(per)}
    if len(per) >= 10:
        q = statistics.quantiles(per, n=10)
        out.update(p10=round(q[0], 5), median=round(statistics.median(per), 5), p90=round(q[-1], 5))
    return out


def scaling_of(workload):
    """'weak' when every rank's work is fixed as N grows (gemm: 8192 rows per GPU; sweep-n: n rows per
    GPU; attention: batch 2 per GPU), 'strong' when the total problem is fixed and split over the
    ranks (batched 64 x 1024^3, rowreduce/allgather 65536 rows, dual/glu 8192^3)."""
    return "strong" if workload in ("batched", "batched-beta1", "rowreduce", "allgather", "allgather-fused", "dual",
                                    "glu") else "weak"


def metric_for(workload):
    return ATTN_METRIC if workload == "attention" else METRIC


# ----------------------------------------------------------------------------- helpers
def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return {"burst": d.get("bf16_tflops", 1590.0), "sustained": d.get("bf16_tflops_sustained", 1400.0),
                "source": "measured (MEASURED_PEAKS.json, cuBLAS bf16; fp16 dense peak = bf16 dense peak)"}
    return {"burst": 1590.0, "sustained": 1400.0,
            "source": "fallback (B200_PROFILING.md: 1.59 PF burst / ~1.4 PF sustained)"}


def load_traffic(workload):
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d.get(workload)
    return None


class ClockSampler:
    """NVML sampling of SM clock / power / clock-event reasons during the timed region."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
        0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
        0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, dev_index, period=0.005):
        self.samples = []
        self.reasons = set()
        self.max_mhz = None
        self._stop = threading.Event()
        self.ok = False
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(dev_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            pass
        self.period = period

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                mhz = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h) if hasattr(
                    nv, "nvmlDeviceGetCurrentClocksEventReasons") else nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
                pw = nv.nvmlDeviceGetPowerUsage(self.h) / 1000.0
                self.samples.append((mhz, r, pw))
                for bit, name in self.REASONS.items():
                    if r & bit and bit != 0x1:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["nvml_unavailable"]}
        mhz = [s[0] for s in self.samples]
        return {"sm_mhz": statistics.median(mhz), "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(mhz), "power_w_max": round(max(s[2] for s in self.samples), 1),
                "sm_mhz_min": min(mhz)}

    def rejected(self):
        bad = {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"}
        s = self.summary()
        if self.reasons & bad:
            return True
        if s["sm_mhz"] and self.max_mhz and s["sm_mhz"] < 0.5 * self.max_mhz and not self.reasons:
            return True
        return False


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


# ----------------------------------------------------------------------------- workloads
def make_workload(name, rank, world, device):
    """Returns dict with: flops_per_step (this rank), step(i) callable, e2e_step(i) callable,
    h2d/d2h bytes, oracle sampler, description."""
    import numpy as np
    import torch

    import paper_2504_07004_b200 as cy
    import synth
    from paper_2504_07004_b200.dist import sharded_gemm, sharded_gemm_rowreduce
    from paper_2504_07004_b200.stream import HostGemmPipeline, HostPipeline

    f16 = torch.float16

    def up(bits):
        return torch.from_numpy(np.ascontiguousarray(bits).view(np.int16)).view(torch.float16).to(device)

    def pinned(bits):
        t = torch.from_numpy(np.ascontiguousarray(bits).view(np.int16)).view(torch.float16)
        return t.pin_memory()

    W = {}

    def l2_label(nsets, set_bytes):
        tot = nsets * set_bytes
        return (f"{nsets} input set(s) rotating, {tot / 1e6:.0f} MB of operands "
                + ("(> 126 MB L2: not L2-resident)" if tot > 126e6 else "(L2-resident)"))

    if name in ("gemm", "rowreduce", "allgather", "allgather-fused") or name.startswith("sweep-"):
        if name.startswith("sweep-"):
            n = int(name.split("-")[1])
            m_rank, k = n, n
            desc = f"fp16 GEMM {n}^3 (configs[1] sweep point), 1 GPU" if world == 1 else \
                f"fp16 GEMM ({n}*P) x {n} x {n}, M-sharded over P={world}"
        elif name == "gemm":
            n = k = 8192
            m_rank = 8192
            desc = ("fp16 GEMM 8192^3 (configs[1] 8192 point)" if world == 1 else
                    f"fp16 GEMM {8192 * world} x 8192 x 8192 M-sharded over {world} GPUs (configs[4] shape, no reduction)")
        elif name == "allgather-fused":
            n = k = 8192
            m_rank = 65536 // world
            desc = (f"fp16 GEMM 65536 x 8192 x 8192 M-sharded over {world} GPU(s), replicated D by fused replication "
                     "(epilogue stores every tile into every rank's D over peer mappings; SURVEY NEXT-2)")
        else:
            n = k = 8192
            m_rank = 65536 // world
            desc = (f"fp16 GEMM 65536 x 8192 x 8192 + fused row reduction y(i)=sum_k A(i,k) (configs[4]), "
                    f"M-sharded over {world} GPU(s)" + (", D and y exchanged (chunked NCCL point-to-point overlapped "
                                                        "with the compute; replicated result)" if name == "allgather" else ""))
        sets = []
        host_sets = []
        set_bytes = m_rank * k * 2 + k * n * 2
        # enough rotating sets that the operands exceed 2x the 126 MB L2 (one set when a set is > 400 MB)
        nsets = 1 if set_bytes >= 400e6 else min(64, max(2, -(-int(300e6) // set_bytes)))
        W["l2"] = l2_label(nsets, set_bytes)
        for s in range(nsets):
            A = synth.uniform((m_rank, k), synth.seed_for(4 if name in ("rowreduce", "allgather") else 1, 10 * rank + s))
            B = synth.uniform((k, n), synth.seed_for(1, 1000 + s))  # replicated across ranks
            if s < 2:
                host_sets.append((A, B))
            sets.append((up(A), up(B)))
        D = torch.empty((m_rank, n), dtype=torch.float16, device=device)
        y = torch.empty((m_rank,), dtype=torch.float32, device=device)
        flops = 2.0 * m_rank * n * k
        if name == "gemm" or name.startswith("sweep-"):
            def step(i):
                a, b = sets[i % nsets]
                cy.gemm(a, b, out=D)
        elif name == "rowreduce":
            def step(i):
                a, b = sets[i % nsets]
                cy.gemm_rowreduce(a, b, out=D, y=y)
        elif name == "allgather-fused":
            def step(i):
                a, b = sets[i % nsets]
                sharded_gemm(a, b, m_total=m_rank * world, replicate="fused")
        else:
            def step(i):
                a, b = sets[i % nsets]
                sharded_gemm_rowreduce(a, b, m_total=m_rank * world, replicate=True)
        if name in ("allgather", "allgather-fused"):
            # the exchange's physical bound: every rank receives (P-1)/P of D (and y)
            # over NVLink; measured peer copy 770 GB/s per direction (B200_PROFILING.md)
            recv = (world - 1) / world * (65536 * n * 2 + (65536 * 4 if name == "allgather" else 0))
            W["exchange"] = {"recv_bytes_per_rank": int(recv), "nvlink_gbs": 770.0,
                             "nvlink_bound_ms": round(recv / 770e9 * 1e3, 4),
                             "compute_ms_at_peak": None}
        hA = [pinned(h[0]) for h in host_sets]
        hB = [pinned(h[1]) for h in host_sets]
        hD = torch.empty((m_rank, n), dtype=torch.float16).pin_memory()
        pipe = None
        if name == "gemm" or name.startswith("sweep-"):
            pipe = HostGemmPipeline(m_rank, n, k, device=device)
        elif name == "rowreduce":
            pipe = HostPipeline([((m_rank, k), f16), ((k, n), f16)], [((m_rank, n), f16), ((m_rank,), torch.float32)],
                                lambda i, o, st: cy.gemm_rowreduce(i[0], i[1], out=o[0], y=o[1], stream=st),
                                device=device)
            hy = torch.empty((m_rank,), dtype=torch.float32).pin_memory()

        def e2e_step(i):
            j = i % len(hA)  # (the host keeps the first two input sets)
            if pipe is not None and name == "rowreduce":
                pipe.submit((hA[j], hB[j]), (hD, hy))
                return
            if pipe is not None:  # public host-streaming API: H2D / kernel / D2H overlapped
                pipe.submit(hA[j], hB[j], hD)
                return
            a = hA[j].to(device, non_blocking=True)
            b = hB[j].to(device, non_blocking=True)
            if name == "allgather":  # the same replicated call, full D and y back to the host
                Df, yf = sharded_gemm_rowreduce(a, b, m_total=m_rank * world, replicate=True)
                hDf.copy_(Df, non_blocking=True)
                hyf.copy_(yf, non_blocking=True)
            elif name == "allgather-fused":
                hDf.copy_(sharded_gemm(a, b, m_total=m_rank * world, replicate="fused"), non_blocking=True)
            else:
                cy.gemm(a, b, out=D)
                hD.copy_(D, non_blocking=True)
        d2h = hD.numel() * 2 + (4 * m_rank if name == "rowreduce" else 0)
        if name in ("allgather", "allgather-fused"):
            hDf = torch.empty((m_rank * world, n), dtype=torch.float16).pin_memory()
            hyf = torch.empty((m_rank * world,), dtype=torch.float32).pin_memory()
            d2h = hDf.numel() * 2 + (hyf.numel() * 4 if name == "allgather" else 0)
        W["pipe"] = pipe

        W.update(flops=flops, step=step, e2e_step=e2e_step, desc=desc,
                 h2d=hA[0].numel() * 2 + hB[0].numel() * 2, d2h=d2h,
                 shape={"m": m_rank * world, "n": n, "k": k, "m_per_gpu": m_rank},
                 oracle_case=(("rowreduce" if name in ("rowreduce", "allgather") else "gemm"), host_sets[0]),
                 kernel_flops=flops)
    elif name in ("batched", "batched-beta1"):
        L_total, m = 64, 1024
        L = L_total // world
        beta = 1.0 if name == "batched-beta1" else 0.0
        A = synth.uniform((L, m, m), synth.seed_for(2, 10 * rank))
        B = synth.uniform((L, m, m), synth.seed_for(2, 10 * rank + 1))
        A2 = synth.uniform((L, m, m), synth.seed_for(2, 10 * rank + 2))
        B2 = synth.uniform((L, m, m), synth.seed_for(2, 10 * rank + 3))
        sets = [(up(A), up(B)), (up(A2), up(B2))]
        Cs = [None, None]
        if beta != 0:
            Cs = [up(synth.uniform((L, m, m), synth.seed_for(2, 10 * rank + 4 + j))) for j in range(2)]
        D = torch.empty((L, m, m), dtype=torch.float16, device=device)
        W["l2"] = l2_label(2, (2 + (beta != 0)) * L * m * m * 2)

        def step(i):
            a, b = sets[i % 2]
            cy.gemm_batched(a, b, Cs[i % 2], 1.0, beta, out=D)
        hA, hB = pinned(A), pinned(B)
        hD = torch.empty((L, m, m), dtype=torch.float16).pin_memory()

        pipe = HostPipeline([((L, m, m), f16), ((L, m, m), f16)], [((L, m, m), f16)],
                            lambda i, o, st: cy.gemm_batched(i[0], i[1], out=o[0], stream=st), device=device)

        def e2e_step(i):
            pipe.submit((hA, hB), (hD,))
        W["pipe"] = pipe
        W.update(flops=2.0 * L * m ** 3, step=step, e2e_step=e2e_step,
                 desc=f"batched fp16 GEMM 64 x 1024^3 (configs[2]), batch-sharded over {world} GPU(s)"
                      + (", D = A*B + C (beta = 1)" if beta != 0 else ""),
                 h2d=2 * hA.numel() * 2, d2h=hD.numel() * 2, shape={"batch": L_total, "m": m, "n": m, "k": m},
                 oracle_case=("batched", (A, B)), kernel_flops=2.0 * L * m ** 3)
    elif name == "glu":
        n = 8192
        m_rank = n // world if world > 1 else n
        A = synth.uniform((m_rank, n), synth.seed_for(3, 10 * rank))
        B0 = synth.uniform((n, n), synth.seed_for(3, 1001))
        B1 = synth.uniform((n, n), synth.seed_for(3, 1002))
        dA, dB0, dB1 = up(A), up(B0), up(B1)
        D0 = torch.empty((m_rank, n), dtype=torch.float16, device=device)
        W["l2"] = l2_label(1, (m_rank * n + 2 * n * n) * 2)

        def step(i):
            cy.dual_gemm_glu(dA, dB0, dB1, act="silu", out=D0)
        hA, hB0, hB1 = pinned(A), pinned(B0), pinned(B1)
        hD0 = torch.empty((m_rank, n), dtype=torch.float16).pin_memory()

        pipe = HostPipeline([((m_rank, n), f16), ((n, n), f16), ((n, n), f16)], [((m_rank, n), f16)],
                            lambda i, o, st: cy.dual_gemm_glu(i[0], i[1], i[2], act="silu", out=o[0], stream=st),
                            device=device)

        def e2e_step(i):
            pipe.submit((hA, hB0, hB1), (hD0,))
        W["pipe"] = pipe
        W.update(flops=4.0 * m_rank * n * n, step=step, e2e_step=e2e_step,
                 desc="GLU dual-GEMM D = silu(A*B0) * (A*B1), 8192^3 (SURVEY NEXT-3, P:1532)",
                 h2d=(hA.numel() + hB0.numel() + hB1.numel()) * 2, d2h=hD0.numel() * 2,
                 shape={"m": m_rank * world, "n": n, "k": n}, oracle_case=("glu", (A, B0, B1)),
                 kernel_flops=4.0 * m_rank * n * n)
    elif name == "dual":
        n = 8192
        m_rank = n // world if world > 1 else n
        A = synth.uniform((m_rank, n), synth.seed_for(3, 10 * rank))
        B0 = synth.uniform((n, n), synth.seed_for(3, 1001))
        B1 = synth.uniform((n, n), synth.seed_for(3, 1002))
        dA, dB0, dB1 = up(A), up(B0), up(B1)
        D0 = torch.empty((m_rank, n), dtype=torch.float16, device=device)
        D1 = torch.empty_like(D0)
        W["l2"] = l2_label(1, (m_rank * n + 2 * n * n) * 2)

        def step(i):
            cy.dual_gemm(dA, dB0, dB1, mode="pair", out0=D0, out1=D1)
        hA, hB0, hB1 = pinned(A), pinned(B0), pinned(B1)
        hD0 = torch.empty((m_rank, n), dtype=torch.float16).pin_memory()
        hD1 = torch.empty_like(hD0).pin_memory()

        pipe = HostPipeline([((m_rank, n), f16), ((n, n), f16), ((n, n), f16)], [((m_rank, n), f16)] * 2,
                            lambda i, o, st: cy.dual_gemm(i[0], i[1], i[2], mode="pair", out0=o[0], out1=o[1],
                                                          stream=st), device=device)

        def e2e_step(i):
            pipe.submit((hA, hB0, hB1), (hD0, hD1))
        W["pipe"] = pipe
        W.update(flops=4.0 * m_rank * n * n, step=step, e2e_step=e2e_step,
                 desc=f"dual-GEMM D=(A*B0, A*B1), 8192^3 (configs[3])" + (f", M-sharded over {world}" if world > 1 else ""),
                 h2d=(hA.numel() + hB0.numel() + hB1.numel()) * 2, d2h=2 * hD0.numel() * 2,
                 shape={"m": m_rank * world, "n": n, "k": n}, oracle_case=("dual", (A, B0, B1)),
                 kernel_flops=4.0 * m_rank * n * n)
    elif name == "attention":
        # FA forward, FP16, HeadDim 128, non-causal; 16 heads x 8192 tokens x batch 2
        # (16K tokens per GPU; reading R16), batch-sharded: each rank runs its own batch slice.
        b, h, s_len, d = 2, 16, 8192, 128
        sets, host = [], []
        for s_i in range(2):
            Q, K, V = (synth.uniform((b * h, s_len, d), synth.seed_for(6, 10 * rank + 3 * s_i + t)) for t in range(3))
            host.append((Q, K, V))
            sets.append(tuple(up(x).view(b, h, s_len, d) for x in (Q, K, V)))
        O = torch.empty((b, h, s_len, d), dtype=torch.float16, device=device)
        lse = torch.empty((b, h, s_len), dtype=torch.float32, device=device)
        W["l2"] = l2_label(2, 3 * b * h * s_len * d * 2)

        def step(i):
            q, k, v = sets[i % 2]
            cy.attention(q, k, v, out=O, lse=lse)
        hQ, hK, hV = (pinned(x).view(b, h, s_len, d) for x in host[0])
        hO = torch.empty((b, h, s_len, d), dtype=torch.float16).pin_memory()

        qkv = ((b, h, s_len, d), f16)
        pipe = HostPipeline([qkv] * 3, [qkv], lambda i, o, st: cy.attention(i[0], i[1], i[2], out=o[0], lse=lse,
                                                                          stream=st), device=device)

        def e2e_step(i):
            pipe.submit((hQ, hK, hV), (hO,))
        W["pipe"] = pipe
        fl = 4.0 * b * h * s_len * s_len * d
        W.update(flops=fl, step=step, e2e_step=e2e_step,
                 desc=f"FA forward fp16 HeadDim 128, non-causal, batch {b} x 16 heads x 8192 (P:1594-1636, SURVEY NEXT-4)"
                      + (f", batch-sharded over {world}" if world > 1 else ""),
                 h2d=3 * hQ.numel() * 2, d2h=hO.numel() * 2,
                 shape={"batch": b * world, "heads": h, "seq": s_len, "head_dim": d, "causal": False},
                 oracle_case=("attention", host[0][:3] + (b * h,)), kernel_flops=fl)
    else:
        raise SystemExit(f"unknown workload {name}")
    return W


def oracle_unit_fn(kind, arrs):
    """The fp64 C oracle, as it stands, on a subset of the workload's output units: returns
    (fn(units), FLOP per unit, number of units, unit name).  A unit is one output row (all columns,
    full K) or, for the batched workload, one whole 1024^3 GEMM of the batch."""
    import oracle

    if kind == "batched":
        A, B = arrs

        def fn(units):
            for r in units:
                oracle.gemm("f16", A[r], B[r])
        return fn, 2.0 * A.shape[1] * A.shape[2] * B.shape[2], A.shape[0], "whole 1024^3 GEMMs of the batch"
    if kind == "dual":
        A, B0, B1 = arrs
        return (lambda rows: oracle.dual_gemm("f16", "pair", A, B0, B1, rows=rows), 4.0 * B0.shape[1] * A.shape[1],
                A.shape[0], "rows (all columns, full K) of both products")
    if kind == "glu":
        A, B0, B1 = arrs
        return (lambda rows: oracle.dual_glu("f16", "silu", A, B0, B1, rows=rows), 4.0 * B0.shape[1] * A.shape[1],
                A.shape[0], "rows (all columns, full K)")
    if kind == "rowreduce":
        A, B = arrs

        def fn(rows):
            oracle.gemm("f16", A, B, rows=rows % A.shape[0])
            oracle.rowsum("f16", A, rows=rows % A.shape[0])
        return fn, 2.0 * B.shape[1] * A.shape[1] + A.shape[1], 65536, "rows (all columns, full K) + row sums"
    A, B = arrs
    return (lambda rows: oracle.gemm("f16", A, B, rows=rows), 2.0 * B.shape[1] * A.shape[1], A.shape[0],
            "rows (all columns, full K)")


def oracle_calibrate(fn, m, nth):
    """t(units) = fixed (operand decode) + units * per_unit, from two probes; the second probe grows
    until its extra time stands clear of the run-to-run noise of the fixed part."""
    import numpy as np

    p1 = max(1, min(m // 2, max(2 * nth, 8)))
    t0 = time.perf_counter()
    fn(np.arange(p1))
    t1 = time.perf_counter() - t0
    p2 = min(m, 2 * p1)
    while True:
        t0 = time.perf_counter()
        fn(np.arange(p2))
        t2 = time.perf_counter() - t0
        if t2 - t1 >= max(0.3, 0.2 * t1) or p2 >= m or t2 > 20.0:
            break
        p2 = min(m, 2 * p2)
    per = max((t2 - t1) / max(1, p2 - p1), 1e-6)
    return max(t1 - per * p1, 0.0), per, p1


def oracle_baseline(case, budget_s=12.0):
    """Time the fp64 C oracle, as it stands, on a bounded sample of the same workload (one call
    sized to ~budget_s of CPU work: >= 512 rows)."""
    import numpy as np

    import oracle

    kind, arrs = case
    oracle.set_threads(len(os.sched_getaffinity(0)))
    nth = oracle.num_threads()
    if kind == "attention":
        return attention_sample(*arrs, budget_s=budget_s)
    fn, per_unit, m, unit = oracle_unit_fn(kind, arrs)
    fixed, per, p1 = oracle_calibrate(fn, m, nth)
    floor = 1 if kind == "batched" else min(m, 512)
    nunits = int(min(m, max(floor, p1, (budget_s - fixed) / per)))
    units = np.linspace(0, m - 1, nunits).astype(np.int64)
    t0 = time.perf_counter()
    fn(units)
    dt = time.perf_counter() - t0
    return {"value": per_unit * nunits / dt / 1e12, "unit": "TFLOP/s", "cores": nth, "kind": "oracle",
            "sample": f"{nunits} of {m} {unit} of the same inputs, fp64 C oracle, {dt:.1f} s"}


def attention_sample(Q, K, V, bh, budget_s=12.0, rng=None):
    """Time the fp64 oracle's attention, as it stands, on query rows sampled from one head.
    Each sampled row costs 4*sk*d FLOP (scores + P.V), the same work per row as the kernel."""
    import numpy as np

    import oracle

    oracle.set_threads(len(os.sched_getaffinity(0)))
    nth = oracle.num_threads()
    sq, d = Q.shape[1], Q.shape[2]
    sk = K.shape[1]
    per_row = 4.0 * sk * d
    rng = rng or np.random.default_rng(0)

    def run(nrows):
        hsel = int(rng.integers(0, bh))
        rows = np.sort(rng.choice(sq, nrows, replace=False))
        t0 = time.perf_counter()
        oracle.attention("f16", np.ascontiguousarray(Q[hsel:hsel + 1, rows]), K[hsel:hsel + 1], V[hsel:hsel + 1])
        return time.perf_counter() - t0

    probe = max(2 * nth, 8)
    dt0 = run(probe)
    nrows = int(min(sq, max(probe, probe * budget_s / max(dt0, 1e-3))))
    dt = run(nrows)
    return {"value": per_row * nrows / dt / 1e12, "unit": "TFLOP/s", "cores": nth, "kind": "oracle",
            "sample": f"{nrows} random query rows of one head (all {sk} keys, HeadDim {d}), fp64 C oracle, {dt:.1f} s"}


# ----------------------------------------------------------------------------- main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--workload", default="gemm")
    ap.add_argument("--impl", default="cypress_b200", choices=["cypress_b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--config", type=int, default=-1, help="force a GEMM config id (tuning; default: heuristic)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--graph", action="store_true",
                    help="capture the K timed steps in a CUDA graph and time its replay (no host launch gaps)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-launch under torchrun (the driver's launch form)
        import socket

        with socket.socket() as so:
            so.bind(("127.0.0.1", 0))
            port = so.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
        os.execv(sys.executable, cmd)
    rank, world, local = dist_env()
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; launch one process per GPU")

    if args.impl == "reference":
        return reference_arm(args, rank, world)

    import torch

    # BENCH_FORCE_DEVICE / BENCH_BACKEND: test-only overrides that run several ranks on one GPU
    # (gloo) to exercise the multi-rank code path; production runs use one GPU per rank + NCCL.
    if "BENCH_FORCE_DEVICE" in os.environ:
        local = int(os.environ["BENCH_FORCE_DEVICE"])
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist

        backend = os.environ.get("BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=device)
        else:
            dist.init_process_group(backend)
    import paper_2504_07004_b200 as cy

    if args.config >= 0:
        cy.force_config(args.config)
    W = make_workload(args.workload, rank, world, device)
    stream = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            import torch.distributed as dist

            dist.barrier()
        torch.cuda.synchronize()

    def maxred(x):
        if world == 1:
            return x
        import torch.distributed as dist

        on_dev = dist.get_backend() == "nccl"
        t = torch.tensor([x], dtype=torch.float64, device=device if on_dev else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def timed(fn, steps, warmup, sample_clocks=True, pipe=None, use_graph=False):
        for i in range(warmup):
            fn(i)
        if pipe is not None:
            pipe.synchronize()
        barrier()
        # per-step events only when steps are long enough that recording them costs nothing
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        fn(warmup)
        if pipe is not None:
            pipe.join(stream)
        e1.record(stream)
        torch.cuda.synchronize()
        per_step = e0.elapsed_time(e1) > 0.2 and pipe is None and not use_graph
        starts = [torch.cuda.Event(enable_timing=True) for _ in range(steps if per_step else 1)]
        ends = [torch.cuda.Event(enable_timing=True) for _ in range(steps if per_step else 1)]
        n0 = cy.launch_count()
        graph = None
        if use_graph and pipe is None:
            graph = torch.cuda.CUDAGraph()
            side = torch.cuda.Stream()
            side.wait_stream(stream)
            with torch.cuda.stream(side):
                with torch.cuda.graph(graph, stream=side):
                    for i in range(steps):
                        fn(warmup + 1 + i)
            stream.wait_stream(side)
            torch.cuda.synchronize()
        sampler = ClockSampler(local)
        with sampler:
            barrier()
            if graph and pipe is None:
                # CUDA graph of the K steps (captured above): replay = device-bound step rate
                starts[0].record(stream)
                graph.replay()
                ends[0].record(stream)
            elif per_step:
                for i in range(steps):
                    starts[i].record(stream)
                    fn(warmup + 1 + i)
                    ends[i].record(stream)
            else:
                starts[0].record(stream)
                if pipe is not None:
                    pipe.wait_for(stream)
                for i in range(steps):
                    fn(warmup + 1 + i)
                if pipe is not None:
                    pipe.join(stream)
                ends[0].record(stream)
            barrier()
        launches = cy.launch_count() - n0
        total_ms = starts[0].elapsed_time(ends[-1])
        per = [s.elapsed_time(e) for s, e in zip(starts, ends)] if per_step else [total_ms / steps]
        return total_ms, per, launches, sampler

    attempts = 0
    while True:
        attempts += 1
        total_ms, per, launches, sampler = timed(W["step"], args.steps, args.warmup, use_graph=args.graph)
        if not sampler.rejected() or attempts >= 2:
            break
    total_ms = maxred(total_ms)
    kern_ms = maxred(statistics.mean(per))
    ms_per_step = total_ms / args.steps
    value = W["flops"] * world / (ms_per_step * 1e-3) / 1e12
    peaks = load_peaks()
    achieved = W["kernel_flops"] / (kern_ms * 1e-3) / 1e12
    # The roofline denominator follows what the clocks did during the timed region: the sustained
    # (power-capped) cuBLAS figure when sw_power_cap was active AND pulled the median SM clock below
    # 90 % of its maximum (the sustained figure was measured at ~1.35 GHz), the burst figure
    # otherwise (a short region can see the cap flag while still running near full clock).
    cs = sampler.summary()
    power_capped = ("sw_power_cap" in sampler.reasons and cs.get("sm_mhz") is not None
                    and cs.get("sm_max_mhz") and cs["sm_mhz"] < 0.9 * cs["sm_max_mhz"])
    peak = peaks["sustained"] if power_capped else peaks["burst"]

    e2e = None
    if not args.no_e2e:
        e_steps = max(3, min(args.steps, 20))
        e_total, _, _, _ = timed(W["e2e_step"], e_steps, 3, pipe=W.get("pipe"))
        e_total = maxred(e_total)
        e2e = {"value": W["flops"] * world / (e_total / e_steps * 1e-3) / 1e12, "unit": "TFLOP/s",
               "h2d_bytes_per_step": int(W["h2d"]), "d2h_bytes_per_step": int(W["d2h"]),
               "ms_per_step": e_total / e_steps, "path": (f"{type(W['pipe']).__name__}: pinned H2D, C-ABI call and D2H on three streams, overlapped across steps"
                        if W.get("pipe") is not None else "pinned host -> device copies + C-ABI call + D -> pinned host")}

    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        cpu = oracle_baseline(W["oracle_case"])
        if world > 1:
            cpu["sample"] += f"; rank 0's inputs, timed after the GPU region while the other {world - 1} rank(s) wait"

    if rank == 0:
        kinfo = cy.last_kernel_info() if args.workload != "attention" else None
        out = {
            "metric": metric_for(args.workload), "value": round(value, 2), "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_per_step, 5), "higher_is_better": True,
            "scaling": scaling_of(args.workload), "vs_baseline": None, "dtype": "f16",
            "data": "synthetic: seeded uniform[-1,1] rounded to fp16 (synth/), PCG64",
            "config": {"workload": W["desc"], **W["shape"],
                       "parallelism": (f"batch shards x{world}, no collective" if args.workload in ("batched", "batched-beta1", "attention")
                                       else f"M-row shards x{world}, B replicated, D and y exchanged by chunked NCCL point-to-point overlapped with the compute"
                                       if args.workload == "allgather"
                                       else f"M-row shards x{world}, B replicated, fused replication (epilogue peer stores, device barriers)"
                                       if args.workload == "allgather-fused"
                                       else f"M-row shards x{world}, B replicated, no collective"),
                       "l2": W["l2"],
                       "kernel_config": (kinfo if args.workload != "attention" else
                                         "attn_fwd_kernel: 2 x 128-row query tiles per CTA, 128-key blocks, TMEM S/P/O, 12 warps (setmaxnreg 208/72)")},
            "pct_of_dense_peak": round(100.0 * value / world / peak, 2),
            "pct_of_nominal_2250": round(100.0 * value / world / 2250.0, 2),
            "roofline": {"bound": "tensor", "achieved": round(achieved, 2), "peak": peak, "unit": "TFLOP/s",
                         "frac": round(achieved / peak, 4), "traffic": load_traffic(args.workload),
                         "peak_source": peaks["source"] + ("; sustained figure (sw_power_cap active, median SM clock < 90 % of max during the timed region)"
                                                           if power_capped else "; burst figure (SM clock near max during the timed region)"),
                         "frac_of_burst": round(achieved / peaks["burst"], 4),
                         "frac_of_sustained": round(achieved / peaks["sustained"], 4),
                         "kernel_ms": round(kern_ms, 5)},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "exchange": ({**W["exchange"], "compute_ms_at_peak": round(W["kernel_flops"] / (peak * 1e12) * 1e3, 4),
                          "measured_ms_per_step": round(ms_per_step, 4)} if "exchange" in W else None),
            "step_ms": step_stats(per),
            "gpu_launches": int(launches),
            "clocks": sampler.summary(),
            "timing": "CUDA events on the launching stream; barrier+sync both sides; max over ranks"
                      + ("; K steps captured in one CUDA graph, replay timed" if args.graph else ""),
        }
        print(json.dumps(out), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


def reference_arm(args, rank, world):
    """--impl reference: the fp64 CPU oracle (the only reference this tier has), timed as it
    stands on the host cores, each step a bounded sample of the same workload: >= 512 output rows
    (all columns, full K) or, batched, whole GEMMs of the batch -- the same sampling as the
    cpu_baseline leg of the GPU arm, so the two agree."""
    if rank != 0:
        return
    import numpy as np

    import oracle
    import synth

    oracle.build()
    oracle.set_threads(len(os.sched_getaffinity(0)))  # torchrun sets OMP_NUM_THREADS=1
    nth = oracle.num_threads()
    name = args.workload
    if name == "gemm" or name.startswith("sweep-"):
        n = 8192 if name == "gemm" else int(name.split("-")[1])
        case = ("gemm", (synth.uniform((n, n), synth.seed_for(1, 0)), synth.uniform((n, n), synth.seed_for(1, 1000))))
        desc = f"fp16 GEMM {n}^3" + (f" x{world} M-shards" if world > 1 else "")
    elif name in ("rowreduce", "allgather", "allgather-fused"):
        # the sampled rows come from one 2048-row block of A (the oracle's cost per row is the same)
        case = ("rowreduce" if name != "allgather-fused" else "gemm",
                (synth.uniform((2048, 8192), synth.seed_for(4, 0)), synth.uniform((8192, 8192), synth.seed_for(1, 1000))))
        desc = "fp16 GEMM 65536 x 8192 x 8192" + (" + row reduction" if name != "allgather-fused" else "")
    elif name in ("batched", "batched-beta1"):
        case = ("batched", (synth.uniform((64, 1024, 1024), synth.seed_for(2, 0)),
                            synth.uniform((64, 1024, 1024), synth.seed_for(2, 1))))
        desc = "batched fp16 GEMM 64 x 1024^3"
    elif name in ("glu", "dual"):
        n = 8192
        case = (name, tuple(synth.uniform((n, n), synth.seed_for(3, j)) for j in (0, 1001, 1002)))
        desc = "GLU dual-GEMM silu(A*B0)*(A*B1) 8192^3" if name == "glu" else "dual-GEMM pair 8192^3"
    elif name == "attention":
        bsz, h, s_len, d = 2, 16, 8192, 128
        Q, K, V = (synth.uniform((bsz * h, s_len, d), synth.seed_for(6, t)) for t in range(3))
        desc = f"FA forward fp16 HeadDim 128, non-causal, batch {bsz} x {h} heads x {s_len}"
        steps = min(args.steps, 10)
        warm = min(args.warmup, 3)
        rng = np.random.default_rng(0)
        for _ in range(warm):
            attention_sample(Q, K, V, bsz * h, budget_s=1.0, rng=rng)
        t0 = time.perf_counter()
        vals = [attention_sample(Q, K, V, bsz * h, budget_s=2.0, rng=rng) for _ in range(steps)]
        dt = time.perf_counter() - t0
        value = statistics.mean(v["value"] for v in vals)
        out = {"impl": "reference", "metric": ATTN_METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world,
               "steps": steps, "warmup": warm, "ms_per_step": dt / steps * 1e3, "higher_is_better": True,
               "scaling": scaling_of(name), "vs_baseline": None, "dtype": "f64",
               "data": "synthetic: seeded uniform[-1,1] rounded to fp16 (synth/), PCG64",
               "config": {"workload": desc, "parallelism": "CPU oracle, rank 0 only"},
               "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": vals[0]["cores"], "kind": "oracle",
                                "sample": f"per step: {vals[0]['sample']}"},
               "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(out), flush=True)
        return
    else:
        raise SystemExit(f"unknown workload {name}")
    kind = case[0]
    fn, per_unit, m, unit = oracle_unit_fn(*case)
    fixed, per, p1 = oracle_calibrate(fn, m, nth)
    # each step: >= 512 rows (batched: >= 1 GEMM), sized to ~10 s of CPU work -- the size of the
    # cpu_baseline leg's sample (12 s), so the fixed per-call cost (operand decode) weighs the same
    floor = 1 if kind == "batched" else min(m, 512)
    units_per_step = int(min(m, max(floor, (10.0 - fixed) / per)))
    steps = min(args.steps, 10)
    warm = min(args.warmup, 3)
    rng = np.random.default_rng(0)
    warm_units = int(min(m, max(1, (1.0 - fixed) / per)))
    for _ in range(warm):
        fn(np.sort(rng.choice(m, warm_units, replace=False)))
    t0 = time.perf_counter()
    for _ in range(steps):
        fn(np.sort(rng.choice(m, units_per_step, replace=False)))
    dt = time.perf_counter() - t0
    value = per_unit * units_per_step * steps / dt / 1e12
    sample = (f"{units_per_step} random {unit} per step of {desc}; {steps} steps in {dt:.1f} s "
              f"(calibrated fixed cost per call {fixed:.2f} s, {per * 1e3:.2f} ms per unit)")
    out = {"impl": "reference", "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world,
           "steps": steps, "warmup": warm, "ms_per_step": dt / steps * 1e3, "higher_is_better": True,
           "scaling": scaling_of(name), "vs_baseline": None, "dtype": "f64",
           "data": "synthetic: seeded uniform[-1,1] rounded to fp16 (synth/), PCG64",
           "config": {"workload": desc, "parallelism": "CPU oracle, rank 0 only"},
           "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": nth, "kind": "oracle", "sample": sample},
           "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
