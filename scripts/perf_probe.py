"""Perf probe (GPU box): per-variant time, achieved TFLOP/s, energy per GEMM and SM clock,
ours vs torch.matmul (cuBLAS, informational only) on identical inputs.

python scripts/perf_probe.py [--n 8192] [--iters 100] [--cfgs 0,1,2] [--dist uniform|zeros|randn] [--ks ...]
"""
import argparse
import os
import statistics
import sys
import threading
import time

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))

import torch  # noqa: E402

import paper_2504_07004_b200 as cy  # noqa: E402

try:
    import pynvml

    pynvml.nvmlInit()
    H = pynvml.nvmlDeviceGetHandleByIndex(0)
except Exception:  # pragma: no cover
    pynvml = None


def energy_mj():
    return pynvml.nvmlDeviceGetTotalEnergyConsumption(H) if pynvml else 0


class Clk:
    def __init__(self):
        self.s = []
        self.stop = False

    def run(self):
        while not self.stop:
            try:
                self.s.append((pynvml.nvmlDeviceGetClockInfo(H, pynvml.NVML_CLOCK_SM),
                               pynvml.nvmlDeviceGetPowerUsage(H) / 1000))
            except Exception:
                pass
            time.sleep(0.002)


def measure(fn, iters, warm=10, flops=1.0):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    clk = Clk()
    th = threading.Thread(target=clk.run, daemon=True) if pynvml else None
    if th:
        th.start()
    e0 = energy_mj()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        fn()
    b.record()
    torch.cuda.synchronize()
    e1 = energy_mj()
    clk.stop = True
    if th:
        th.join()
    ms = a.elapsed_time(b) / iters
    mhz = statistics.median([s[0] for s in clk.s]) if clk.s else 0
    pw = statistics.median([s[1] for s in clk.s]) if clk.s else 0
    return ms, flops / ms / 1e9, (e1 - e0) / iters, mhz, pw


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=8192)
    ap.add_argument("--m", type=int, default=0)
    ap.add_argument("--k", type=int, default=0)
    ap.add_argument("--iters", type=int, default=100)
    ap.add_argument("--cfgs", default="0")
    ap.add_argument("--dist", default="uniform")
    ap.add_argument("--torch", action="store_true")
    ap.add_argument("--dtype", default="f16")
    args = ap.parse_args()
    n = args.n
    m = args.m or n
    k = args.k or n
    dt = torch.float16 if args.dtype == "f16" else torch.bfloat16
    g = torch.Generator(device="cuda").manual_seed(0)
    mk = {"uniform": lambda s: torch.empty(s, device="cuda", dtype=dt).uniform_(-1, 1, generator=g),
          "randn": lambda s: torch.randn(s, device="cuda", dtype=dt, generator=g),
          "zeros": lambda s: torch.zeros(s, device="cuda", dtype=dt)}[args.dist]
    sets = [(mk((m, k)), mk((k, n))) for _ in range(2)]
    D = torch.empty((m, n), device="cuda", dtype=dt)
    flops = 2.0 * m * n * k
    it = [0]

    def ours():
        a, b = sets[it[0] & 1]
        it[0] += 1
        cy.gemm(a, b, out=D)

    def theirs():
        a, b = sets[it[0] & 1]
        it[0] += 1
        torch.matmul(a, b, out=D)

    for c in [int(x) for x in args.cfgs.split(",")]:
        cy.force_config(c)
        ms, tf, mj, mhz, pw = measure(ours, args.iters, flops=flops)
        print(f"{args.dist} {m}x{n}x{k} cfg{c} {cy.config_info(c)}: {ms:.4f} ms {tf:8.1f} TFLOP/s "
              f"{mj:7.1f} mJ/gemm  sm {mhz} MHz  {pw:.0f} W", flush=True)
    cy.force_config(-1)
    if args.torch:
        ms, tf, mj, mhz, pw = measure(theirs, args.iters, flops=flops)
        print(f"{args.dist} {m}x{n}x{k} torch.matmul: {ms:.4f} ms {tf:8.1f} TFLOP/s {mj:7.1f} mJ/gemm  "
              f"sm {mhz} MHz  {pw:.0f} W", flush=True)


if __name__ == "__main__":
    main()
