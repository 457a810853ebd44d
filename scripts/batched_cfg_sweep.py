"""Batched 64 x 1024^3 (BASELINE configs[2]) per config and beta, device time per launch.
Launches queued back to back over 4 rotating input sets (> 2x L2), CUDA events; cuBLAS bmm
beside it for context.  Usage: python scripts/batched_cfg_sweep.py [L] [iters]"""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch

import paper_2504_07004_b200 as cy

L = int(sys.argv[1]) if len(sys.argv) > 1 else 64
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 200
g = torch.Generator(device="cuda").manual_seed(0)
mk = lambda: torch.empty((L, 1024, 1024), device="cuda", dtype=torch.float16).uniform_(-1, 1, generator=g)  # noqa
sets = [(mk(), mk(), mk()) for _ in range(4)]
D = torch.empty((L, 1024, 1024), device="cuda", dtype=torch.float16)
fl = 2.0 * L * 1024 ** 3


def t(fn):
    for i in range(10):
        fn(i)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(iters):
        fn(i)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters * 1e3


for beta in (0.0, 1.0):
    for cfg in [-1] + list(range(cy.num_configs())):
        cy.force_config(cfg)
        us = t(lambda i: cy.gemm_batched(sets[i % 4][0], sets[i % 4][1], sets[i % 4][2], 1.0, beta, out=D))
        ki = cy.last_kernel_info()
        print(f"beta={beta} cfg={cfg:2d} {ki['cta_group']}x{ki['tile_m']}x{ki['tile_n']} st{ki['stages']}: "
              f"{us:8.2f} us {fl / us / 1e6:8.1f} TFLOP/s", flush=True)
    cy.force_config(-1)
    if beta == 0.0:
        us = t(lambda i: torch.bmm(sets[i % 4][0], sets[i % 4][1], out=D))
    else:
        us = t(lambda i: torch.baddbmm(sets[i % 4][2], sets[i % 4][0], sets[i % 4][1], out=D))
    print(f"beta={beta} cuBLAS: {us:8.2f} us {fl / us / 1e6:8.1f} TFLOP/s", flush=True)
