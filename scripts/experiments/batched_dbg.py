"""Batched 64 x 1024^3: time configs 0 and 5 with a given library (product or experiment build).
Usage: python scripts/experiments/batched_dbg.py [lib.so] [label]"""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
from paper_2504_07004_b200 import _lib  # noqa: E402

if len(sys.argv) > 1 and sys.argv[1] != "-":
    _lib.use_library(os.path.abspath(sys.argv[1]))
label = sys.argv[2] if len(sys.argv) > 2 else "product"
import torch  # noqa: E402

import paper_2504_07004_b200 as cy  # noqa: E402

L, iters = 64, 200
g = torch.Generator(device="cuda").manual_seed(0)
mk = lambda: torch.empty((L, 1024, 1024), device="cuda", dtype=torch.float16).uniform_(-1, 1, generator=g)  # noqa
sets = [(mk(), mk()) for _ in range(4)]
D = torch.empty((L, 1024, 1024), device="cuda", dtype=torch.float16)
fl = 2.0 * L * 1024 ** 3
for cfg in (0, 5):
    cy.force_config(cfg)
    for i in range(10):
        cy.gemm_batched(*sets[i % 4], out=D)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(iters):
        cy.gemm_batched(*sets[i % 4], out=D)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / iters * 1e3
    print(f"{label} {os.environ.get('CY_SCHED', '')}{os.environ.get('CY_GROUP_M', '')} cfg{cfg}: {us:8.2f} us "
          f"{fl / us / 1e6:7.1f} TFLOP/s", flush=True)
