"""Split-K calibration grid: device time (CUDA-graph replay) of every splittable config x split count
for small-output / long-K shapes, beside the library's auto choice and cuBLAS.
Usage: python scripts/splitk_grid.py"""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch  # noqa: E402

import paper_2504_07004_b200 as cy  # noqa: E402
from kscan_probe import graph_time  # noqa: E402

SHAPES = [(1024, 1024, 1024), (1024, 1024, 4096), (1024, 1024, 16384), (2048, 2048, 2048), (2048, 2048, 8192),
          (512, 512, 16384), (256, 256, 65536), (1024, 8192, 8192)]
for m, n, k in SHAPES:
    a = torch.empty((m, k), device="cuda", dtype=torch.float16).uniform_(-1, 1)
    b = torch.empty((k, n), device="cuda", dtype=torch.float16).uniform_(-1, 1)
    d = torch.empty((m, n), device="cuda", dtype=torch.float16)
    print(f"{m}x{n}x{k}: auto {graph_time(lambda: cy.gemm(a, b, out=d)):7.2f} "
          f"(s{cy.last_splits()} c{cy.last_config()})  cuBLAS {graph_time(lambda: torch.matmul(a, b, out=d)):7.2f}",
          flush=True)
    for cfg in range(5):
        cy.force_config(cfg)
        row = []
        for sp in (1, 2, 4, 8):
            if cfg in (0, 1) and sp == 8:
                continue
            us = graph_time(lambda: cy.gemm(a, b, out=d, splits=sp))
            row.append(f"s{sp}:{us:7.2f}")
        print(f"   c{cfg} " + " ".join(row), flush=True)
    cy.force_config(-1)
