"""Split-K (NEXT-1) device time per launch under CUDA-graph replay: unsplit (splits=1), the
library's choice (auto) and forced split counts, beside cuBLAS, for small-output / long-K shapes.
Usage: python scripts/splitk_probe.py"""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch  # noqa: E402

import paper_2504_07004_b200 as cy  # noqa: E402
from kscan_probe import graph_time  # noqa: E402

SHAPES = [(1024, 1024, 1024), (2048, 2048, 2048), (1024, 1024, 4096), (1024, 1024, 8192), (1024, 1024, 16384),
          (2048, 2048, 8192), (512, 512, 16384), (1024, 8192, 8192), (256, 256, 65536)]
for m, n, k in SHAPES:
    a = torch.empty((m, k), device="cuda", dtype=torch.float16).uniform_(-1, 1)
    b = torch.empty((k, n), device="cuda", dtype=torch.float16).uniform_(-1, 1)
    d = torch.empty((m, n), device="cuda", dtype=torch.float16)
    line = [f"{m}x{n}x{k}:"]
    for sp in (1, None, 2, 4, 8):
        us = graph_time(lambda: cy.gemm(a, b, out=d, splits=sp))
        cy.gemm(a, b, out=d, splits=sp)
        line.append(f"s{sp if sp else 'auto'}({cy.last_splits()},c{cy.last_config()}) {us:7.2f}")
    line.append(f"cuBLAS {graph_time(lambda: torch.matmul(a, b, out=d)):7.2f} us")
    print(" ".join(line), flush=True)
