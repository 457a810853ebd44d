"""B-multicast 4-CTA clusters with one 256-wide accumulator (config 7) vs configs 0/5, graph replay."""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch  # noqa: E402

import paper_2504_07004_b200 as cy  # noqa: E402
from kscan_probe import graph_time  # noqa: E402

for m, n, k in [(2048, 2048, 2048), (4096, 4096, 4096), (1024, 8192, 8192), (2048, 2048, 8192), (8192, 8192, 8192)]:
    a = torch.empty((m, k), device="cuda", dtype=torch.float16).uniform_(-1, 1)
    b = torch.empty((k, n), device="cuda", dtype=torch.float16).uniform_(-1, 1)
    d = torch.empty((m, n), device="cuda", dtype=torch.float16)
    row = [f"{m}x{n}x{k}:"]
    for cfg in (-1, 0, 5, 6, 7):
        cy.force_config(cfg)
        row.append(f"c{cfg} {graph_time(lambda: cy.gemm(a, b, out=d, splits=1), reps=20):8.2f}")
    cy.force_config(-1)
    row.append(f"cuBLAS {graph_time(lambda: torch.matmul(a, b, out=d), reps=20):8.2f}")
    print(" ".join(row), flush=True)
L = 64
A = torch.empty((L, 1024, 1024), device="cuda", dtype=torch.float16).uniform_(-1, 1)
B = torch.empty((L, 1024, 1024), device="cuda", dtype=torch.float16).uniform_(-1, 1)
D = torch.empty((L, 1024, 1024), device="cuda", dtype=torch.float16)
row = ["batched 64x1024^3:"]
for cfg in (-1, 0, 5, 6, 7):
    cy.force_config(cfg)
    row.append(f"c{cfg} {graph_time(lambda: cy.gemm_batched(A, B, out=D, splits=1), reps=50):8.2f}")
cy.force_config(-1)
row.append(f"cuBLAS {graph_time(lambda: torch.bmm(A, B, out=D), reps=50):8.2f}")
print(" ".join(row), flush=True)
