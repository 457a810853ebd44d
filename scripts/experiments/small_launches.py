"""Small square GEMMs, ours (auto config) and torch.matmul back to back: run under
ncu --metrics gpu__time_duration.sum to read kernel durations beside graph-replay step times."""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
import torch

import paper_2504_07004_b200 as cy

for n in [int(x) for x in (sys.argv[1:] or ["1024", "2048"])]:
    a = torch.empty((n, n), device="cuda", dtype=torch.float16).uniform_(-1, 1)
    b = torch.empty((n, n), device="cuda", dtype=torch.float16).uniform_(-1, 1)
    d = torch.empty((n, n), device="cuda", dtype=torch.float16)
    for _ in range(10):
        cy.gemm(a, b, out=d)
    torch.cuda.synchronize()
    for _ in range(10):
        torch.matmul(a, b, out=d)
    torch.cuda.synchronize()
    print(n, cy.last_kernel_info(), cy.last_splits(), flush=True)
