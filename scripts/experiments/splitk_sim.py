"""What split-K would buy at small sizes, without building it: device time (CUDA-graph replay) of
the per-split work alone (2 or 4 x the tiles at K/2 or K/4) vs the unsplit GEMM."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
import torch
import paper_2504_07004_b200 as cy
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from kscan_probe import graph_time  # noqa: E402

def t(m, n, k, cfg):
    a = torch.empty((m, k), device="cuda", dtype=torch.float16).uniform_(-1, 1)
    b = torch.empty((k, n), device="cuda", dtype=torch.float16).uniform_(-1, 1)
    d = torch.empty((m, n), device="cuda", dtype=torch.float16)
    cy.force_config(cfg)
    r = graph_time(lambda: cy.gemm(a, b, out=d))
    cy.force_config(-1)
    return r

for n in (1024, 1536):
    for cfg in (0, 1, 2, 3, 4):
        base = t(n, n, n, cfg)
        s2 = t(2 * n, n, n // 2, cfg)
        s4 = t(4 * n, n, n // 4, cfg)
        print(f"n={n} cfg{cfg}: unsplit {base:6.2f} us | split-2 work {s2:6.2f} | split-4 work {s4:6.2f}", flush=True)
