"""One workload, a few launches (for ncu): python one_gemm.py g8192 | rr65536 | b64 [launches]"""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
import torch

import paper_2504_07004_b200 as cy

w = sys.argv[1]
nl = int(sys.argv[2]) if len(sys.argv) > 2 else 3
u = lambda *s: torch.empty(s, device="cuda", dtype=torch.float16).uniform_(-1, 1)  # noqa
if w.startswith("g"):
    n = int(w[1:])
    a, b, d = u(n, n), u(n, n), u(n, n)
    run = lambda: cy.gemm(a, b, out=d)  # noqa
elif w.startswith("rr"):
    m = int(w[2:])
    a, b, d = u(m, 8192), u(8192, 8192), u(m, 8192)
    y = torch.empty(m, device="cuda", dtype=torch.float32)
    run = lambda: cy.gemm_rowreduce(a, b, out=d, y=y)  # noqa
else:
    L = int(w[1:])
    a, b, d = u(L, 1024, 1024), u(L, 1024, 1024), u(L, 1024, 1024)
    run = lambda: cy.gemm_batched(a, b, out=d)  # noqa
for _ in range(nl):
    run()
torch.cuda.synchronize()
