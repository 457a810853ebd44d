"""Batched 64 x 1024^3 with operands from HBM (distinct batches) vs L2-resident (every batch reads
almost the same A/B: batch stride 8 elements).  Graph-replay device time per launch."""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch  # noqa: E402

import paper_2504_07004_b200 as cy  # noqa: E402
from kscan_probe import graph_time  # noqa: E402

L = 64
u = lambda *s: torch.empty(s, device="cuda", dtype=torch.float16).uniform_(-1, 1)  # noqa
fl = 2.0 * L * 1024 ** 3
sets = [(u(L, 1024, 1024), u(L, 1024, 1024)) for _ in range(4)]
baseA, baseB = u(1024 * 1024 + 8 * L), u(1024 * 1024 + 8 * L)
Ar = torch.as_strided(baseA, (L, 1024, 1024), (8, 1024, 1))
Br = torch.as_strided(baseB, (L, 1024, 1024), (8, 1024, 1))
D = torch.empty((L, 1024, 1024), device="cuda", dtype=torch.float16)
it = [0]


def hbm():
    it[0] += 1
    a, b = sets[it[0] % 4]
    cy.gemm_batched(a, b, out=D)


def l2():
    cy.gemm_batched(Ar, Br, out=D)


for c in [int(x) for x in (sys.argv[1:] or ["-1", "0"])]:
    cy.force_config(c)
    th = min(graph_time(hbm, 20) for _ in range(3))
    tl = min(graph_time(l2, 20) for _ in range(3))
    print(f"cfg {c}: HBM operands {th:8.2f} us {fl / th / 1e6:6.0f} TF | L2-resident operands {tl:8.2f} us {fl / tl / 1e6:6.0f} TF", flush=True)
