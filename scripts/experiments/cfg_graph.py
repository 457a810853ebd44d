"""Graph-replay device time per launch for forced GEMM configs on square / batched shapes.
python scripts/experiments/cfg_graph.py CFGS SHAPES   e.g.  -1,0,7 1024,2048,4096,b64"""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch  # noqa: E402

from paper_2504_07004_b200 import _lib  # noqa: E402

if os.environ.get("CY_EXP_LIB"):  # A/B against an experiment build
    _lib.use_library(os.path.abspath(os.environ["CY_EXP_LIB"]))
import paper_2504_07004_b200 as cy  # noqa: E402
from kscan_probe import graph_time  # noqa: E402

cfgs = [int(c) for c in sys.argv[1].split(",")]
for sh in sys.argv[2].split(","):
    if sh.startswith("b"):
        L = int(sh[1:])
        sets = [tuple(torch.empty((L, 1024, 1024), device="cuda", dtype=torch.float16).uniform_(-1, 1) for _ in range(2))
                for _ in range(4)]
        d = torch.empty((L, 1024, 1024), device="cuda", dtype=torch.float16)
        fl = 2.0 * L * 1024 ** 3
        it = [0]

        def run():
            it[0] += 1
            a, b = sets[it[0] % 4]
            cy.gemm_batched(a, b, out=d)
    else:
        n = int(sh)
        a = torch.empty((n, n), device="cuda", dtype=torch.float16).uniform_(-1, 1)
        b = torch.empty((n, n), device="cuda", dtype=torch.float16).uniform_(-1, 1)
        d = torch.empty((n, n), device="cuda", dtype=torch.float16)
        fl = 2.0 * n ** 3

        def run():
            cy.gemm(a, b, out=d)
    line = [f"{os.path.basename(os.environ.get('CY_EXP_LIB', 'product'))[:18]:18s} {sh:6s}"]
    for c in cfgs:
        cy.force_config(c)
        us = min(graph_time(run, reps=20 if fl > 1e11 else 50) for _ in range(3))
        line.append(f"c{c}:{us:8.2f}us {fl / us / 1e6:6.0f}TF")
    cy.force_config(-1)
    print(" | ".join(line), flush=True)
