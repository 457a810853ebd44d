"""Small-shape device time per launch for every GEMM config (forced) vs the host heuristic and torch."""
import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
import torch
import paper_2504_07004_b200 as cy


def dev_time(fn, reps=200):
    for _ in range(20):
        fn()
    big = torch.empty((8192, 8192), device="cuda", dtype=torch.float16)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.matmul(big, big)  # queue the launches behind a long kernel
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3  # us


for n in [int(x) for x in (sys.argv[1:] or ["1024", "2048", "3072", "4096"])]:
    a = torch.empty((n, n), device="cuda", dtype=torch.float16).uniform_(-1, 1)
    b = torch.empty((n, n), device="cuda", dtype=torch.float16).uniform_(-1, 1)
    d = torch.empty((n, n), device="cuda", dtype=torch.float16)
    cy.force_config(-1)
    t = dev_time(lambda: cy.gemm(a, b, out=d))
    line = [f"n={n}: auto(cfg {cy.last_config()}) {t:7.2f}us"]
    for c in range(cy.num_configs()):
        cy.force_config(c)
        line.append(f"c{c} {dev_time(lambda: cy.gemm(a, b, out=d)):7.2f}")
    cy.force_config(-1)
    line.append(f"torch {dev_time(lambda: torch.matmul(a, b, out=d)):7.2f}")
    print(" | ".join(line), flush=True)
