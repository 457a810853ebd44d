"""M-shard probe: an m x 8192 x 8192 GEMM (the 8192^3 problem strong-scaled over 8192/m GPUs), every config
forced vs the heuristic vs torch.matmul, device time per launch with the launches queued behind a long kernel."""
import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
import torch
import paper_2504_07004_b200 as cy
from small_probe_util import dev_time

n = k = 8192
for m in [int(x) for x in (sys.argv[1:] or ["1024", "2048", "4096"])]:
    sets = [(torch.empty((m, k), device="cuda", dtype=torch.float16).uniform_(-1, 1),
             torch.empty((k, n), device="cuda", dtype=torch.float16).uniform_(-1, 1)) for _ in range(2)]
    d = torch.empty((m, n), device="cuda", dtype=torch.float16)
    it = [0]

    def run(f):
        def g():
            a, b = sets[it[0] % 2]
            it[0] += 1
            f(a, b)
        return g
    cy.force_config(-1)
    t = dev_time(run(lambda a, b: cy.gemm(a, b, out=d)))
    fl = 2.0 * m * n * k
    line = [f"m={m}: auto(cfg {cy.last_config()}) {t:7.2f}us {fl / t / 1e6:6.0f}TF"]
    for c in range(cy.num_configs()):
        cy.force_config(c)
        t = dev_time(run(lambda a, b: cy.gemm(a, b, out=d)))
        line.append(f"c{c} {t:7.2f}")
    cy.force_config(-1)
    t = dev_time(run(lambda a, b: torch.matmul(a, b, out=d)))
    line.append(f"torch {t:7.2f}us {fl / t / 1e6:6.0f}TF")
    print("  ".join(line), flush=True)
