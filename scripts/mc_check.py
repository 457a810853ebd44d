"""Quick parity + throughput check of one forced GEMM config against torch (fp32-accumulated) at a few shapes."""
import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch
import paper_2504_07004_b200 as cy

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 6
for (m, n, k) in ((512, 512, 64), (1024, 512, 256), (1000, 704, 304), (2048, 2048, 1024), (4096, 4096, 4096)):
    a = torch.randint(-2, 3, (m, k), device="cuda").half()
    b = torch.randint(-2, 3, (k, n), device="cuda").half()
    cy.force_config(cfg)
    d = cy.gemm(a, b)
    torch.cuda.synchronize()
    ref = (a.float() @ b.float()).half()
    print(f"cfg {cy.last_config()} {m}x{n}x{k}: exact={torch.equal(d, ref)}", flush=True)
