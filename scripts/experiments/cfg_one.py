"""One forced-config GEMM, checked against torch (debugging a config):
python scripts/experiments/cfg_one.py CFG M N K"""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
import torch

import paper_2504_07004_b200 as cy

cfg, m, n, k = (int(x) for x in sys.argv[1:5])
g = torch.Generator(device="cuda").manual_seed(0)
a = torch.randint(-3, 4, (m, k), device="cuda", generator=g).half()
b = torch.randint(-3, 4, (k, n), device="cuda", generator=g).half()
cy.force_config(cfg)
d = cy.gemm(a, b)
torch.cuda.synchronize()
ref = (a.float() @ b.float()).half()
print("cfg", cy.last_config(), cy.last_kernel_info(), "exact:", bool(torch.equal(d, ref)),
      "max err", (d.float() - ref.float()).abs().max().item())
