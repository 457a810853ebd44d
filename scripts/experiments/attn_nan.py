"""Locate non-finite / wrong rows of an attention build against torch (fp32) on a peaky input:
CY_EXP_LIB=LIB python scripts/experiments/attn_nan.py [qscale] [sq] [sk]"""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
import torch

from paper_2504_07004_b200 import _lib

if os.environ.get("CY_EXP_LIB"):
    _lib.use_library(os.path.abspath(os.environ["CY_EXP_LIB"]))
import paper_2504_07004_b200 as cy

qs = float(sys.argv[1]) if len(sys.argv) > 1 else 8.0
sq = int(sys.argv[2]) if len(sys.argv) > 2 else 640
sk = int(sys.argv[3]) if len(sys.argv) > 3 else 640
g = torch.Generator(device="cuda").manual_seed(0)
Q = (torch.rand((1, 4, sq, 128), device="cuda", generator=g) * 2 - 1).mul(qs).half()
K = (torch.rand((1, 4, sk, 128), device="cuda", generator=g) * 2 - 1).half()
V = (torch.rand((1, 4, sk, 128), device="cuda", generator=g) * 2 - 1).half()
O, lse = cy.attention(Q, K, V)
torch.cuda.synchronize()
S = (Q.float() @ K.float().transpose(-1, -2)) * 128 ** -0.5
ref = torch.softmax(S, -1) @ V.float()
bad = ~torch.isfinite(O.float())
print("nonfinite", int(bad.sum()), "rows", torch.nonzero(bad.any(-1))[:8].tolist())
err = (O.float() - ref).abs().amax(-1)
print("max err", float(err[torch.isfinite(err)].max()), "rows err>1e-2", int((err > 1e-2).sum()), torch.nonzero(err > 1e-2)[:8].tolist())
lref = torch.logsumexp(S, -1)
print("lse max diff", float((lse - lref).abs()[torch.isfinite(lse)].max()), "nonfinite lse", int((~torch.isfinite(lse)).sum()))
