import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch
import paper_2504_07004_b200 as cy
s = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
b = int(sys.argv[2]) if len(sys.argv) > 2 else 1
Q, K, V = (torch.empty((b, 16, s, 128), device="cuda", dtype=torch.float16).uniform_(-1, 1) for _ in range(3))
for _ in range(3):
    cy.attention(Q, K, V)
torch.cuda.synchronize()
