import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch
import paper_2504_07004_b200 as cy
s = int(sys.argv[1]) if len(sys.argv) > 1 else 256
Q, K, V = (torch.empty((1, 1, s, 128), device="cuda", dtype=torch.float16).uniform_(-1, 1) for _ in range(3))
O, lse = cy.attention(Q, K, V)
torch.cuda.synchronize()
ref = torch.nn.functional.scaled_dot_product_attention(Q.float(), K.float(), V.float())
print("max err", (O.float() - ref).abs().max().item())
