"""Run torch.matmul (cuBLAS, informational comparator only) n^3 a few times (for ncu)."""
import sys
import torch
n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
a = torch.empty((n, n), device="cuda", dtype=torch.float16).uniform_(-1, 1)
b = torch.empty((n, n), device="cuda", dtype=torch.float16).uniform_(-1, 1)
for _ in range(6):
    c = torch.matmul(a, b)
torch.cuda.synchronize()
