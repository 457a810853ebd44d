"""Which cuBLAS kernel torch.matmul runs for the small / split-K shapes (run under ncu)."""
import torch
for (m, n, k) in [(1024, 1024, 1024), (2048, 2048, 2048), (1024, 1024, 4096), (1024, 1024, 16384), (512, 512, 16384)]:
    a = torch.randn(m, k, device="cuda", dtype=torch.float16)
    b = torch.randn(k, n, device="cuda", dtype=torch.float16)
    for _ in range(3):
        torch.matmul(a, b)
torch.cuda.synchronize()
