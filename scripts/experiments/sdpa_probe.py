"""Run torch SDPA (informational comparator) at the attention bench shape, for ncu inspection."""
import torch
b, h, s, d = 2, 16, 8192, 128
Q, K, V = (torch.empty((b, h, s, d), device="cuda", dtype=torch.float16).uniform_(-1, 1) for _ in range(3))
for _ in range(3):
    torch.nn.functional.scaled_dot_product_attention(Q, K, V)
torch.cuda.synchronize()
