"""Batched L x 1024^3 probe (for ncu and timing)."""
import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
import torch
import paper_2504_07004_b200 as cy
L = int(sys.argv[1]) if len(sys.argv) > 1 else 8
cfg = int(sys.argv[2]) if len(sys.argv) > 2 else -1
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 200
g = torch.Generator(device="cuda").manual_seed(0)
sets = [(torch.empty((L, 1024, 1024), device="cuda", dtype=torch.float16).uniform_(-1, 1, generator=g),
         torch.empty((L, 1024, 1024), device="cuda", dtype=torch.float16).uniform_(-1, 1, generator=g)) for _ in range(4)]
D = torch.empty((L, 1024, 1024), device="cuda", dtype=torch.float16)
cy.force_config(cfg)
for i in range(10):
    cy.gemm_batched(*sets[i % 4], out=D)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for i in range(iters):
    cy.gemm_batched(*sets[i % 4], out=D)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / iters
print(f"L={L} cfg{cfg} {cy.last_kernel_info()}: {ms * 1e3:.2f} us  {2 * L * 1024 ** 3 / ms / 1e9:.1f} TFLOP/s", flush=True)
for name, f in (("torch.bmm", lambda a, b: torch.bmm(a, b, out=D)),):
    for i in range(10):
        f(*sets[i % 4])
    torch.cuda.synchronize()
    e0.record()
    for i in range(iters):
        f(*sets[i % 4])
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / iters
    print(f"L={L} {name}: {ms * 1e3:.2f} us  {2 * L * 1024 ** 3 / ms / 1e9:.1f} TFLOP/s", flush=True)
