"""Name and launch geometry of the kernel torch.matmul (cuBLAS) runs for an fp16 8192^3 GEMM (informational)."""
import torch
from torch.profiler import profile, ProfilerActivity

a = torch.empty((8192, 8192), device="cuda", dtype=torch.float16).uniform_(-1, 1)
b = torch.empty_like(a)
for _ in range(3):
    torch.matmul(a, b)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    torch.matmul(a, b)
    torch.cuda.synchronize()
for e in prof.events():
    if e.device_type.name == "CUDA":
        print(e.name)
