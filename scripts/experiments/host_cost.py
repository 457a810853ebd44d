"""Host cost per call (wall clock, GPU work negligible): the Python binding, the raw ctypes call, and
torch.matmul for reference.  python scripts/experiments/host_cost.py [n]"""
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
import torch

import paper_2504_07004_b200 as cy
from paper_2504_07004_b200 import _lib

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
a = torch.randn(n, n, device="cuda", dtype=torch.float16)
b = torch.randn(n, n, device="cuda", dtype=torch.float16)
d = torch.empty(n, n, device="cuda", dtype=torch.float16)
lib = _lib.load()
st = torch.cuda.current_stream().cuda_stream


def wall(fn, it=3000):
    for _ in range(100):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(it):
        fn()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    return (t1 - t0) / it * 1e6


print(f"cy.gemm(out=)       {wall(lambda: cy.gemm(a, b, out=d)):6.2f} us/call")
print(f"raw ctypes cy_gemm  {wall(lambda: lib.cy_gemm(0, n, n, n, 1.0, a.data_ptr(), n, b.data_ptr(), n, 0.0, None, n, d.data_ptr(), n, st)):6.2f} us/call")
print(f"torch.matmul(out=)  {wall(lambda: torch.matmul(a, b, out=d)):6.2f} us/call")
