"""Host cost per call (no synchronisation inside the loop): the Python binding, the raw C-ABI call
with pre-marshalled arguments, and torch.matmul (informational), at a tiny shape."""
import os, sys, time
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
import torch
import paper_2504_07004_b200 as cy
from paper_2504_07004_b200 import _lib

n = 256
a = torch.empty((n, n), device="cuda", dtype=torch.float16).uniform_(-1, 1)
b = torch.empty((n, n), device="cuda", dtype=torch.float16).uniform_(-1, 1)
d = torch.empty((n, n), device="cuda", dtype=torch.float16)
lib = _lib.load()
s = torch._C._cuda_getCurrentRawStream(0)
args = (0, n, n, n, 1.0, a.data_ptr(), n, b.data_ptr(), n, 0.0, None, n, d.data_ptr(), n, s)


def timeit(fn, N=20000):
    for _ in range(200):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(N):
        fn()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    return 1e6 * (t1 - t0) / N


print(f"binding cy.gemm(out=)  {timeit(lambda: cy.gemm(a, b, out=d)):6.2f} us/call")
print(f"raw C-ABI cy_gemm       {timeit(lambda: lib.cy_gemm(*args)):6.2f} us/call")
print(f"torch.matmul(out=)      {timeit(lambda: torch.matmul(a, b, out=d)):6.2f} us/call")
print(f"torch.empty (reference) {timeit(lambda: torch.empty((n, n), device='cuda', dtype=torch.float16)):6.2f} us/call")
