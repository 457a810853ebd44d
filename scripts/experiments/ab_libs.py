"""A/B of several library builds on the same box, interleaved: 8192^3 GEMM, batched 64x1024^3
(beta 0 and 1), dual 8192^3.  Each lib runs in its own subprocess (one library per process);
rounds alternate so clock drift hits every lib alike.
Usage: python scripts/experiments/ab_libs.py ROUNDS lib1.so[=label] lib2.so ..."""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.join(HERE, "..", "..")

CHILD = r'''
import os, sys, torch
sys.path.insert(0, __ROOT__)
from paper_2504_07004_b200 import _lib
if __LIB__ != "-": _lib.use_library(__LIB__)
import paper_2504_07004_b200 as cy
def t(fn, iters):
    for i in range(5): fn(i)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(iters): fn(i)
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters * 1e3
g = torch.Generator(device="cuda").manual_seed(0)
u = lambda *s: torch.empty(s, device="cuda", dtype=torch.float16).uniform_(-1, 1, generator=g)
A = [u(8192, 8192) for _ in range(2)]; B = [u(8192, 8192) for _ in range(2)]; D = u(8192, 8192); D1 = u(8192, 8192)
us = t(lambda i: cy.gemm(A[i % 2], B[i % 2], out=D), 100)
print(f"{__LABEL__:10s} gemm8192  {us:9.2f} us {2*8192**3/us/1e6:8.1f} TF", flush=True)
us = t(lambda i: cy.dual_gemm(A[i % 2], B[0], B[1], out0=D, out1=D1), 50)
print(f"{__LABEL__:10s} dual8192  {us:9.2f} us {4*8192**3/us/1e6:8.1f} TF", flush=True)
del A, B, D, D1
Ab = [u(64, 1024, 1024) for _ in range(4)]; Bb = [u(64, 1024, 1024) for _ in range(4)]; Cb = [u(64, 1024, 1024) for _ in range(4)]
Db = u(64, 1024, 1024)
for beta in (0.0, 1.0):
    us = t(lambda i: cy.gemm_batched(Ab[i % 4], Bb[i % 4], Cb[i % 4], 1.0, beta, out=Db), 200)
    print(f"{__LABEL__:10s} batched b{beta:.0f} {us:9.2f} us {2*64*1024**3/us/1e6:8.1f} TF", flush=True)
'''

rounds = int(sys.argv[1])
libs = []
for a in sys.argv[2:]:
    path, _, label = a.partition("=")
    libs.append((path if path == "-" else os.path.abspath(path), label or os.path.basename(path)))
for r in range(rounds):
    for path, label in libs:
        code = CHILD.replace("__ROOT__", repr(ROOT)).replace("__LIB__", repr(path)).replace("__LABEL__", repr(label))
        subprocess.run([sys.executable, "-c", code], check=False)
