"""Kernel-level timeline of every CTA of one GEMM launch (trace build: scripts/build_experiment.py
gtrace CY_GEMM_TRACE=1).  Per CTA, clock64 cycles after its own entry of:
  pro  prologue done (barriers, TMEM, cluster sync)   full  first stage full at the MMA issuer (leaders)
  mma  last accumulator committed (leaders)            st    last D store issued (epilogue warp 0)
  done last D store complete                            sync  reached the final cluster sync
  exit TMEM freed
and the entry skew (globaltimer, ns) across CTAs.  Usage: python scripts/gemm_ktrace.py M N K [cfg] [splits]"""
import ctypes
import os
import statistics
import sys

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
sys.path.insert(0, ROOT)
from paper_2504_07004_b200 import _lib  # noqa: E402

_lib.use_library(os.path.join(ROOT, "build", "exp", "libcypress_gtrace.so"))
import torch  # noqa: E402

import paper_2504_07004_b200 as cy  # noqa: E402

m, n, k = (int(x) for x in sys.argv[1:4])
cfg = int(sys.argv[4]) if len(sys.argv) > 4 else -1
splits = int(sys.argv[5]) if len(sys.argv) > 5 else None
lib = _lib.load()
lib.cy_gemm_ktrace_read.argtypes = [ctypes.POINTER(ctypes.c_ulonglong), ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_int]
cy.force_config(cfg)
a = torch.empty((m, k), device="cuda", dtype=torch.float16).uniform_(-1, 1)
b = torch.empty((k, n), device="cuda", dtype=torch.float16).uniform_(-1, 1)
d = torch.empty((m, n), device="cuda", dtype=torch.float16)
ev = (ctypes.c_ulonglong * (1024 * 8))()
gt = (ctypes.c_ulonglong * 1024)()
for i in range(20):
    cy.gemm(a, b, out=d, splits=splits)
torch.cuda.synchronize()
lib.cy_gemm_ktrace_read(ev, gt, 1)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
cy.gemm(a, b, out=d, splits=splits)
e1.record()
torch.cuda.synchronize()
lib.cy_gemm_ktrace_read(ev, gt, 0)
ctas = [c for c in range(1024) if ev[c * 8]]
g0 = min(gt[c] for c in ctas)
print(f"{m}x{n}x{k} cfg {cy.last_kernel_info()} splits {cy.last_splits()}: {len(ctas)} CTAs, event time {e0.elapsed_time(e1) * 1e3:.1f} us")
names = ["pro", "full", "mma", "st", "done", "sync", "exit"]
print("entry skew ns: max", max(gt[c] for c in ctas) - g0)
for j, nm in enumerate(names, start=1):
    v = [ev[c * 8 + j] - ev[c * 8] for c in ctas if ev[c * 8 + j]]
    if v:
        print(f"{nm:5s} cycles after entry: min {min(v):7d} median {int(statistics.median(v)):7d} max {max(v):7d}  (n={len(v)})")
