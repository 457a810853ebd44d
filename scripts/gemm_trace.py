"""Per-tile event trace of one CTA of the GEMM kernel (trace build: scripts/build_experiment.py
gtrace CY_GEMM_TRACE=1).  Prints, per tile of CTA 0, the clock64 offsets (cycles) of:
  P0 producer has the tile   P1 first stage free   P2 last load issued
  M0 MMA has the tile        M1 accumulator free   M2 first stage full   M3 tfull committed
  Mw cycles the MMA thread waited on full stages;  Ma1 cycles waiting for accumulator 1 (split)
  E0 epilogue has the tile   E1 tfull seen   E2 acc0 released  E3 acc1 released  E4 last store issued
  Ew cycles the epilogue waited for a free staging slot / C tile
Usage: python scripts/gemm_trace.py WORKLOAD [cfg]  (batched | batched-beta1 | gemm<n>, e.g. gemm8192)"""
import ctypes
import os
import sys

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
sys.path.insert(0, ROOT)
from paper_2504_07004_b200 import _lib  # noqa: E402

_lib.use_library(os.path.join(ROOT, "build", "exp", os.environ.get("CY_TRACE_LIB", "libcypress_gtrace.so")))
import torch  # noqa: E402

import paper_2504_07004_b200 as cy  # noqa: E402

w = sys.argv[1] if len(sys.argv) > 1 else "batched"
cfg = int(sys.argv[2]) if len(sys.argv) > 2 else -1
lib = _lib.load()
lib.cy_gemm_trace_read.argtypes = [ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_int]
g = torch.Generator(device="cuda").manual_seed(0)
cy.force_config(cfg)
if w.startswith("batched"):
    mk = lambda: torch.empty((64, 1024, 1024), device="cuda", dtype=torch.float16).uniform_(-1, 1, generator=g)  # noqa
    sets = [(mk(), mk(), mk()) for _ in range(2)]
    D = torch.empty((64, 1024, 1024), device="cuda", dtype=torch.float16)
    beta = 1.0 if w == "batched-beta1" else 0.0
    run = lambda i: cy.gemm_batched(sets[i % 2][0], sets[i % 2][1], sets[i % 2][2], 1.0, beta, out=D)  # noqa
else:
    sz = int(w[4:])  # gemm<n>: n^3
    mk = lambda: torch.empty((sz, sz), device="cuda", dtype=torch.float16).uniform_(-1, 1, generator=g)  # noqa
    sets = [(mk(), mk()) for _ in range(2)]
    D = torch.empty((sz, sz), device="cuda", dtype=torch.float16)
    run = lambda i: cy.gemm(sets[i % 2][0], sets[i % 2][1], out=D)  # noqa
buf = (ctypes.c_ulonglong * (64 * 16))()
for i in range(20):
    run(i)
torch.cuda.synchronize()
lib.cy_gemm_trace_read(buf, 1)  # clear
run(20)
torch.cuda.synchronize()
lib.cy_gemm_trace_read(buf, 0)
ev = [[buf[t * 16 + e] for e in range(16)] for t in range(64)]
t0 = min(x for row in ev for j, x in enumerate(row) if x and j not in (7, 13, 14))
print(f"{w} cfg {cy.last_kernel_info()}")
print("tile     P0     P1     P2 |     M0     M1     M2     M3     Mw    Ma1 |     E0     E1     E2     E3     E4     Ew")
for t, r in enumerate(ev):
    if not r[0] and not r[3]:
        continue
    rel = lambda j: (r[j] - t0) if r[j] else -1  # noqa
    print(f"{t:4d} {rel(0):6d} {rel(1):6d} {rel(2):6d} | {rel(3):6d} {rel(4):6d} {rel(5):6d} {rel(6):6d} {r[7]:6d} {r[14]:6d} | "
          f"{rel(8):6d} {rel(9):6d} {rel(10):6d} {rel(11):6d} {rel(12):6d} {r[13]:6d}")

# epilogue chunk timeline of the first tile (general chunk loop only): per warp and chunk, cycles
# (from the tile's tfull seen) at: load start, TMEM loaded, staging slot ready, store issued
lib.cy_gemm_etrace_read.argtypes = [ctypes.POINTER(ctypes.c_ulonglong)]
et = (ctypes.c_ulonglong * (8 * 8 * 8))()
lib.cy_gemm_etrace_read(et)
base = ev[0][9]
if base and any(et[i] for i in range(512)):
    print("epilogue chunks (cycles from tfull seen): warp q: load0 loaded slot st.shared-done fenced stored")
    for w_ in range(8):
        for q in range(8):
            v = [et[(w_ * 8 + q) * 8 + e] for e in range(6)]
            if any(v):
                print(f"  w{w_} q{q}: " + " ".join(f"{(x - base) if x else -1:6d}" for x in v))

# MMA issuer of the first tile (non-split accumulators only): per k-block, cycles from the tile's
# first stage full to (stage full seen, its MMAs issued)
lib.cy_gemm_mtrace_read.argtypes = [ctypes.POINTER(ctypes.c_ulonglong)]
mt = (ctypes.c_ulonglong * 256)()
lib.cy_gemm_mtrace_read(mt)
if mt[0]:
    b0 = mt[0]  # (event 0 of k-block 0)
    print("MMA issuer per k-block (cycles from the first full seen): loop_top full_seen issued committed")
    for kb in range(64):
        if not mt[4 * kb]:
            break
        print(f"  kb {kb:2d}: " + " ".join(f"{mt[4 * kb + e] - b0:7d}" for e in (2, 0, 1, 3)))
