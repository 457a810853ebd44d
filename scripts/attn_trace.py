"""Per-block event timeline of one attention CTA (build with -DCY_ATTN_TRACE into LIB.so).
python scripts/attn_trace.py LIB.so [b s causal]"""
import ctypes, sys, os
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch
from paper_2504_07004_b200 import _lib
_lib.LIB_PATH = os.path.abspath(sys.argv[1])
import paper_2504_07004_b200 as cy

b = int(sys.argv[2]) if len(sys.argv) > 2 else 2
s = int(sys.argv[3]) if len(sys.argv) > 3 else 8192
causal = len(sys.argv) > 4 and sys.argv[4] == "1"
Q, K, V = (torch.empty((b, 16, s, 128), device="cuda", dtype=torch.float16).uniform_(-1, 1) for _ in range(3))
for _ in range(5):
    cy.attention(Q, K, V, causal=causal)
torch.cuda.synchronize()
lib = _lib.load()
buf = (ctypes.c_ulonglong * (16 * 2 * 64))()
lib.cy_attn_trace.argtypes = [ctypes.c_void_p]
assert lib.cy_attn_trace(ctypes.cast(buf, ctypes.c_void_p)) == 0
T = [[[buf[(ev * 2 + t) * 64 + j] for j in range(64)] for t in range(2)] for ev in range(16)]
t0 = min(x for ev in range(8) for t in range(2) for x in T[ev][t] if x)
names = {0: "S_full", 1: "max_done", 2: "exp_done", 3: "P_ready", 4: "mma_Phalf", 5: "mma_Pfull", 6: "S_issued", 7: "mma_Vfull"}
print("j  " + "  ".join(f"{names[ev]}{t}" for ev in range(8) for t in range(2) if not (ev == 7 and t == 1)))
for j in range(0, 64):
    row = []
    for ev in range(8):
        for t in range(2):
            if ev == 7 and t == 1:
                continue
            v = T[ev][t][j]
            row.append(f"{(v - t0) if v else -1:>10d}")
    print(f"{j:2d} " + " ".join(row))
# per-block period and phase durations (steady state j = 8..55)
import statistics as st
def d(a, b, t, j0=8, j1=56, shift=0):
    return st.median(T[b][t][j + shift] - T[a][t][j] for j in range(j0, j1))
for t in range(2):
    per = st.median(T[0][t][j + 1] - T[0][t][j] for j in range(8, 56))
    print(f"tile {t}: period {per:.0f} | S_full->max_done {d(0, 1, t):.0f} | max->exp_done {d(1, 2, t):.0f} | "
          f"exp_done->P_ready {d(2, 3, t):.0f} | P_ready->mma_Pfull {d(3, 5, t):.0f} | mma_Pfull->S_issued(j+1) {d(5, 6, t, shift=1):.0f} | "
          f"S_issued(j+1)->S_full(j+1) {st.median(T[0][t][j + 1] - T[6][t][j + 1] for j in range(8, 56)):.0f}")

for t in range(2):
    print(f"tile {t}: S_full -> TMEM loads done {d(0, 11, t):.0f} | loads done -> max_done {d(11, 1, t):.0f}")
print("producer / MMA operand waits (cycles, j = 8..55 median):")
kf = st.median(T[10][0][j] - T[8][0][j] for j in range(8, 56))
vf = st.median(T[7][0][j] - T[9][0][j] for j in range(8, 56))
print(f"K_j: empty-wait done -> MMA sees full {kf:.0f} | V_j: empty-wait done -> MMA sees V full {vf:.0f}")
for j in range(8, 16):
    print(f"j={j}: Kempty {T[8][0][j]-t0} Kfull(mma) {T[10][0][j]-t0} Vempty {T[9][0][j]-t0} Vfull(mma) {T[7][0][j]-t0} "
          f"Phalf0 ready(mma) {T[4][0][j]-t0} Sissued1(j) {T[6][1][j]-t0}")
