"""A/B attention throughput of library builds: python scripts/attn_ab.py LIB.so [LIB2.so ...]
(each build is run in its own process by the caller; env knobs such as CY_ATTN_EMU are read per call)."""
import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
import torch
from paper_2504_07004_b200 import _lib
_lib.LIB_PATH = os.path.abspath(sys.argv[1])
import paper_2504_07004_b200 as cy


def bench(fn, iters=40):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / iters


tag = os.path.basename(sys.argv[1]) + " emu=" + os.environ.get("CY_ATTN_EMU", "0")
out = []
for causal, bsz, s in ((False, 2, 8192), (False, 8, 2048), (True, 1, 16384), (True, 4, 4096)):
    g = torch.Generator(device="cuda").manual_seed(0)
    Q, K, V = (torch.empty((bsz, 16, s, 128), device="cuda", dtype=torch.float16).uniform_(-1, 1, generator=g)
               for _ in range(3))
    flops = 4.0 * bsz * 16 * s * s * 128 / (2 if causal else 1)
    ms = bench(lambda: cy.attention(Q, K, V, causal=causal))
    out.append(f"{'c' if causal else 'n'}{bsz}x{s} {flops / ms / 1e9:6.0f}")
print(f"{tag:22s} " + "  ".join(out), flush=True)
