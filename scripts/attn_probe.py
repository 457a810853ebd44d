"""Attention throughput: ours vs torch SDPA (informational comparator), FA benchmark shapes."""
import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch
from paper_2504_07004_b200 import _lib
if os.environ.get("CY_EXP_LIB"):  # A/B against an experiment build
    _lib.use_library(os.path.abspath(os.environ["CY_EXP_LIB"]))
import paper_2504_07004_b200 as cy

def bench(fn, iters=30):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / iters

h, d = 16, 128
for causal in (False, True):
    for s in (1024, 2048, 4096, 8192, 16384):
        bsz = max(1, 16384 // s)
        g = torch.Generator(device="cuda").manual_seed(0)
        Q, K, V = (torch.empty((bsz, h, s, d), device="cuda", dtype=torch.float16).uniform_(-1, 1, generator=g) for _ in range(3))
        flops = 4.0 * bsz * h * s * s * d / (2 if causal else 1)
        ms = bench(lambda: cy.attention(Q, K, V, causal=causal))
        ms_t = bench(lambda: torch.nn.functional.scaled_dot_product_attention(Q, K, V, is_causal=causal))
        print(f"causal={causal} b={bsz} h={h} s={s}: ours {ms*1e3:8.1f} us {flops/ms/1e9:7.1f} TF | sdpa {ms_t*1e3:8.1f} us {flops/ms_t/1e9:7.1f} TF", flush=True)
