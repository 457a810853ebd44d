"""Attention throughput at two shapes (env knobs such as CY_ATTN_EMU are read by the library)."""
import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
import torch
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

tag = os.environ.get("CY_ATTN_EMU", "0")
for causal, bsz, s in ((False, 2, 8192), (False, 8, 2048), (True, 1, 16384), (True, 4, 4096)):
    g = torch.Generator(device="cuda").manual_seed(0)
    Q, K, V = (torch.empty((bsz, 16, s, 128), device="cuda", dtype=torch.float16).uniform_(-1, 1, generator=g) for _ in range(3))
    flops = 4.0 * bsz * 16 * s * s * 128 / (2 if causal else 1)
    ms = bench(lambda: cy.attention(Q, K, V, causal=causal))
    print(f"emu={tag} causal={causal} b={bsz} s={s}: {ms*1e3:8.1f} us {flops/ms/1e9:7.1f} TF", flush=True)
