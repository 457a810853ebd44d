"""cuBLAS (torch.matmul, informational comparator) vs ours at n^3: 1000 back-to-back launches over 2
rotating input sets, TFLOP/s and the SM clock sampled during the run (same harness as bench.py)."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch
import paper_2504_07004_b200 as cy
from bench import ClockSampler

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
sets = [(torch.empty((n, n), device="cuda", dtype=torch.float16).uniform_(-1, 1),
         torch.empty((n, n), device="cuda", dtype=torch.float16).uniform_(-1, 1)) for _ in range(2)]
d = torch.empty((n, n), device="cuda", dtype=torch.float16)
for name, fn in (("ours", lambda a, b: cy.gemm(a, b, out=d)), ("cublas", lambda a, b: torch.matmul(a, b, out=d)),
                 ("ours", lambda a, b: cy.gemm(a, b, out=d)), ("cublas", lambda a, b: torch.matmul(a, b, out=d))):
    for i in range(10):
        fn(*sets[i % 2])
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(0) as cs:
        e0.record()
        for i in range(1000):
            fn(*sets[i % 2])
        e1.record()
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 1000
    s = cs.summary()
    print(f"{name:6s} {2 * n ** 3 / ms / 1e9:7.1f} TFLOP/s  sm_mhz {s['sm_mhz']}  power_max {s.get('power_w_max')}  "
          f"per SM-GHz {2 * n ** 3 / ms / 1e9 / 148 / (s['sm_mhz'] / 1000):.2f} TF", flush=True)
