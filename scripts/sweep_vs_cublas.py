"""Square fp16 GEMM sweep (BASELINE configs[1]): ours vs torch.matmul (cuBLAS, informational), device
time per launch with launches queued back to back, 2 rotating input sets, uniform[-1,1]."""
import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch
import paper_2504_07004_b200 as cy


def dev_time(fn, reps):
    for i in range(5):
        fn(i)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(reps):
        fn(i)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


for n in (1024, 2048, 4096, 8192, 16384):
    sets = [(torch.empty((n, n), device="cuda", dtype=torch.float16).uniform_(-1, 1),
             torch.empty((n, n), device="cuda", dtype=torch.float16).uniform_(-1, 1)) for _ in range(2)]
    d = torch.empty((n, n), device="cuda", dtype=torch.float16)
    reps = max(20, min(2000, int(2e13 / (2 * n ** 3))))
    fl = 2.0 * n ** 3
    res = []
    for r in range(2):
        t_ours = dev_time(lambda i: cy.gemm(*sets[i % 2], out=d), reps)
        t_cub = dev_time(lambda i: torch.matmul(*sets[i % 2], out=d), reps)
        res.append((t_ours, t_cub))
    t_ours = min(x[0] for x in res)
    t_cub = min(x[1] for x in res)
    print(f"n={n}: ours {t_ours:9.2f} us {fl / t_ours / 1e6:7.1f} TF | cuBLAS {t_cub:9.2f} us {fl / t_cub / 1e6:7.1f} TF | "
          f"ratio {t_cub / t_ours:.3f}", flush=True)
