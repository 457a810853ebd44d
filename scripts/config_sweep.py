"""Time every GEMM config on a set of shapes (uniform fp16), print a table + the heuristic's pick."""
import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch
import paper_2504_07004_b200 as cy

shapes = [(1, 1024, 1024, 1024), (1, 2048, 2048, 2048), (1, 4096, 4096, 4096), (1, 8192, 8192, 8192),
          (1, 16384, 16384, 16384), (64, 1024, 1024, 1024), (8, 1024, 1024, 1024), (16, 1024, 1024, 1024),
          (1, 1024, 8192, 8192), (1, 8192, 8192, 1024), (1, 65536, 8192, 8192), (1, 4096, 4096, 1024)]
g = torch.Generator(device="cuda").manual_seed(0)
ncfg = cy.num_configs()
print("shape".ljust(26), " ".join(f"cfg{c}:{cy.config_info(c)['tile_m']}x{cy.config_info(c)['tile_n']}".rjust(14) for c in range(ncfg)), "  heuristic")
for (L, m, n, k) in shapes:
    A = torch.empty((L, m, k), device="cuda", dtype=torch.float16).uniform_(-1, 1, generator=g)
    B = torch.empty((L, k, n), device="cuda", dtype=torch.float16).uniform_(-1, 1, generator=g)
    D = torch.empty((L, m, n), device="cuda", dtype=torch.float16)
    flops = 2.0 * L * m * n * k
    iters = max(5, min(300, int(3e13 / flops)))
    res = []
    for c in list(range(ncfg)) + [-1]:
        cy.force_config(c)
        fn = (lambda: cy.gemm(A[0], B[0], out=D[0])) if L == 1 else (lambda: cy.gemm_batched(A, B, out=D))
        for _ in range(5):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(iters):
            fn()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / iters
        res.append((flops / ms / 1e9, cy.last_config()))
    cy.force_config(-1)
    best = max(range(ncfg), key=lambda i: res[i][0])
    print(f"{L}x{m}x{n}x{k}".ljust(26), " ".join(f"{r[0]:14.1f}" for r in res[:ncfg]),
          f"  pick cfg{res[-1][1]} {res[-1][0]:.1f} (best cfg{best})", flush=True)
