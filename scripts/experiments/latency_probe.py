"""Small-shape latency: host time per call (wall) and device time per launch (events), ours vs torch.matmul."""
import sys, os, time
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
import torch
import paper_2504_07004_b200 as cy

for n in (256, 512, 1024, 2048):
    a = torch.empty((n, n), device="cuda", dtype=torch.float16).uniform_(-1, 1)
    b = torch.empty((n, n), device="cuda", dtype=torch.float16).uniform_(-1, 1)
    d = torch.empty((n, n), device="cuda", dtype=torch.float16)
    for name, fn in (("ours", lambda: cy.gemm(a, b, out=d)), ("torch", lambda: torch.matmul(a, b, out=d))):
        for _ in range(50):
            fn()
        torch.cuda.synchronize()
        N = 2000
        t0 = time.perf_counter()
        for _ in range(N):
            fn()
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        # device time per launch, launches queued behind a long kernel so the host is not the limit
        big = torch.empty((8192, 8192), device="cuda", dtype=torch.float16)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.matmul(big, big)  # keeps the GPU busy while the launches queue
        e0.record()
        for _ in range(200):
            fn()
        e1.record()
        torch.cuda.synchronize()
        dev = e0.elapsed_time(e1) / 200
        print(f"n={n:5d} {name:5s}: host {1e6 * (t1 - t0) / N:6.2f} us/call, wall {1e6 * (t2 - t0) / N:6.2f} us/call, "
              f"device {1e3 * dev:6.2f} us/launch -> {2 * n ** 3 / (dev * 1e-3) / 1e12:7.1f} TFLOP/s", flush=True)
