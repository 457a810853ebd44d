"""Shared timing helper for the probes: device time per launch, launches queued behind a long kernel."""
import torch


def dev_time(fn, reps=100):
    for _ in range(10):
        fn()
    big = torch.empty((8192, 8192), device="cuda", dtype=torch.float16)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.matmul(big, big)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3
