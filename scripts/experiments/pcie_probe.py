"""PCIe copy rates on this box (pinned host memory): H2D alone, D2H alone, both at once, and H2D in
2 / 4 concurrent chunks.  python scripts/experiments/pcie_probe.py"""
import torch

MB = 1 << 20
h_in = torch.empty(256 * MB, dtype=torch.uint8).pin_memory()
h_out = torch.empty(128 * MB, dtype=torch.uint8).pin_memory()
d_in = torch.empty(256 * MB, dtype=torch.uint8, device="cuda")
d_out = torch.empty(128 * MB, dtype=torch.uint8, device="cuda")
s1, s2, s3 = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def h2d():
    with torch.cuda.stream(s1):
        d_in.copy_(h_in, non_blocking=True)


def d2h():
    with torch.cuda.stream(s2):
        h_out.copy_(d_out, non_blocking=True)


def both():
    h2d()
    d2h()


def h2d_chunks(c):
    def f():
        n = h_in.numel() // c
        for i in range(c):
            with torch.cuda.stream((s1, s3)[i % 2]):
                d_in[i * n:(i + 1) * n].copy_(h_in[i * n:(i + 1) * n], non_blocking=True)
    return f


t = timed(h2d)
print(f"H2D 256 MiB alone     {t:6.3f} ms  {256 * MB / t / 1e6:6.1f} GB/s")
t = timed(d2h)
print(f"D2H 128 MiB alone     {t:6.3f} ms  {128 * MB / t / 1e6:6.1f} GB/s")
t = timed(both)
print(f"H2D 256 + D2H 128     {t:6.3f} ms  (H2D alone would be {256 * MB / 55e6:.3f} ms at 55 GB/s)")
for c in (2, 4):
    t = timed(h2d_chunks(c))
    print(f"H2D in {c} chunks / 2 streams {t:6.3f} ms  {256 * MB / t / 1e6:6.1f} GB/s")
