"""Fast GPU sanity sweep: every config x a few shapes, integer inputs, prints mismatches.
Usage (GPU box): python scripts/quick_check.py [cfg ...]"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "..", "tests"))

import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2504_07004_b200 as cy  # noqa: E402
import synth  # noqa: E402
from gpu_util import to_bits, to_dev  # noqa: E402


def report(tag, got, want):
    bad = (got != want)
    print(f"{tag}: {'OK' if not bad.any() else f'MISMATCH {bad.sum()}/{bad.size}'}", flush=True)
    if bad.any():
        idx = np.argwhere(bad)[:4]
        for i in idx:
            i = tuple(i)
            print("   ", i, got[i].view(np.float16) if got.dtype == np.uint16 else got[i],
                  want[i].view(np.float16) if want.dtype == np.uint16 else want[i], flush=True)


cfgs = [int(c) for c in sys.argv[1:]] or list(range(cy.num_configs()))
print(torch.cuda.get_device_name(0), "configs", [cy.config_info(c) for c in cfgs], flush=True)
for cfg in cfgs:
    cy.force_config(cfg)
    for (m, n, k) in [(128, 64, 64), (256, 256, 64), (256, 256, 256), (300, 520, 200), (1000, 1023, 129)]:
        A, B, _ = synth.gemm_inputs(m, n, k, seed=1, kind="int")
        t0 = time.time()
        D = cy.gemm(to_dev(A, "f16"), to_dev(B, "f16"))
        torch.cuda.synchronize()
        report(f"cfg{cfg} int {m}x{n}x{k} ({time.time() - t0:.2f}s)", to_bits(D),
               oracle.encode("f16", oracle.gemm("f16", A, B)))
    k = 128
    _, B, _ = synth.gemm_inputs(k, 256, k, seed=2)
    I = synth.f64_to_bits(np.eye(k), "f16")
    D = cy.gemm(to_dev(I, "f16"), to_dev(B, "f16"))
    torch.cuda.synchronize()
    report(f"cfg{cfg} identity", to_bits(D), B)
cy.force_config(-1)
for cfg in [-1, 0, 1, 3]:
    cy.force_config(cfg)
    A, B0, B1, _, _ = synth.dual_inputs(300, 264, 200, seed=3, kind="int")
    d0, d1 = cy.dual_gemm(to_dev(A, "f16"), to_dev(B0, "f16"), to_dev(B1, "f16"), mode="pair")
    torch.cuda.synchronize()
    r0, r1 = oracle.dual_gemm("f16", "pair", A, B0, B1)
    report(f"dual pair cfg{cfg}", to_bits(d0), oracle.encode("f16", r0))
    report(f"dual pair D1 cfg{cfg}", to_bits(d1), oracle.encode("f16", r1))
    ds = cy.dual_gemm(to_dev(A, "f16"), to_dev(B0, "f16"), to_dev(B1, "f16"), mode="sum")
    torch.cuda.synchronize()
    report(f"dual sum cfg{cfg}", to_bits(ds), oracle.encode("f16", oracle.dual_gemm("f16", "sum", A, B0, B1)))
    A, B, _ = synth.gemm_inputs(700, 300, 513, seed=4, kind="int")
    D, y = cy.gemm_rowreduce(to_dev(A, "f16"), to_dev(B, "f16"))
    torch.cuda.synchronize()
    report(f"rowreduce D cfg{cfg}", to_bits(D), oracle.encode("f16", oracle.gemm("f16", A, B)))
    report(f"rowreduce y cfg{cfg}", y.cpu().numpy().astype(np.float64), oracle.rowsum("f16", A))
cy.force_config(-1)
# speed probe
for n in (4096, 8192):
    a = torch.randn(n, n, device="cuda", dtype=torch.float16)
    b = torch.randn(n, n, device="cuda", dtype=torch.float16)
    for cfg in (0, 1, 2):
        cy.force_config(cfg)
        for _ in range(3):
            cy.gemm(a, b)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            cy.gemm(a, b)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
        print(f"n={n} cfg{cfg}: {ms:.3f} ms  {2 * n ** 3 / ms / 1e9:.1f} TFLOP/s", flush=True)
    e0.record()
    for _ in range(10):
        torch.matmul(a, b)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"n={n} torch.matmul: {ms:.3f} ms  {2 * n ** 3 / ms / 1e9:.1f} TFLOP/s", flush=True)
