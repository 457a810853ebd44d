"""Helpers shared by the -m gpu parity tests (marshalling and comparison only)."""
import numpy as np

import oracle

TORCH_DT = {"f16": "float16", "bf16": "bfloat16"}


def to_dev(bits, dtype, device="cuda"):
    """Upload 16-bit patterns.  2-D matrices get their row stride padded to a multiple of 8
    elements (the TMA 16-byte rule) and are returned as a [:, :cols] view."""
    import torch

    bits = np.ascontiguousarray(bits)
    if bits.ndim == 2 and bits.shape[1] % 8:
        cols = bits.shape[1]
        padded = np.zeros((bits.shape[0], (cols + 7) // 8 * 8), np.uint16)
        padded[:, :cols] = bits
        t = torch.from_numpy(padded.view(np.int16)).view(getattr(torch, TORCH_DT[dtype])).to(device)
        return t[:, :cols]
    t = torch.from_numpy(bits.view(np.int16))
    return t.view(getattr(torch, TORCH_DT[dtype])).to(device)


def to_bits(t):
    import torch

    return t.detach().contiguous().view(torch.int16).cpu().numpy().view(np.uint16)


def decode(bits, dtype):
    bits = np.asarray(bits, dtype=np.uint16)
    if dtype == "f16":
        return bits.view(np.float16).astype(np.float64)
    return (bits.astype(np.uint32) << 16).view(np.float32).astype(np.float64)


def assert_within_tol(D_bits, D_ref, k, dtype, sum_terms=1, what=""):
    """BASELINE.json north_star: |D - D_ref| <= 2^-8 |D_ref| + 1e-3 sqrt(K) per element
    (sqrt(2K) for dual SUM)."""
    D = decode(D_bits, dtype)
    tol = oracle.tolerance(D_ref, k, sum_terms)
    err = np.abs(D - D_ref)
    bad = ~(err <= tol)
    if bad.any():
        idx = np.argwhere(bad)[:5]
        raise AssertionError(f"{what}: {bad.sum()} / {bad.size} elements out of tolerance; first "
                             f"{[(tuple(i), D[tuple(i)], D_ref[tuple(i)]) for i in idx]}")
    return float((err / np.maximum(tol, 1e-30)).max()) if err.size else 0.0


def assert_bits_equal(got, want, what=""):
    got = np.asarray(got)
    want = np.asarray(want)
    assert got.shape == want.shape, (what, got.shape, want.shape)
    neq = got != want
    if neq.any():
        idx = np.argwhere(neq)[:5]
        raise AssertionError(f"{what}: {neq.sum()} / {neq.size} elements differ; first "
                             f"{[(tuple(i), hex(got[tuple(i)]), hex(want[tuple(i)])) for i in idx]}")
