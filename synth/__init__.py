"""Seeded synthetic input generators shared by tests, bench and smoke.

This module holds NO arithmetic of the method (no products, sums or
rounding of results): it only draws inputs.  Both the oracle side and the
CUDA side consume what it returns; neither imports the other.

Recipe (reading R9 of the paper's unspecified
"values drawn from the same random distribution"):

* generator: ``numpy.random.Generator(PCG64(seed))``, one stream per tensor;
* seed: ``20250407 + 100 * config_id + s`` (``seed_for``);
* float inputs: uniform[-1, 1) in float64, then rounded to the 16-bit input
  format (fp16 via numpy's IEEE binary16 cast, bf16 via float32 then
  round-to-nearest-even on the top 16 bits) -- the rounded values ARE the
  inputs, so there is no rounding of the method here;
* integer-valued inputs: integers in [-2, 2] (``integers``), exactly
  representable in both formats, so every partial sum of a K <= 2^21 GEMM is
  an integer below 2^24 and fp32 accumulation is exact (reading R11).

All returns are numpy ``uint16`` arrays of raw bit patterns.
"""
from __future__ import annotations

import numpy as np

BASE_SEED = 20250407


def seed_for(config_id: int, s: int = 0) -> int:
    return BASE_SEED + 100 * int(config_id) + int(s)


def _rng(seed):
    return np.random.Generator(np.random.PCG64(seed))


def f64_to_bits(x: np.ndarray, dtype: str) -> np.ndarray:
    """Cast float64 values that are the chosen inputs to 16-bit patterns."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    if dtype in ("f16", "fp16", "float16"):
        return x.astype(np.float16).view(np.uint16)
    if dtype in ("bf16", "bfloat16"):
        f = x.astype(np.float32).view(np.uint32).astype(np.uint64)
        # round-to-nearest-even on the low 16 bits of the float32 pattern
        lsb = (f >> 16) & 1
        r = (f + 0x7FFF + lsb) >> 16
        nan = np.isnan(x)
        r = np.where(nan, 0x7FC0, r)
        return r.astype(np.uint16)
    raise ValueError(dtype)


_CHUNK = 1 << 24


def uniform(shape, seed: int, dtype: str = "f16", lo: float = -1.0, hi: float = 1.0) -> np.ndarray:
    """uniform[lo, hi) drawn in float64, then cast to the 16-bit input format.
    Large arrays are drawn in sequential chunks of one stream (same values as one draw)."""
    rng = _rng(seed)
    total = int(np.prod(shape))
    if total <= _CHUNK:
        return f64_to_bits(rng.uniform(lo, hi, size=shape), dtype)
    out = np.empty(total, dtype=np.uint16)
    for s in range(0, total, _CHUNK):
        e = min(total, s + _CHUNK)
        out[s:e] = f64_to_bits(rng.uniform(lo, hi, size=e - s), dtype)
    return out.reshape(shape)


def integers(shape, seed: int, dtype: str = "f16", lo: int = -2, hi: int = 2) -> np.ndarray:
    """Integer-valued inputs in [lo, hi] (inclusive), exact in fp16/bf16."""
    x = _rng(seed).integers(lo, hi + 1, size=shape).astype(np.float64)
    return f64_to_bits(x, dtype)


def gemm_inputs(m, n, k, seed, dtype="f16", kind="uniform", with_c=False, batch=None):
    """A (m x k), B (k x n)[, C (m x n)] drawn in the order A, B, C from seeds seed, seed+1, seed+2."""
    gen = uniform if kind == "uniform" else integers
    pre = () if batch is None else (batch,)
    A = gen(pre + (m, k), seed, dtype)
    B = gen(pre + (k, n), seed + 1, dtype)
    C = gen(pre + (m, n), seed + 2, dtype) if with_c else None
    return A, B, C


def dual_inputs(m, n, k, seed, dtype="f16", kind="uniform", with_c=False):
    """A, B0, B1[, C0, C1] from seeds seed .. seed+4."""
    gen = uniform if kind == "uniform" else integers
    A = gen((m, k), seed, dtype)
    B0 = gen((k, n), seed + 1, dtype)
    B1 = gen((k, n), seed + 2, dtype)
    C0 = gen((m, n), seed + 3, dtype) if with_c else None
    C1 = gen((m, n), seed + 4, dtype) if with_c else None
    return A, B0, B1, C0, C1


def sample_rows(m: int, tile: int = 128, n_random: int = 64, seed: int = 7) -> np.ndarray:
    """Rows the oracle recomputes one by one at full size: the first and last
    row of every ``tile``-row block plus ``n_random`` random rows (sorted, unique)."""
    first = np.arange(0, m, tile)
    last = np.minimum(first + tile - 1, m - 1)
    rnd = _rng(seed).integers(0, m, size=min(n_random, m)) if m else np.array([], dtype=np.int64)
    return np.unique(np.concatenate([first, last, rnd]).astype(np.int64))
