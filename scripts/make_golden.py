"""Write tests/golden/*.json fixtures.  Calls only oracle/ (and synth/ for inputs).

The paper prints no worked numeric example (its figures are stripped),
so the fixtures are (a) the SPEC's stated examples and (b) small
integer-valued cases whose expected values the script cross-checks against exact
int64 arithmetic before writing.  Run:  python scripts/make_golden.py
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import synth  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")


def dec(bits):
    return np.asarray(bits, np.uint16).view(np.float16).astype(np.float64)


def write(name, obj):
    with open(os.path.join(OUT, name), "w") as f:
        json.dump(obj, f, separators=(",", ":"))
        f.write("\n")


def main():
    os.makedirs(OUT, exist_ok=True)
    # (1) SPEC S:577: integer GEMM equals the triple loop exactly (fp16 inputs, 16x24x40).
    A, B, C = synth.gemm_inputs(16, 24, 40, seed=synth.seed_for(0, 99), kind="int", with_c=True)
    D = oracle.gemm("f16", A, B, C, alpha=1.0, beta=1.0)
    exact = dec(A).astype(np.int64) @ dec(B).astype(np.int64) + dec(C).astype(np.int64)
    assert np.array_equal(D, exact.astype(np.float64))
    write("gemm_int_16x24x40.json", {
        "cite": "GEMM D = alpha*A.B + beta*C (P:125, P:1513; alpha/beta R4); SPEC S:577 integer exactness",
        "op": "gemm", "dtype": "f16", "alpha": 1.0, "beta": 1.0,
        "A": A.tolist(), "B": B.tolist(), "C": C.tolist(),
        "D_bits": oracle.encode("f16", D).tolist()})
    # (2) SPEC S:579: A = all-ones 64x64 -> y(i) = 64.
    ones = synth.f64_to_bits(np.ones((64, 64)), "f16")
    y = oracle.rowsum("f16", ones)
    assert np.all(y == 64.0)
    write("rowsum_ones_64x64.json", {
        "cite": "y(i) = sum_k A(i,k) (P:1579); SPEC S:579 all-ones example",
        "op": "rowsum", "dtype": "f16", "A": ones.tolist(), "y": y.tolist()})
    # (3) K = 1 outer product with a rounding tie: D = RN(a*b) (R7), bf16.
    a = np.array([[1 + 2 ** -7], [3.0], [-1.5]])
    b = np.array([[1 + 2 ** -7, 1.0 + 2 ** -6]])
    A3 = synth.f64_to_bits(a, "bf16")
    B3 = synth.f64_to_bits(b, "bf16")
    D3 = oracle.gemm("bf16", A3, B3)
    write("gemm_bf16_k1_ties.json", {
        "cite": "K=1 GEMM is one exact product + one RN-even rounding (R7)",
        "op": "gemm", "dtype": "bf16", "alpha": 1.0, "beta": 0.0,
        "A": A3.tolist(), "B": B3.tolist(), "C": None,
        "D_bits": oracle.encode("bf16", D3).tolist()})
    print("wrote fixtures to", OUT)


if __name__ == "__main__":
    main()
