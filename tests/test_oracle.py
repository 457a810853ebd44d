"""Pins for the fp64 oracle (oracle/oracle.c) against things other than itself.

Each test pins the oracle to the mathematics or to an independent library:
* codecs vs numpy.float16 / float32 bit views over all 65536 patterns and
  constructed round-to-nearest-even ties (R7);
* GEMM / dual / row-sum vs exact rational brute force (Python Fractions) on
  tiny shapes, within the fp64 summation bound k*2^-53*sum|a||b|;
* special cases that reduce to a library routine (numpy.matmul in float64,
  exact int64 matmul for integer inputs);
* closed forms (identity, permutation, diagonal powers of two, all-ones);
* the paper's definitions' invariants (dual SUM with B1 = 0 is a GEMM --
  SPEC S:578; all-ones row sum = K -- SPEC S:579; y independent of B).
A plausible mistake (dropped term, wrong sign, transposed operand, wrong
index, double rounding) fails at least one of these.
"""
from fractions import Fraction

import numpy as np
import pytest
import torch

import synth

pytestmark = []


# --------------------------------------------------------------------------- codecs

def test_half_decode_all_patterns(orc):
    bits = np.arange(65536, dtype=np.uint32).astype(np.uint16)
    got = orc.decode("f16", bits)
    ref = bits.view(np.float16).astype(np.float64)
    nan = np.isnan(ref)
    assert np.array_equal(np.isnan(got), nan)
    assert np.array_equal(got[~nan], ref[~nan])
    # signed zeros preserved
    assert np.signbit(got[0x8000]) and not np.signbit(got[0])


def test_bf16_decode_all_patterns(orc):
    bits = np.arange(65536, dtype=np.uint32)
    got = orc.decode("bf16", bits.astype(np.uint16))
    ref = (bits << 16).astype(np.uint32).view(np.float32).astype(np.float64)
    nan = np.isnan(ref)
    assert np.array_equal(np.isnan(got), nan)
    assert np.array_equal(got[~nan], ref[~nan])


def _half_ties():
    """Exact midpoints between every pair of adjacent finite fp16 values (>= 0),
    plus the overflow midpoint 65520 (halfway between 65504 and 2^16)."""
    v = np.arange(0, 0x7C00, dtype=np.uint16).view(np.float16).astype(np.float64)
    mids = (v[:-1] + v[1:]) / 2.0  # exact in fp64
    return np.concatenate([mids, [65520.0]])


def test_half_encode_vs_numpy(orc):
    rng = np.random.default_rng(1)
    x = np.concatenate([
        rng.uniform(-1, 1, 200000),
        rng.standard_normal(100000) * 1e3,
        rng.uniform(-7e4, 7e4, 50000),          # includes overflow
        rng.uniform(-1e-5, 1e-5, 50000),        # subnormals
        rng.uniform(-6.2e-5, 6.2e-5, 50000),    # subnormal/normal boundary
        _half_ties(), -_half_ties(),
        [0.0, -0.0, np.inf, -np.inf, 65504.0, 65519.99, 65520.0, 2.0 ** -24, 2.0 ** -25,
         3 * 2.0 ** -26, 2.0 ** -14 - 2.0 ** -25],
    ])
    got = orc.encode("f16", x)
    ref = x.astype(np.float16).view(np.uint16)
    assert np.array_equal(got, ref)


def test_half_encode_ties_to_even(orc):
    # 1 + 2^-11 is halfway between 1 and 1+2^-10: ties to even -> 1.0 (0x3C00)
    # 1 + 3*2^-11 is halfway between 1+2^-10 and 1+2^-9 -> 1+2^-9 (0x3C02)
    got = orc.encode("f16", np.array([1 + 2.0 ** -11, 1 + 3 * 2.0 ** -11, 2049.0, 2051.0]))
    assert list(got) == [0x3C00, 0x3C02, 0x6800, 0x6802]
    # NaN -> quiet NaN
    assert (orc.encode("f16", np.array([np.nan]))[0] & 0x7C00) == 0x7C00


def test_bf16_encode_vs_torch(orc):
    rng = np.random.default_rng(2)
    # float32-exact inputs so torch's float32 -> bf16 RN-even is a single rounding
    x32 = np.concatenate([
        rng.uniform(-1, 1, 200000), rng.standard_normal(100000) * 1e30,
        rng.uniform(-1e-38, 1e-38, 50000),
    ]).astype(np.float32)
    # exact midpoints between adjacent bf16 values
    b = np.arange(0, 0x7F80, 7, dtype=np.uint32)
    lo = (b << 16).view(np.float32).astype(np.float64)
    hi = ((b + 1) << 16).view(np.float32).astype(np.float64)
    mids = ((lo + hi) / 2).astype(np.float32)  # exact: 9 significant bits
    x32 = np.concatenate([x32, mids, -mids])
    got = orc.encode("bf16", x32.astype(np.float64))
    ref = torch.from_numpy(x32).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(got, ref)
    # overflow: max bf16 is (2-2^-7)*2^127; the midpoint to 2^128 rounds to inf
    big = np.array([(2 - 2.0 ** -8) * 2.0 ** 127, (2 - 2.0 ** -7) * 2.0 ** 127])
    assert list(orc.encode("bf16", big)) == [0x7F80, 0x7F7F]


# --------------------------------------------------------------------------- GEMM

def _frac(dtype, bits):
    return [[Fraction(float(v)) for v in row] for row in np_decode(dtype, bits)]


def np_decode(dtype, bits):
    """Independent decoder (numpy views), not the oracle's."""
    bits = np.asarray(bits, dtype=np.uint16)
    if dtype == "f16":
        return bits.view(np.float16).astype(np.float64)
    return (bits.astype(np.uint32) << 16).view(np.float32).astype(np.float64)


def _exact_gemm(dtype, A, B, C, alpha, beta):
    a, b = _frac(dtype, A), _frac(dtype, B)
    (m, k), n = A.shape, B.shape[1]
    c = _frac(dtype, C) if C is not None else None
    D, S = [], []
    for i in range(m):
        drow, srow = [], []
        for j in range(n):
            s = sum((a[i][kk] * b[kk][j] for kk in range(k)), Fraction(0))
            bound = sum((abs(a[i][kk] * b[kk][j]) for kk in range(k)), Fraction(0))
            d = Fraction(alpha) * s + (Fraction(beta) * c[i][j] if beta != 0 else 0)
            drow.append(d)
            srow.append(bound)
        D.append(drow)
        S.append(srow)
    return D, S


@pytest.mark.parametrize("dtype", ["f16", "bf16"])
@pytest.mark.parametrize("shape", [(1, 1, 1), (3, 5, 7), (6, 4, 8), (5, 7, 1), (2, 3, 0)])
@pytest.mark.parametrize("ab", [(1.0, 0.0), (0.5, -2.0), (-1.25, 0.75)])
def test_gemm_vs_exact_rationals(orc, dtype, shape, ab):
    m, n, k = shape
    alpha, beta = ab
    A, B, C = synth.gemm_inputs(m, n, k, seed=11 + m + 10 * n + 100 * k, dtype=dtype, with_c=True)
    D = orc.gemm(dtype, A, B, C, alpha, beta)
    E, S = _exact_gemm(dtype, A, B, C, alpha, beta)
    for i in range(m):
        for j in range(n):
            err = abs(Fraction(D[i, j]) - E[i][j])
            # fp64: k-term sum error <= k*2^-53*sum|ab|, then alpha*, +beta*c: 3 more roundings
            bound = (k + 3) * Fraction(2) ** -53 * (abs(Fraction(alpha)) * S[i][j] + abs(E[i][j]) + 1)
            assert err <= bound, (i, j, float(err), float(bound))


def test_gemm_vs_numpy_matmul(orc):
    m, n, k = 67, 45, 130
    A, B, _ = synth.gemm_inputs(m, n, k, seed=5)
    D = orc.gemm("f16", A, B)
    ref = np_decode("f16", A) @ np_decode("f16", B)
    assert np.allclose(D, ref, rtol=1e-13, atol=1e-13)


@pytest.mark.parametrize("dtype", ["f16", "bf16"])
def test_gemm_integer_exact_vs_int64(orc, dtype):
    m, n, k = 40, 33, 517
    A, B, C = synth.gemm_inputs(m, n, k, seed=9, dtype=dtype, kind="int", with_c=True)
    ai = np_decode(dtype, A).astype(np.int64)
    bi = np_decode(dtype, B).astype(np.int64)
    ci = np_decode(dtype, C).astype(np.int64)
    D = orc.gemm(dtype, A, B, C, alpha=2.0, beta=-3.0)
    assert np.array_equal(D, (2 * (ai @ bi) - 3 * ci).astype(np.float64))


def test_gemm_strided_leading_dims(orc):
    A, B, _ = synth.gemm_inputs(20, 24, 40, seed=3)
    Abig = np.zeros((20, 56), np.uint16)
    Abig[:, :40] = A
    Bbig = np.zeros((40, 32), np.uint16)
    Bbig[:, :24] = B
    assert np.array_equal(orc.gemm("f16", Abig[:, :40], Bbig[:, :24]), orc.gemm("f16", A, B))


def test_gemm_row_subset(orc):
    A, B, C = synth.gemm_inputs(50, 20, 30, seed=4, with_c=True)
    full = orc.gemm("f16", A, B, C, 1.5, 0.5)
    rows = np.array([0, 7, 49, 13])
    assert np.array_equal(orc.gemm("f16", A, B, C, 1.5, 0.5, rows=rows), full[rows])


def test_gemm_closed_forms(orc):
    k = 64
    I = synth.f64_to_bits(np.eye(k), "f16")
    _, B, _ = synth.gemm_inputs(k, 48, k, seed=21)
    A, _, _ = synth.gemm_inputs(37, 48, k, seed=22)
    # A = I  =>  D = B ;  B = I  =>  D = A  (exact)
    assert np.array_equal(orc.encode("f16", orc.gemm("f16", I, B)), B)
    assert np.array_equal(orc.encode("f16", orc.gemm("f16", A, I)), A)
    # row permutation P: D = P.B ; column permutation Q: D = A.Q
    perm = np.random.default_rng(0).permutation(k)
    P = synth.f64_to_bits(np.eye(k)[perm], "f16")
    assert np.array_equal(orc.encode("f16", orc.gemm("f16", P, B)), B[perm])
    Q = synth.f64_to_bits(np.eye(k)[:, perm], "f16")
    assert np.array_equal(orc.encode("f16", orc.gemm("f16", A, Q)), A[:, perm])
    # diag(2^e): rows of B scaled exactly
    e = np.arange(k) % 7 - 3
    Dg = synth.f64_to_bits(np.diag(2.0 ** e), "f16")
    assert np.array_equal(orc.gemm("f16", Dg, B), np_decode("f16", B) * (2.0 ** e)[:, None])
    # all-ones: D = K
    ones_a = synth.f64_to_bits(np.ones((8, 300)), "f16")
    ones_b = synth.f64_to_bits(np.ones((300, 9)), "f16")
    assert np.all(orc.gemm("f16", ones_a, ones_b) == 300.0)


def test_gemm_alpha_beta_special(orc):
    A, B, C = synth.gemm_inputs(16, 24, 32, seed=31, with_c=True)
    # alpha = 0, beta = 1  =>  D = C exactly
    assert np.array_equal(orc.encode("f16", orc.gemm("f16", A, B, C, 0.0, 1.0)), C)
    # beta = 0: C is not read -- NaN-poisoned C must not leak
    Cnan = np.full_like(C, 0x7E00)
    D0 = orc.gemm("f16", A, B, None, 1.0, 0.0)
    assert not np.isnan(orc.gemm("f16", A, B, Cnan, 1.0, 0.0)).any()
    # alpha = 2^e scales exactly
    assert np.array_equal(orc.gemm("f16", A, B, None, 0.25, 0.0), D0 * 0.25)


def test_gemm_k1_outer_product_single_rounding(orc):
    # K = 1: D = RN(a*b), one exact product and one rounding (R7)
    A, B, _ = synth.gemm_inputs(64, 64, 1, seed=41)
    got = orc.encode("f16", orc.gemm("f16", A, B))
    ref = (np_decode("f16", A) * np_decode("f16", B)).astype(np.float16).view(np.uint16)
    assert np.array_equal(got, ref)


def test_gemm_k0(orc):
    _, _, C = synth.gemm_inputs(5, 6, 1, seed=1, with_c=True)
    A = np.zeros((5, 0), np.uint16)
    B = np.zeros((0, 6), np.uint16)
    assert np.array_equal(orc.gemm("f16", A, B, C, 1.0, 2.0), 2.0 * np_decode("f16", C))


def test_gemm_batched_is_independent_gemms(orc):
    L, m, n, k = 5, 17, 19, 23
    A, B, C = synth.gemm_inputs(m, n, k, seed=51, batch=L, with_c=True)
    D = orc.gemm_batched("f16", A, B, C, 1.0, 1.0)
    for b in range(L):
        assert np.array_equal(D[b], orc.gemm("f16", A[b], B[b], C[b], 1.0, 1.0))
    ref = np.einsum("bik,bkj->bij", np_decode("f16", A), np_decode("f16", B)) + np_decode("f16", C)
    assert np.allclose(D, ref, rtol=1e-13, atol=1e-13)


# --------------------------------------------------------------------------- dual GEMM

def test_dual_sum_with_zero_b1_is_gemm(orc):
    # "Dual-GEMM, B2 = 0 -> output equals plain GEMM output"
    A, B0, B1, C0, _ = synth.dual_inputs(33, 40, 70, seed=61, with_c=True)
    Z = np.zeros_like(B1)
    assert np.array_equal(orc.dual_gemm("f16", "sum", A, B0, Z, C0, None, 1.0, 0.5),
                          orc.gemm("f16", A, B0, C0, 1.0, 0.5))


def test_dual_pair_is_two_gemms(orc):
    A, B0, B1, C0, C1 = synth.dual_inputs(21, 30, 50, seed=62, with_c=True)
    D0, D1 = orc.dual_gemm("f16", "pair", A, B0, B1, C0, C1, 1.5, -1.0)
    assert np.array_equal(D0, orc.gemm("f16", A, B0, C0, 1.5, -1.0))
    assert np.array_equal(D1, orc.gemm("f16", A, B1, C1, 1.5, -1.0))


@pytest.mark.parametrize("shape", [(3, 4, 5), (5, 2, 8)])
def test_dual_sum_vs_exact_rationals(orc, shape):
    m, n, k = shape
    A, B0, B1, C, _ = synth.dual_inputs(m, n, k, seed=63 + k, with_c=True)
    D = orc.dual_gemm("f16", "sum", A, B0, B1, C, None, 0.75, 1.5)
    a, b0, b1, c = (_frac("f16", X) for X in (A, B0, B1, C))
    for i in range(m):
        for j in range(n):
            s = sum((a[i][kk] * (b0[kk][j] + b1[kk][j]) for kk in range(k)), Fraction(0))
            S = sum((abs(a[i][kk] * b0[kk][j]) + abs(a[i][kk] * b1[kk][j]) for kk in range(k)), Fraction(0))
            e = Fraction(0.75) * s + Fraction(1.5) * c[i][j]
            assert abs(Fraction(D[i, j]) - e) <= (2 * k + 3) * Fraction(2) ** -53 * (S + abs(e) + 1)


def test_dual_integer_exact(orc):
    A, B0, B1, _, _ = synth.dual_inputs(30, 20, 300, seed=64, kind="int")
    ai, b0, b1 = (np_decode("f16", X).astype(np.int64) for X in (A, B0, B1))
    assert np.array_equal(orc.dual_gemm("f16", "sum", A, B0, B1), (ai @ b0 + ai @ b1).astype(float))


# --------------------------------------------------------------------------- row reduction

def test_rowsum_all_ones_is_k(orc):
    # "A = all-ones 64x64 -> y(i) = 64"
    ones = synth.f64_to_bits(np.ones((64, 64)), "f16")
    assert np.all(orc.rowsum("f16", ones) == 64.0)


def test_rowsum_identity_and_numpy(orc):
    I = synth.f64_to_bits(np.eye(50), "bf16")
    assert np.all(orc.rowsum("bf16", I) == 1.0)
    A, _, _ = synth.gemm_inputs(77, 1, 333, seed=71)
    assert np.allclose(orc.rowsum("f16", A), np_decode("f16", A).sum(axis=1), rtol=1e-14, atol=1e-14)


def test_rowsum_vs_exact_and_rows(orc):
    A, _, _ = synth.gemm_inputs(6, 1, 9, seed=72)
    y = orc.rowsum("f16", A)
    a = _frac("f16", A)
    for i in range(6):
        assert abs(Fraction(y[i]) - sum(a[i], Fraction(0))) <= 9 * Fraction(2) ** -53 * 9
    assert np.array_equal(orc.rowsum("f16", A, rows=[5, 0]), y[[5, 0]])
    # total of an integer matrix equals the sum of its row sums
    Ai, _, _ = synth.gemm_inputs(40, 1, 100, seed=73, kind="int")
    assert orc.rowsum("f16", Ai).sum() == np_decode("f16", Ai).astype(np.int64).sum()


# --------------------------------------------------------------------------- golden fixtures

def test_golden_fixtures(orc):
    """tests/golden/*.txt were written by scripts/make_golden.py (oracle only);
    each file's header cites the definition it exercises."""
    import glob
    import json
    import os

    files = sorted(glob.glob(os.path.join(os.path.dirname(__file__), "golden", "*.json")))
    assert files, "no golden fixtures"
    for f in files:
        g = json.load(open(f))
        dt = g["dtype"]
        A = np.array(g["A"], dtype=np.uint16)
        if g["op"] == "gemm":
            B = np.array(g["B"], dtype=np.uint16)
            C = np.array(g["C"], dtype=np.uint16) if g.get("C") is not None else None
            D = orc.encode(dt, orc.gemm(dt, A, B, C, g["alpha"], g["beta"]))
            assert np.array_equal(D, np.array(g["D_bits"], dtype=np.uint16)), f
        elif g["op"] == "rowsum":
            assert np.array_equal(orc.rowsum(dt, A), np.array(g["y"], dtype=np.float64)), f


# --------------------------------------------------------------------------- GLU (NEXT-3)

def test_act_vs_torch_float64(orc):
    x = np.concatenate([np.linspace(-30, 30, 2001), [0.0, 1e-8, -1e-8, 88.0, -88.0]])
    t = torch.from_numpy(x)
    assert np.allclose(orc.act("silu", x), torch.nn.functional.silu(t).numpy(), rtol=1e-15, atol=1e-300)
    # the tanh form cancels (1 + tanh -> 0) for x << 0: compare with an absolute floor of 1e-15 |x|
    g = torch.nn.functional.gelu(t, approximate="tanh").numpy()
    assert (np.abs(orc.act("gelu_tanh", x) - g) <= 1e-14 * np.abs(g) + 1e-15 * np.abs(x)).all()


def test_silu_identities(orc):
    # silu(x) - silu(-x) = x  (x*s(x) + x*s(-x)... = x since s(x) + s(-x) = 1), silu(0) = 0,
    # slope at 0 = 1/2, silu(x) -> x for large x, -> 0 for very negative x
    x = np.linspace(-20, 20, 401)
    assert np.allclose(orc.act("silu", x) - orc.act("silu", -x), x, rtol=0, atol=1e-13)
    assert orc.act("silu", [0.0])[0] == 0.0
    h = 1e-6
    assert abs((orc.act("silu", [h])[0] - orc.act("silu", [-h])[0]) / (2 * h) - 0.5) < 1e-9
    assert abs(orc.act("silu", [40.0])[0] - 40.0) < 1e-12 and abs(orc.act("silu", [-40.0])[0]) < 1e-15


def test_dual_glu_vs_products(orc):
    """GLU = act(alpha*A.B0) * (alpha*A.B1); integer inputs make both products exact, so the check
    reduces to the (library-pinned) activation of exact integers."""
    A, B0, B1, _, _ = synth.dual_inputs(37, 29, 120, seed=161, kind="int")
    for name, fn in (("silu", torch.nn.functional.silu),
                     ("gelu_tanh", lambda t: torch.nn.functional.gelu(t, approximate="tanh"))):
        D = orc.dual_glu("f16", name, A, B0, B1, alpha=0.5)
        x0 = 0.5 * (np_decode("f16", A).astype(np.int64) @ np_decode("f16", B0).astype(np.int64))
        x1 = 0.5 * (np_decode("f16", A).astype(np.int64) @ np_decode("f16", B1).astype(np.int64))
        ref = fn(torch.from_numpy(x0.astype(np.float64))).numpy() * x1
        assert np.allclose(D, ref, rtol=1e-14, atol=1e-12)
    rows = np.array([3, 0, 36])
    assert np.array_equal(orc.dual_glu("f16", "silu", A, B0, B1, rows=rows), orc.dual_glu("f16", "silu", A, B0, B1)[rows])


# --------------------------------------------------------------------------- attention (NEXT-4)

def _t64(dtype, bits):
    return torch.from_numpy(np_decode(dtype, bits))


@pytest.mark.parametrize("causal", [False, True])
def test_attention_vs_torch_sdpa_float64(orc, causal):
    """Library special case: torch scaled_dot_product_attention in float64 on the decoded inputs."""
    bh, sq, sk, d = 3, 37, 37 if causal else 53, 64
    Q = synth.uniform((bh, sq, d), 231)
    K = synth.uniform((bh, sk, d), 232)
    V = synth.uniform((bh, sk, d), 233)
    O, lse = orc.attention("f16", Q, K, V, causal=causal)
    ref = torch.nn.functional.scaled_dot_product_attention(_t64("f16", Q), _t64("f16", K), _t64("f16", V),
                                                           is_causal=causal).numpy()
    assert np.allclose(O, ref, rtol=1e-12, atol=1e-13)
    s = torch.einsum("hid,hjd->hij", _t64("f16", Q), _t64("f16", K)) / np.sqrt(d)
    if causal:
        s = s.masked_fill(torch.ones(sq, sk, dtype=torch.bool).triu(1), float("-inf"))
    assert np.allclose(lse, torch.logsumexp(s, dim=-1).numpy(), rtol=1e-13, atol=1e-13)


def test_attention_closed_forms(orc):
    d = 128
    V = synth.uniform((2, 40, d), 234)
    K = synth.uniform((2, 40, d), 235)
    # Q = 0: every score is 0, P is uniform -> O = mean of the V rows, lse = log(sk)
    Q0 = synth.f64_to_bits(np.zeros((2, 5, d)), "f16")
    O, lse = orc.attention("f16", Q0, K, V)
    assert np.allclose(O, np_decode("f16", V).mean(axis=1, keepdims=True).repeat(5, axis=1), rtol=0, atol=1e-15)
    assert np.allclose(lse, np.log(40.0), rtol=0, atol=1e-15)
    # one key: O = that V row exactly; causal row 0 sees only key 0
    O1, _ = orc.attention("f16", Q0[:, :1], K[:, :1], V[:, :1])
    assert np.array_equal(O1[:, 0], np_decode("f16", V[:, 0]))
    Qr = synth.uniform((2, 40, d), 236)
    Oc, _ = orc.attention("f16", Qr, K, V, causal=True)
    assert np.array_equal(Oc[:, 0], np_decode("f16", V[:, 0]))
    # constant V rows: O = the constant for any scores
    Vc = synth.f64_to_bits(np.full((2, 40, d), 0.375), "f16")
    Oq, _ = orc.attention("f16", Qr, K, Vc)
    assert np.allclose(Oq, 0.375, rtol=1e-15, atol=0)
