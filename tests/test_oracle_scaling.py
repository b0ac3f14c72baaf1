"""Pins for Part 1 / Alg. 1 lines 1-5 of the oracle: exponents, trunc, residues.

The FAST rule (reading R4) is pinned by what it must guarantee (the
Cauchy-Schwarz bound ||2^e a||_2 <= 2^T, checked in exact rational arithmetic)
and by how much it may give away (at most 2 bits below the largest exponent
that satisfies the bound), plus a hand-derived worked example.
"""
from fractions import Fraction
import math

import numpy as np
import pytest

from conftest import golden
from paper_2504_08009_b200.inputs import phi_matrix_np, dyadic_matrix_np


def _exact_sq_norm(vals, e):
    return sum(Fraction(float(v)) ** 2 for v in vals) * Fraction(2) ** (2 * int(e))


def _best_exponent(vals, T):
    """max{e : ||2^e v||_2 <= 2^T}, exactly."""
    s = sum(Fraction(float(v)) ** 2 for v in vals)
    # ||v|| 2^e <= 2^T  <=>  s 4^e <= 4^T
    lo, hi = -3000, 3000
    while lo < hi:
        mid = (lo + hi + 1) // 2
        if s * Fraction(4) ** mid <= Fraction(4) ** T:
            lo = mid
        else:
            hi = mid - 1
    return lo


def test_worked_example(oracle):
    A = np.array([[1.0, 0.5]])
    B = np.array([[0.25], [-3.0]])
    for row in golden("worked_example_fast.txt"):
        N, e, f = int(row[0]), int(row[1]), int(row[2])
        Ap = [int(v) for v in row[3:5]]
        Bp = [int(v) for v in row[5:7]]
        X, C = int(row[7]), float(row[8])
        assert list(oracle.scale_rows(A, N)) == [e]
        assert list(oracle.scale_cols(B, N)) == [f]
        assert list(oracle.trunc_rows(A, [e])[0]) == Ap
        assert list(oracle.trunc_cols(B, [f])[0]) == Bp
        Cg, Xg = oracle.crt(oracle.modmul(oracle.residues(oracle.trunc_rows(A, [e]), N),
                                          oracle.residues(oracle.trunc_cols(B, [f]), N)),
                            [e], [f], want_X=True)
        assert oracle.limbs_to_int(Xg[0, 0]) == X
        assert Cg[0, 0] == C
    # N = 3: B' = [128, -1536] has the Eq. (1) tie 128 -> -128 modulo 256
    Br = oracle.residues(oracle.trunc_cols(B, [9]), 3)
    assert list(Br[0, 0]) == [-128, 0]


@pytest.mark.parametrize("N", [2, 3, 8, 14, 16, 17, 20])
@pytest.mark.parametrize("phi", [0.0, 0.5, 2.0, 8.0])
def test_fast_rule_cauchy_schwarz_and_tightness(oracle, N, phi):
    T = oracle.constants(N)["T"]
    A = phi_matrix_np(6, 700, phi, seed=11 + N)        # 700 > 2 chunks of 256, ragged tail
    A[3, 100:] = 0.0
    A[4, :] *= 2.0 ** -1060                              # subnormal row
    e = oracle.scale_rows(A, N)
    for i in range(A.shape[0]):
        assert _exact_sq_norm(A[i], e[i]) <= Fraction(4) ** T
        best = _best_exponent(A[i], T)
        assert best - 2 <= e[i] <= best, (i, e[i], best)
    # columns use the same rule
    f = oracle.scale_cols(A.T.copy(), N)
    assert list(f) == list(e)


def test_fast_rule_special_rows(oracle):
    A = np.zeros((3, 300))
    A[1, 5] = np.nan
    A[2, 7] = -np.inf
    e = oracle.scale_rows(A, 14)
    assert e[0] == 0                                     # zero row
    assert e[1] == oracle.EXP_NONFINITE and e[2] == oracle.EXP_NONFINITE


@pytest.mark.parametrize("N", [2, 8, 14, 20])
def test_eq17_rule(oracle, N):
    A = phi_matrix_np(5, 64, 1.0, seed=3)
    ks = oracle.eq17_k(N, 64)
    e = oracle.scale_rows(A, N, mode=oracle.MODE_EQ17)
    for i in range(5):
        mx = max(abs(Fraction(float(v))) for v in A[i]) * Fraction(2) ** int(e[i])
        assert Fraction(2) ** (ks - 1) <= mx < Fraction(2) ** ks
    with pytest.raises(oracle.OracleError):               # budget < 1
        oracle.scale_rows(np.ones((1, 20000)), 2, mode=oracle.MODE_EQ17)


@pytest.mark.parametrize("N", [2, 14, 20])
def test_trunc_is_toward_zero(oracle, N):
    A = phi_matrix_np(4, 300, 1.0, seed=5)
    e = oracle.scale_rows(A, N)
    Ap = oracle.trunc_rows(A, e)
    for i in range(4):
        for l in range(300):
            x = Fraction(float(A[i, l])) * Fraction(2) ** int(e[i])
            v = Fraction(float(Ap[i, l]))
            assert v.denominator == 1
            assert abs(x - v) < 1 and abs(v) <= abs(x)      # trunc


@pytest.mark.parametrize("N", [2, 14, 16, 20])
def test_residues_match_python_ints(oracle, N):
    mods = oracle.constants(N)["moduli"]
    T = oracle.constants(N)["T"]
    A = phi_matrix_np(3, 257, 2.0, seed=9)
    e = oracle.scale_rows(A, N)
    Ap = oracle.trunc_rows(A, e)
    R = oracle.residues(Ap, N)
    assert R.dtype == np.int8
    for i in range(3):
        for l in range(257):
            x = int(Ap[i, l])
            assert abs(x) <= 2 ** T
            for t, m in enumerate(mods):
                r = int(R[t, i, l])
                assert (r - x) % m == 0 and -m <= 2 * r < m
    R1 = oracle.residues(np.array([[300.0]]), 2)
    assert list(R1[:, 0, 0]) == [44, 45]


def test_wide_conversions_against_python(oracle):
    rng = np.random.Generator(np.random.PCG64(1))
    for _ in range(400):
        x = float(np.trunc(np.ldexp(rng.random() - 0.5, int(rng.integers(0, 80)))))
        assert oracle.wide_from_double(x) == int(x)
    for _ in range(400):
        bits = int(rng.integers(1, 160))
        v = int(rng.integers(0, 2**62)) << max(0, bits - 62)
        v = v if rng.random() < 0.5 else -v
        assert oracle.wide_to_double(v) == float(v)          # Python int->float is RN-even
    for v in (2**54 + 1, 2**54 + 2, 2**54 + 6, 2**53 + 1, -(2**54 + 2), 2**100 + 2**47, 0):
        assert oracle.wide_to_double(v) == float(v)
