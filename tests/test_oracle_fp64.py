"""Pins of the FP64 prime-modulus oracle (Sec. 3.2, Eqs.
19-21; oracle/oz2_fp64_oracle.c, readings F1-F4 in DESIGN.md) against what the
paper and the mathematics fix -- not against the oracle itself:

  * Eq. (21) typed from the paper (tests/golden/eq21_primes_q1024.txt);
  * primality by an independent deterministic Miller-Rabin, and "largest":
    no prime between consecutive moduli or above m_1 below 2^b;
  * Eq. (19) q m^2 <= 2^55 and Eq. (20) q (m/2)^2 <= 2^53 for every q = 2^j;
  * m_16 / m_1 = 0.99995...;
  * CRT constants and reconstruction against Python integers;
  * end-to-end: integer inputs give C = AB exactly; inputs that need no
    truncation give the exactly rounded multi-word expansion of AB
    (Fractions); the error falls as s grows.
"""
import math
import os
from fractions import Fraction

import numpy as np
import pytest

from conftest import golden
from paper_2504_08009_b200.inputs import integer_matrix_np, phi_matrix_np, dyadic_matrix_np


def _is_prime(n: int) -> bool:
    """Deterministic Miller-Rabin for n < 3.3e24 (bases 2..41)."""
    if n < 2:
        return False
    small = (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37, 41)
    for p in small:
        if n % p == 0:
            return n == p
    d, r = n - 1, 0
    while d % 2 == 0:
        d //= 2
        r += 1
    for a in small:
        x = pow(a, d, n)
        if x in (1, n - 1):
            continue
        for _ in range(r - 1):
            x = x * x % n
            if x == n - 1:
                break
        else:
            return False
    return True


def test_eq21_typed_from_paper(oracle):
    eq21 = [int(r[0]) for r in golden("eq21_primes_q1024.txt")]
    assert len(eq21) == 16
    assert oracle.fp64_moduli(16, 1024) == eq21
    assert oracle.fp64_prime_bits(1024) == 22                  # "m_1 ~ 2^22 <= sqrt(2^45)"


def test_ratio_m16_m1(oracle):
    m = oracle.fp64_moduli(16, 1024)
    r = m[15] / m[0]
    assert 0.99995 <= r < 0.99996, r                           # "= 0.99995..."


@pytest.mark.parametrize("q", [1, 2, 3, 1000, 1024, 1025, 4096, 65536, 2**20])
def test_moduli_are_the_largest_primes_under_the_bound(oracle, q):
    s = 22
    m = oracle.fp64_moduli(s, q)
    b = oracle.fp64_prime_bits(q)
    assert b == (55 - (q - 1).bit_length()) // 2                # F1, ceil(log2 q) = bitlen(q - 1)
    assert all(_is_prime(v) for v in m)
    assert m == sorted(m, reverse=True) and len(set(m)) == s
    assert m[0] < 2**b
    # largest: no prime skipped above m_1 or between consecutive moduli
    for hi, lo in zip([2**b] + m[:-1], m):
        assert not any(_is_prime(v) for v in range(lo + 1, hi)), (lo, hi)
    for v in m:
        assert q * v * v <= 2**55                               # Eq. (19)
        assert q * ((v - 1) // 2) ** 2 <= 2**53                 # Eq. (20): residues |r| <= (m-1)/2


def test_crt_constants_and_roundtrip(oracle):
    import random
    rng = random.Random(5)
    for s, q in ((2, 1024), (7, 4096), (16, 1024), (22, 2**16)):
        c = oracle.fp64_constants(s, q)
        m = c["moduli"]
        M = math.prod(m)
        assert c["M"] == M
        for t in range(s):
            assert c["w"][t] % m[t] == 1                         # w_t = M_t y_t == 1 (mod m_t)
            assert all(c["w"][t] % m[u] == 0 for u in range(s) if u != t)
            assert 1 <= c["y"][t] < m[t]
        L, T = c["L"], c["T"]
        assert 2 ** (L + 1) <= M - 2 < 2 ** (L + 2)             # 2^L <= M/2 - 1 < 2^(L+1)
        assert T == L // 2
        for X in [-(M - 1) // 2, (M - 1) // 2, 0, 1, -1] + [rng.randrange(-(M - 1) // 2, (M - 1) // 2 + 1)
                                                          for _ in range(50)]:
            assert oracle.fp64_crt_scalar(s, q, [X % v for v in m]) == X


def _words_exact(ab: Fraction, v: int) -> list:
    """The exactly rounded v-word expansion (F3): w_1 = RN(x), w_2 = RN(x - w_1), ..."""
    out, r = [], ab
    for _ in range(v):
        w = float(r)                                            # Fraction -> float is RN
        out.append(w)
        r -= Fraction(w)
    return out


def test_integer_inputs_exact(oracle):
    A = integer_matrix_np(9, 40, 2**30, seed=1)
    B = integer_matrix_np(40, 7, 2**30, seed=2)
    C = oracle.fp64_dgemm(A, B, 12, v=3)
    exact = [[sum(int(a) * int(b) for a, b in zip(A[i], B[:, j])) for j in range(7)] for i in range(9)]
    for i in range(9):
        for j in range(7):
            assert Fraction(C[0, i, j]) + Fraction(C[1, i, j]) + Fraction(C[2, i, j]) == exact[i][j]
            assert C[:, i, j].tolist() == _words_exact(Fraction(exact[i][j]), 3)


@pytest.mark.parametrize("s,v", [(16, 2), (16, 3), (20, 3)])
def test_no_truncation_gives_exact_multiword(oracle, s, v):
    """Dyadic inputs with short mantissas and a small exponent range: 2^e a and
    2^f b are integers (no truncation), so X = (DA)(BE) and
    the words are the exactly rounded expansion of AB."""
    A = dyadic_matrix_np(6, 96, 20, 30, seed=3)
    B = dyadic_matrix_np(96, 5, 20, 30, seed=4)
    C, e, f = oracle.fp64_dgemm(A, B, s, v, want_exponents=True)
    for i in range(6):
        for j in range(5):
            ab = sum(Fraction(a) * Fraction(b) for a, b in zip(A[i], B[:, j]))
            assert C[:, i, j].tolist() == _words_exact(ab, v), (i, j)


def test_error_falls_with_s(oracle):
    """Accuracy grows with the number of moduli (M ~ s m_s, so
    k_A + k_B grows with s), here on phi = 2 inputs with 2-word output."""
    A = phi_matrix_np(8, 64, 2.0, seed=5)
    B = phi_matrix_np(64, 6, 2.0, seed=6)
    exact = [[sum(Fraction(a) * Fraction(b) for a, b in zip(A[i], B[:, j])) for j in range(6)] for i in range(8)]
    absab = np.abs(A) @ np.abs(B)
    errs = []
    for s in (4, 6, 8, 10, 12):
        C = oracle.fp64_dgemm(A, B, s, 2)
        err = max(abs(float(Fraction(C[0, i, j]) + Fraction(C[1, i, j]) - exact[i][j])) / absab[i, j]
                  for i in range(8) for j in range(6))
        errs.append(err)
    assert all(b < a for a, b in zip(errs, errs[1:]) if a > 2.0**-100), errs
    assert errs[0] > 2.0**-60 and errs[-1] < 2.0**-100, errs


def _trunc_fraction(x: Fraction) -> int:
    return math.floor(x) if x >= 0 else math.ceil(x)


def test_double_word_scaled_trunc(oracle):
    """Reading F6 (Eqs. 22-23): trunc(2^e (a1 + a2)) equals the truncation of the
    exact rational sum, including sums that sit on an integer with a tiny second
    word of the other sign and second words that underflow when scaled."""
    import random
    rng = random.Random(7)
    u = 2.0 ** -53
    cases = []
    for _ in range(3000):
        a1 = rng.uniform(-1, 1) * 2.0 ** rng.randint(-30, 30)
        a2 = a1 * u * rng.uniform(-1, 1)
        cases.append((a1, a2, rng.randint(-40, 120)))
    for n in (1.0, 5.0, -7.0, 2.0 ** 60, -(2.0 ** 70) - 2.0 ** 18):   # integral x1, tiny opposite x2
        for a2 in (-1e-300, 1e-300, -5e-324, 5e-324, -(2.0 ** -80), 2.0 ** -80, 0.0):
            cases.append((n, a2, 0))
            cases.append((n * 0.5, a2, 1))
    cases.append((3.0, -1e-310, -1000))                                  # scaled a1 < 1: 0
    cases.append((2.0 ** 100, -(2.0 ** 47), 50))                         # |a2| = u |a1|
    for a1, a2, e in cases:
        exact = (Fraction(a1) + Fraction(a2)) * Fraction(2) ** e
        assert oracle.fp64_scaled_trunc_mw(a1, a2, e) == _trunc_fraction(exact), (a1, a2, e)


@pytest.mark.parametrize("s,v", [(16, 3), (22, 4)])
def test_double_word_inputs_exact_multiword(oracle, s, v):
    """Double-word inputs whose words need no truncation (short mantissas, small
    exponent range): the result is the exactly rounded v-word expansion of
    (A1 + A2)(B1 + B2)."""
    A1 = dyadic_matrix_np(5, 64, 20, 20, seed=11)
    B1 = dyadic_matrix_np(64, 4, 20, 20, seed=12)
    A2 = dyadic_matrix_np(5, 64, 20, 20, seed=13) * 2.0 ** -60
    B2 = dyadic_matrix_np(64, 4, 20, 20, seed=14) * 2.0 ** -60
    A2 = np.where(np.abs(A2) <= np.abs(A1) * 2.0 ** -53, A2, 0.0)         # Eq. (23)
    B2 = np.where(np.abs(B2) <= np.abs(B1) * 2.0 ** -53, B2, 0.0)
    C = oracle.fp64_dgemm(A1, B1, s, v, A2=A2, B2=B2)
    for i in range(5):
        for j in range(4):
            ab = sum((Fraction(a) + Fraction(a2)) * (Fraction(b) + Fraction(b2))
                     for a, a2, b, b2 in zip(A1[i], A2[i], B1[:, j], B2[:, j]))
            assert C[:, i, j].tolist() == _words_exact(ab, v), (i, j)
