"""Pins for Alg. 1 lines 6-10 and the whole oracle pipeline.

The reconstruction is pinned to the exact integer product A'B' computed in
Python ints (X is unique and equals A'B' when (13) holds),
the end-to-end result to closed forms (integer inputs, identity, inputs that
need no truncation => correctly rounded AB) and to an a-priori error bound,
and the exact reference (Kulisch accumulator) to Python Fractions.
"""
from fractions import Fraction
import math

import numpy as np
import pytest

from paper_2504_08009_b200.inputs import phi_matrix_np, integer_matrix_np, dyadic_matrix_np


def test_modmul_spec_example(oracle):
    A = np.array([[[1, 2], [3, 4]]], np.int8)
    BT = np.array([[[5, 7], [6, 8]]], np.int8)            # B = [[5, 6], [7, 8]] stored transposed
    assert oracle.modmul(A, BT)[0].tolist() == [[19, 22], [43, 50]]


def test_modmul_against_numpy_int64(oracle):
    rng = np.random.Generator(np.random.PCG64(4))
    for (N, m, n, k) in [(3, 7, 5, 33), (2, 16, 16, 300), (5, 1, 9, 1000)]:
        Ar = rng.integers(-128, 128, size=(N, m, k)).astype(np.int8)
        Br = rng.integers(-128, 128, size=(N, n, k)).astype(np.int8)
        Ar[0, 0, :] = -128
        Br[0, 0, :] = -128
        ref = np.einsum("tik,tjk->tij", Ar.astype(np.int64), Br.astype(np.int64))
        assert np.array_equal(oracle.modmul(Ar, Br).astype(np.int64), ref)


def test_modmul_int32_boundary(oracle):
    # exact in INT32 for q < 2^17
    k = 2**17 - 1
    a = np.full((1, 1, k), -128, np.int8)
    assert int(oracle.modmul(a, a)[0, 0, 0]) == 2**31 - 16384
    a = np.full((1, 1, 2**17), -128, np.int8)
    with pytest.raises(oracle.OracleError):
        oracle.modmul(a, a)


def _python_int_product(Ap, BpT):
    A = [[int(v) for v in row] for row in Ap]
    B = [[int(v) for v in row] for row in BpT]
    return [[sum(x * y for x, y in zip(a, b)) for b in B] for a in A]


@pytest.mark.parametrize("N,mode,phi", [(2, 0, 0.5), (8, 0, 1.0), (14, 0, 0.5), (16, 0, 4.0),
                                        (17, 0, 1.0), (20, 0, 2.0), (8, 1, 0.5), (14, 1, 2.0),
                                        (20, 1, 1.0)])
def test_reconstruction_equals_integer_product(oracle, N, mode, phi):
    m, n, k = 9, 7, 300
    A = phi_matrix_np(m, k, phi, seed=21)
    B = phi_matrix_np(k, n, phi, seed=22)
    e = oracle.scale_rows(A, N, mode)
    f = oracle.scale_cols(B, N, mode)
    Ap = oracle.trunc_rows(A, e)
    BpT = oracle.trunc_cols(B, f)
    Cp = oracle.modmul(oracle.residues(Ap, N), oracle.residues(BpT, N))
    C, X = oracle.crt(Cp, e, f, want_X=True)
    ref = _python_int_product(Ap, BpT)
    M = math.prod(oracle.constants(N)["moduli"])
    for i in range(m):
        for j in range(n):
            x = oracle.limbs_to_int(X[i, j])
            assert x == ref[i][j]
            # condition (13): sum |a'||b'| < M/2
            assert 2 * sum(abs(int(a)) * abs(int(b)) for a, b in zip(Ap[i], BpT[j])) < M
            # line 10: c = RN(X) 2^-(e+f)
            assert C[i, j] == math.ldexp(float(ref[i][j]), -int(e[i] + f[j]))
    # line 7 reduction is the floor-mod of Alg. 1 (independent of the CRT path)
    C2 = oracle.dgemm(A, B, N, mode)
    assert np.array_equal(C, C2)


@pytest.mark.parametrize("N,phi", [(14, 1.0), (16, 0.5)])
def test_large_k_block_product(oracle, N, phi):
    """q >= 2^17 (reading R12): the block-accumulated products still
    reconstruct X = A'B' exactly -- checked against Python integers computed from
    A', B' alone (no modular arithmetic)."""
    m, n, k = 3, 2, 2**17 + 37
    A = phi_matrix_np(m, k, phi, seed=31)
    B = phi_matrix_np(k, n, phi, seed=32)
    C, e, f = oracle.dgemm(A, B, N, return_exponents=True)
    Ap = oracle.trunc_rows(A, e)
    BpT = oracle.trunc_cols(B, f)
    M = math.prod(oracle.constants(N)["moduli"])
    for i in range(m):
        a = [int(v) for v in Ap[i]]
        for j in range(n):
            b = [int(v) for v in BpT[j]]
            x = sum(p * q for p, q in zip(a, b))
            assert 2 * sum(abs(p * q) for p, q in zip(a, b)) < M       # condition (13)
            assert C[i, j] == math.ldexp(float(x), -int(e[i] + f[j]))
    # integer inputs within budget give AB exactly at this k too
    Ai = integer_matrix_np(2, k, 3, seed=33)
    Bi = integer_matrix_np(k, 2, 3, seed=34)
    assert np.array_equal(oracle.dgemm(Ai, Bi, N), (Ai.astype(np.int64) @ Bi.astype(np.int64)).astype(np.float64))


@pytest.mark.parametrize("N", [8, 14, 20])
def test_integer_inputs_exact(oracle, N):
    # integer matrices within budget give AB exactly
    A = integer_matrix_np(10, 64, 1000, seed=1)
    B = integer_matrix_np(64, 12, 1000, seed=2)
    C = oracle.dgemm(A, B, N)
    ref = (A.astype(np.int64) @ B.astype(np.int64)).astype(np.float64)
    assert np.array_equal(C, ref)


def test_identity(oracle):
    B = dyadic_matrix_np(16, 16, 20, 8, seed=3)            # I B = B
    C = oracle.dgemm(np.eye(16), B, 14)
    assert np.array_equal(C, B)


@pytest.mark.parametrize("N", [14, 16, 20])
def test_no_truncation_gives_correctly_rounded_AB(oracle, N):
    # short mantissas and a small exponent range: every 2^e a is an integer, so
    # X = D A B E exactly and C = RN(AB)
    A = dyadic_matrix_np(8, 40, 12, 6, seed=7)
    B = dyadic_matrix_np(40, 8, 12, 6, seed=8)
    e = oracle.scale_rows(A, N)
    f = oracle.scale_cols(B, N)
    assert np.array_equal(oracle.trunc_rows(A, e), np.ldexp(A, e[:, None]))
    C = oracle.dgemm(A, B, N)
    for i in range(8):
        for j in range(8):
            exact = sum(Fraction(float(A[i, l])) * Fraction(float(B[l, j])) for l in range(40))
            assert C[i, j] == float(exact)


def test_exact_reference_against_fractions(oracle):
    rng = np.random.Generator(np.random.PCG64(6))
    for trial in range(30):
        k = int(rng.integers(1, 40))
        a = phi_matrix_np(1, k, 6.0, seed=100 + trial)
        b = phi_matrix_np(k, 1, 6.0, seed=200 + trial)
        if trial % 3 == 0:
            a[0, 0] = 2.0 ** -1070                          # subnormal factor
            b[0, 0] = 3.0
        if trial % 3 == 1 and k > 1:                         # exact cancellation
            a[0, 1] = -a[0, 0]
            b[1, 0] = b[0, 0]
        ab, absab = oracle.exact_entries(a, b, [0], [0])
        ex = sum(Fraction(float(a[0, l])) * Fraction(float(b[l, 0])) for l in range(k))
        exa = sum(abs(Fraction(float(a[0, l])) * Fraction(float(b[l, 0]))) for l in range(k))
        assert ab[0] == float(ex)
        assert absab[0] == float(exa)


@pytest.mark.parametrize("N,phi", [(8, 0.5), (14, 1.0), (16, 2.0), (20, 4.0)])
def test_a_priori_error_bound(oracle, N, phi):
    # |d| < 1 truncation on each side:
    # |c - ab| <= 2^-f sum|a| + 2^-e sum|b| + k 2^-(e+f) + ulp(c)/2
    m, n, k = 6, 6, 500
    A = phi_matrix_np(m, k, phi, seed=31)
    B = phi_matrix_np(k, n, phi, seed=32)
    C, e, f = oracle.dgemm(A, B, N, return_exponents=True)
    for i in range(m):
        for j in range(n):
            exact = sum(Fraction(float(A[i, l])) * Fraction(float(B[l, j])) for l in range(k))
            bound = (Fraction(2) ** -int(f[j]) * sum(abs(Fraction(float(v))) for v in A[i])
                     + Fraction(2) ** -int(e[i]) * sum(abs(Fraction(float(v))) for v in B[:, j])
                     + k * Fraction(2) ** -int(e[i] + f[j])
                     + Fraction(math.ulp(C[i, j])) / 2)
            assert abs(Fraction(float(C[i, j])) - exact) <= bound


def _compwise(C, A, B, pairs, oracle):
    ii, jj = pairs
    ab, absab = oracle.exact_entries(A, B, ii, jj)
    err = np.abs(C[ii, jj] - ab) / absab
    return float(err.max())


def test_error_vs_N_trend_and_dgemm_level(oracle):
    # Eqs. (15)-(17): every added modulus adds ~log2(m)/2 bits
    # per operand until the FP64 floor; 14 or 15 moduli reach
    # DGEMM-level accuracy at phi = 0.5.
    m = n = 24
    k = 1024
    A = phi_matrix_np(m, k, 0.5, seed=41)
    B = phi_matrix_np(k, n, 0.5, seed=42)
    ii, jj = np.meshgrid(np.arange(m), np.arange(n), indexing="ij")
    pairs = (ii.ravel(), jj.ravel())
    errs = {N: _compwise(oracle.dgemm(A, B, N), A, B, pairs, oracle) for N in range(6, 21)}
    for N in range(6, 12):                                   # pre-floor: strictly better
        assert errs[N + 1] < errs[N] / 4
    assert errs[6] > 2.0 ** 30 * errs[15]
    dgemm_err = _compwise(A @ B, A, B, pairs, oracle)
    assert errs[15] <= 2.0 ** -50
    assert errs[15] <= 2 * max(dgemm_err, 2.0 ** -53)
    assert errs[20] <= 2.0 ** -52


def test_nonfinite_propagation_and_degenerate(oracle):
    A = phi_matrix_np(5, 40, 1.0, seed=51)
    B = phi_matrix_np(40, 6, 1.0, seed=52)
    C0 = oracle.dgemm(A, B, 14)
    A[2, 3] = np.nan
    B[7, 4] = np.inf
    C = oracle.dgemm(A, B, 14)
    assert np.isnan(C[2]).all() and np.isnan(C[:, 4]).all()
    mask = np.ones_like(C, bool)
    mask[2] = False
    mask[:, 4] = False
    assert np.array_equal(C[mask], C0[mask])
    assert np.array_equal(oracle.dgemm(np.zeros((3, 0)), np.zeros((0, 4)), 14), np.zeros((3, 4)))
    with pytest.raises(oracle.OracleError):
        oracle.dgemm(np.ones((1, 5)), np.ones((5, 1)), 21)
    with pytest.raises(oracle.OracleError):
        oracle.dgemm(np.ones((1, 5)), np.ones((5, 1)), 1)


def test_gemm_surface_axpby_against_fractions(oracle):
    """Reading R19 (BLAS DGEMM semantics around Algorithm 1): each entry is
    RN(alpha c + RN(beta c_old)); pinned against exact rational arithmetic
    (float(Fraction) rounds to nearest) and the transposes against dgemm."""
    A = phi_matrix_np(6, 40, 1.0, seed=51)
    B = phi_matrix_np(40, 5, 1.0, seed=52)
    Cold = phi_matrix_np(6, 5, 2.0, seed=53)
    c = oracle.dgemm(A, B, 14)
    for alpha, beta in [(1.0, 0.0), (-0.7, 0.0), (1.3, 2.1), (3.0, -1.0), (1e-300, 1e300)]:
        got = oracle.gemm(A, B, 14, alpha, beta, Cold)
        for i in range(6):
            for j in range(5):
                if beta == 0.0:
                    ref = alpha * c[i, j]
                else:
                    ref = float(Fraction(alpha) * Fraction(float(c[i, j])) + Fraction(beta * Cold[i, j]))
                assert got[i, j] == ref, (alpha, beta, i, j)
    # beta == 0: C_old is not read (NaN ignored); alpha == 0: no product
    nan = np.full((6, 5), np.nan)
    assert np.array_equal(oracle.gemm(A, B, 14, 2.0, 0.0, nan), 2.0 * c)
    assert np.array_equal(oracle.gemm(A, B, 14, 0.0, 3.0, Cold), 3.0 * Cold)
    # op(A) = A^T of the stored k x m matrix, op(B) = B^T of the stored n x k matrix
    assert np.array_equal(oracle.gemm(A.T.copy(), B.T.copy(), 14, transA=True, transB=True), c)
