"""CPU pins for the SYRK-structured product ("GEMM, TRMM,
or SYRK"; BLAS DSYRK semantics, reading R19) as the oracle composes it.

oz2_dsyrk converts op(A) once and lets one set of residue planes serve both
operands, which is exact only if Algorithm 1 gives op(A)^T's column exponents
equal to op(A)'s row exponents -- then C = D^-1 X D^-1 with X = A' A'^T
symmetric, so the emulated A A^T is bitwise symmetric.  That is pinned here
for the FAST, EQ17 and ACCU rules, together with the triangle semantics."""
import numpy as np
import pytest

from paper_2504_08009_b200.inputs import phi_matrix_np


@pytest.mark.parametrize("mode", [0, 1, 2])
@pytest.mark.parametrize("N", [5, 14, 18])
def test_emulated_AAT_is_bitwise_symmetric(oracle, mode, N):
    A = phi_matrix_np(23, 300, 1.0, seed=500 + N)
    A[4] *= 2.0 ** 40                                   # rows of very different scale
    A[9] = 0.0
    C, e, f = oracle.dgemm(A, np.ascontiguousarray(A.T), N, mode, return_exponents=True)
    assert np.array_equal(e, f), "column exponents of A^T differ from row exponents of A"
    assert np.array_equal(C.view(np.int64), C.T.view(np.int64)), "emulated A A^T is not symmetric"


@pytest.mark.parametrize("uplo", ["L", "U"])
@pytest.mark.parametrize("trans", [False, True])
def test_syrk_triangle_semantics(oracle, uplo, trans):
    n, k = 17, 40
    A = phi_matrix_np(k, n, 0.5, seed=7) if trans else phi_matrix_np(n, k, 0.5, seed=7)
    C0 = phi_matrix_np(n, n, 1.0, seed=8)
    alpha, beta = -1.5, 0.25
    out = oracle.syrk(A, 14, uplo, trans, alpha, beta, C0)
    Aop = A.T if trans else A
    full = oracle.gemm(Aop, Aop.T, 14, alpha, beta, C0)
    tri = np.tril(np.ones((n, n), bool)) if uplo == "L" else np.triu(np.ones((n, n), bool))
    assert np.array_equal(out[tri].view(np.int64), full[tri].view(np.int64))
    assert np.array_equal(out[~tri].view(np.int64), C0[~tri].view(np.int64)), "other triangle touched"


def test_syrk_integer_closed_form(oracle):
    # small integers need no truncation: the triangle is exactly A A^T (closed form)
    rng = np.random.Generator(np.random.PCG64(3))
    A = rng.integers(-1000, 1000, size=(12, 50)).astype(np.float64)
    out = oracle.syrk(A, 14, "U")
    exact = A @ A.T                                     # integers < 2^53: exact in FP64
    tri = np.triu(np.ones((12, 12), bool))
    assert np.array_equal(out[tri], exact[tri]) and (out[~tri] == 0).all()


@pytest.mark.parametrize("side", ["L", "R"])
@pytest.mark.parametrize("uplo", ["L", "U"])
def test_trmm_oracle_closed_forms(oracle, side, uplo):
    """DTRMM oracle: with a unit diagonal and a zero strict triangle, op(T) = I and
    (for a B that needs no truncation: small integers) the result is alpha B
    exactly; with integer entries it is the exact triangular product."""
    n, m = 9, 7
    rng0 = np.random.Generator(np.random.PCG64(21))
    B = rng0.integers(-1000, 1000, size=(m, n) if side == "R" else (n, m)).astype(np.float64)
    na = n
    Z = np.zeros((na, na))
    out = oracle.trmm(Z, B, 14, side, uplo, unit=True, alpha=-0.5)
    assert np.array_equal(out, -0.5 * B)
    rng = np.random.Generator(np.random.PCG64(22))
    A = rng.integers(-50, 50, size=(na, na)).astype(np.float64)
    Bi = rng.integers(-50, 50, size=B.shape).astype(np.float64)
    T = np.tril(A) if uplo == "L" else np.triu(A)
    for transA in (False, True):
        Top = T.T if transA else T
        exact = Top @ Bi if side == "L" else Bi @ Top
        assert np.array_equal(oracle.trmm(A, Bi, 14, side, uplo, transA), exact)
