"""Oracle for Ozaki scheme II (INT8 moduli) -- TEST INFRASTRUCTURE ONLY.

A ctypes wrapper around ``oz2_oracle.c``: a plain, slow, exact CPU
implementation of Algorithm 1 that shares no code with the
CUDA product path.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py`` (its ``cpu_baseline`` leg and ``--impl reference``) may import
this package.  Every function below forwards to the C function of the same
name, whose header comment cites the PAPER.md passage it follows.

Parity status: every stage is pinned by ``tests/test_oracle_*.py``.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oz2_oracle.c")
_SRCS = [_SRC, os.path.join(_HERE, "oz2_fp64_oracle.c")]
_HDRS = [os.path.join(_HERE, "oz2_wide.h"), os.path.join(_HERE, "oz2_fast_rule.h")]
_LIB = os.path.join(_HERE, "liboz2_oracle.so")

MODE_FAST = 0
MODE_EQ17 = 1
MODE_ACCU = 2
EXP_NONFINITE = -(2**31)
KC = 256

ERRORS = {0: "ok", 1: "invalid argument", 2: "num_moduli out of [2, 20]",
          3: "k >= 2^17", 4: "EQ17 budget < 1", 5: "int32 overflow"}


class OracleError(RuntimeError):
    pass


def build(force: bool = False) -> str:
    """Compile liboz2_oracle.so (gcc, OpenMP, no FP contraction)."""
    if force or not os.path.exists(_LIB) or any(os.path.getmtime(_LIB) < os.path.getmtime(f) for f in _SRCS + _HDRS):
        cmd = ["gcc", "-O2", "-fopenmp", "-ffp-contract=off", "-fPIC", "-shared",
               "-o", _LIB + ".tmp", *_SRCS, "-lm"]
        subprocess.check_call(cmd)
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        i64, i32 = ctypes.c_int64, ctypes.c_int
        L.oz2o_constants.argtypes = [i32, P, P, P, P, P, P]
        L.oz2o_smod_i64.argtypes = [i64, i64]
        L.oz2o_smod_i64.restype = i64
        L.oz2o_smod_i64_long.argtypes = [i64, i64]
        L.oz2o_smod_i64_long.restype = i64
        L.oz2o_crt_scalar.argtypes = [i32, P, P]
        L.oz2o_eq17_k.argtypes = [i32, i64]
        L.oz2o_scale_fast.argtypes = [i64, i64, P, i64, i64, i32, P]
        L.oz2o_scale_eq17.argtypes = [i64, i64, P, i64, i64, i32, i64, P]
        L.oz2o_trunc_scale.argtypes = [i64, i64, P, i64, i64, P, P]
        L.oz2o_trunc_scale.restype = None
        L.oz2o_residues.argtypes = [i64, i64, P, i32, P]
        L.oz2o_modmul.argtypes = [i64, i64, i64, P, P, i32, P]
        L.oz2o_crt.argtypes = [i64, i64, i32, P, P, P, P, i64, P]
        L.oz2o_dgemm.argtypes = [i64, i64, i64, P, i64, P, i64, P, i64, i32, i32, P, P]
        L.oz2o_exact_entries.argtypes = [i64, P, i64, P, i64, i64, P, P, P, P]
        L.oz2o_exact_entries.restype = None
        L.oz2o_wide_to_double.argtypes = [P]
        L.oz2o_wide_to_double.restype = ctypes.c_double
        L.oz2o_wide_from_double.argtypes = [ctypes.c_double, P]
        L.oz2o_wide_from_double.restype = None
        L.oz2o_set_threads.argtypes = [i32]
        L.oz2o_scale_accu.argtypes = [i64, i64, i64, P, i64, P, i64, i32, P, P, P, P]
        L.oz2o_axpby.argtypes = [i64, ctypes.c_double, P, ctypes.c_double, P, P]
        L.oz2o_axpby.restype = None
        L.oz2o_set_threads.restype = None
        L.oz2f_prime_bits.argtypes = [i64]
        L.oz2f_moduli.argtypes = [i32, i64, P]
        L.oz2f_constants.argtypes = [i32, i64, P, P, P, P, P, P]
        L.oz2f_dgemm.argtypes = [i64, i64, i64, P, i64, P, i64, i32, i32, P, i64, P, P]
        L.oz2f_dgemm_mw.argtypes = [i64, i64, i64, P, P, i64, P, P, i64, i32, i32, P, i64, P, P]
        L.oz2f_scaled_trunc_mw.argtypes = [ctypes.c_double, ctypes.c_double, i32, P]
        L.oz2f_scaled_trunc_mw.restype = None
        L.oz2f_crt_scalar.argtypes = [i32, i64, P, P]
        L.oz2o_get_threads.restype = i32
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _check(rc: int):
    if rc != 0:
        raise OracleError(f"oracle error {rc}: {ERRORS.get(rc, '?')}")


def limbs_to_int(limbs) -> int:
    """256-bit two's-complement little-endian limbs -> Python int."""
    v = 0
    for i, x in enumerate(limbs):
        v |= int(x) << (64 * i)
    return v - (1 << 256) if v >> 255 else v


def int_to_limbs(v: int) -> np.ndarray:
    v &= (1 << 256) - 1
    return np.array([(v >> (64 * i)) & ((1 << 64) - 1) for i in range(4)], dtype=np.uint64)


def set_threads(n: int) -> None:
    lib().oz2o_set_threads(int(n))


def get_threads() -> int:
    return int(lib().oz2o_get_threads())


def constants(N: int) -> dict:
    m = np.zeros(N, np.int32)
    y = np.zeros(N, np.int32)
    M = np.zeros(4, np.uint64)
    w = np.zeros((N, 4), np.uint64)
    L = ctypes.c_int32()
    T = ctypes.c_int32()
    _check(lib().oz2o_constants(N, _p(m), _p(y), _p(M), _p(w), ctypes.byref(L), ctypes.byref(T)))
    return {"moduli": [int(v) for v in m], "y": [int(v) for v in y], "M": limbs_to_int(M),
            "w": [limbs_to_int(w[t]) for t in range(N)], "L": L.value, "T": T.value}


def smod(a: int, m: int) -> int:
    return int(lib().oz2o_smod_i64(int(a), int(m)))


def smod_long(a: int, m: int) -> int:
    """Eq. (1) through the wide long-division path (the one the CRT uses)."""
    return int(lib().oz2o_smod_i64_long(int(a), int(m)))


def crt_scalar(N: int, c) -> int:
    arr = np.ascontiguousarray(np.asarray(c, dtype=np.int64))
    out = np.zeros(4, np.uint64)
    _check(lib().oz2o_crt_scalar(N, _p(arr), _p(out)))
    return limbs_to_int(out)


def eq17_k(N: int, q: int) -> int:
    return int(lib().oz2o_eq17_k(N, int(q)))


def _as_f64(X):
    return np.ascontiguousarray(np.asarray(X, dtype=np.float64))


def scale_rows(A, N: int, mode: int = MODE_FAST, q: int | None = None) -> np.ndarray:
    """Exponent vector e (Alg. 1 line 1) for the rows of A (m x k)."""
    A = _as_f64(A)
    m, k = A.shape
    e = np.zeros(m, np.int32)
    if mode == MODE_FAST:
        _check(lib().oz2o_scale_fast(m, k, _p(A), k, 1, N, _p(e)))
    else:
        _check(lib().oz2o_scale_eq17(m, k, _p(A), k, 1, N, k if q is None else q, _p(e)))
    return e


def scale_cols(B, N: int, mode: int = MODE_FAST, q: int | None = None) -> np.ndarray:
    """Exponent vector f (Alg. 1 line 1) for the columns of B (k x n)."""
    B = _as_f64(B)
    k, n = B.shape
    f = np.zeros(n, np.int32)
    if mode == MODE_FAST:
        _check(lib().oz2o_scale_fast(n, k, _p(B), 1, n, N, _p(f)))
    else:
        _check(lib().oz2o_scale_eq17(n, k, _p(B), 1, n, N, k if q is None else q, _p(f)))
    return f


def scale_accu(A, B, N: int):
    """OS II-accu exponents (reading R18): (e, f, rowmax P, colmax P)."""
    A = _as_f64(A)
    B = _as_f64(B)
    m, k = A.shape
    n = B.shape[1]
    e = np.zeros(m, np.int32)
    f = np.zeros(n, np.int32)
    pr = np.zeros(m, np.uint32)
    pc = np.zeros(n, np.uint32)
    _check(lib().oz2o_scale_accu(m, n, k, _p(A), max(k, 1), _p(B), max(n, 1), N, _p(e), _p(f), _p(pr), _p(pc)))
    return e, f, pr, pc


def trunc_rows(A, e) -> np.ndarray:
    """A' = trunc(D A) (Alg. 1 line 2), m x k FP64 integers."""
    A = _as_f64(A)
    m, k = A.shape
    e = np.ascontiguousarray(e, dtype=np.int32)
    out = np.zeros((m, k), np.float64)
    lib().oz2o_trunc_scale(m, k, _p(A), k, 1, _p(e), _p(out))
    return out


def trunc_cols(B, f) -> np.ndarray:
    """B' = trunc(B E) (Alg. 1 line 3), returned transposed: n x k."""
    B = _as_f64(B)
    k, n = B.shape
    f = np.ascontiguousarray(f, dtype=np.int32)
    out = np.zeros((n, k), np.float64)
    lib().oz2o_trunc_scale(n, k, _p(B), 1, n, _p(f), _p(out))
    return out


def residues(Xp, N: int) -> np.ndarray:
    """Eq. (11): int8 planes [N][rows][len] of an FP64-integer matrix."""
    Xp = _as_f64(Xp)
    r, l = Xp.shape
    out = np.zeros((N, r, l), np.int8)
    _check(lib().oz2o_residues(r, l, _p(Xp), N, _p(out)))
    return out


def modmul(Ar, Br) -> np.ndarray:
    """Alg. 1 line 6: int32 [N][m][n] from Ar [N][m][k] and Br [N][n][k]."""
    Ar = np.ascontiguousarray(Ar, dtype=np.int8)
    Br = np.ascontiguousarray(Br, dtype=np.int8)
    N, m, k = Ar.shape
    n = Br.shape[1]
    out = np.zeros((N, m, n), np.int32)
    _check(lib().oz2o_modmul(m, n, k, _p(Ar), _p(Br), N, _p(out)))
    return out


def crt(Cp, e, f, want_X: bool = False):
    """Alg. 1 lines 7-10: C (m x n FP64) from int32 products [N][m][n]."""
    Cp = np.ascontiguousarray(Cp, dtype=np.int32)
    N, m, n = Cp.shape
    e = np.ascontiguousarray(e, dtype=np.int32)
    f = np.ascontiguousarray(f, dtype=np.int32)
    C = np.zeros((m, n), np.float64)
    X = np.zeros((m, n, 4), np.uint64) if want_X else None
    _check(lib().oz2o_crt(m, n, N, _p(Cp), _p(e), _p(f), _p(C), n, _p(X) if want_X else None))
    return (C, X) if want_X else C


def dgemm(A, B, N: int, mode: int = MODE_FAST, return_exponents: bool = False):
    """Algorithm 1 end to end: C ~= A B."""
    A = _as_f64(A)
    B = _as_f64(B)
    m, k = A.shape
    k2, n = B.shape
    assert k == k2
    C = np.zeros((m, n), np.float64)
    e = np.zeros(max(m, 1), np.int32)
    f = np.zeros(max(n, 1), np.int32)
    _check(lib().oz2o_dgemm(m, n, k, _p(A), k, _p(B), n, _p(C), n, N, mode, _p(e), _p(f)))
    return (C, e[:m], f[:n]) if return_exponents else C


def gemm(A, B, N: int, alpha: float = 1.0, beta: float = 0.0, C=None, transA: bool = False,
         transB: bool = False, mode: int = MODE_FAST) -> np.ndarray:
    """alpha op(A) op(B) + beta C around dgemm (reading R19): the transposes are
    plain numpy views, the update is oz2o_axpby."""
    Aop = np.ascontiguousarray(np.asarray(A, np.float64).T if transA else A, dtype=np.float64)
    Bop = np.ascontiguousarray(np.asarray(B, np.float64).T if transB else B, dtype=np.float64)
    m, n = Aop.shape[0], Bop.shape[1]
    Cold = np.zeros((m, n)) if C is None else np.ascontiguousarray(C, dtype=np.float64)
    if alpha == 0.0 or Aop.shape[1] == 0:
        return np.zeros((m, n)) if beta == 0.0 else beta * Cold
    ab = dgemm(Aop, Bop, N, mode)
    out = np.empty((m, n))
    lib().oz2o_axpby(m * n, float(alpha), _p(ab), float(beta), _p(Cold), _p(out))
    return out


def syrk(A, N: int, uplo: str = "L", trans: bool = False, alpha: float = 1.0, beta: float = 0.0, C=None,
         mode: int = MODE_FAST) -> np.ndarray:
    """DSYRK (reading R19): the `uplo` triangle (diagonal
    included) of gemm(op(A), op(A)^T, alpha, beta, C); the other triangle of C
    is returned unchanged (zeros when C is None)."""
    A = np.asarray(A, np.float64)
    Aop = A.T if trans else A
    n = Aop.shape[0]
    Cold = np.zeros((n, n)) if C is None else np.array(C, dtype=np.float64)
    full = gemm(Aop, Aop.T, N, alpha, beta, Cold, mode=mode)
    mask = np.tril(np.ones((n, n), bool)) if uplo.upper() == "L" else np.triu(np.ones((n, n), bool))
    out = Cold.copy()
    out[mask] = full[mask]
    return out


def trmm(A, B, N: int, side: str = "L", uplo: str = "L", transA: bool = False, unit: bool = False,
         alpha: float = 1.0, mode: int = MODE_FAST) -> np.ndarray:
    """DTRMM (reading R19): alpha op(T) B or alpha B op(T)
    with T = the uplo triangle of A (zeros elsewhere; ones on a unit diagonal)."""
    A = np.asarray(A, np.float64)
    T = np.tril(A) if uplo.upper() == "L" else np.triu(A)
    if unit:
        np.fill_diagonal(T, 1.0)
    if side.upper() == "L":
        return gemm(T, B, N, alpha, 0.0, None, transA=transA, mode=mode)
    return gemm(B, T, N, alpha, 0.0, None, transB=transA, mode=mode)


def limbs_matrix_to_ints(X) -> list:
    m, n, _ = X.shape
    return [[limbs_to_int(X[i, j]) for j in range(n)] for i in range(m)]


def exact_entries(A, B, ii, jj):
    """Exact (AB)_ij and (|A||B|)_ij, each rounded once to nearest."""
    A = _as_f64(A)
    B = _as_f64(B)
    k = A.shape[1]
    ii = np.ascontiguousarray(ii, dtype=np.int64)
    jj = np.ascontiguousarray(jj, dtype=np.int64)
    ab = np.zeros(len(ii), np.float64)
    absab = np.zeros(len(ii), np.float64)
    lib().oz2o_exact_entries(k, _p(A), A.shape[1], _p(B), B.shape[1], len(ii), _p(ii), _p(jj),
                             _p(ab), _p(absab))
    return ab, absab


def wide_to_double(v: int) -> float:
    limbs = int_to_limbs(v)
    return float(lib().oz2o_wide_to_double(_p(limbs)))


def wide_from_double(x: float) -> int:
    out = np.zeros(4, np.uint64)
    lib().oz2o_wide_from_double(float(x), _p(out))
    return limbs_to_int(out)


# ---------------------------------------------------------------------------
# FP64 prime-modulus regime (Sec. 3.2; oz2_fp64_oracle.c)
# ---------------------------------------------------------------------------
FP64_WL = 10


def fp64_prime_bits(q: int) -> int:
    """Reading F1: b = floor((55 - ceil(log2 q)) / 2)."""
    return int(lib().oz2f_prime_bits(int(q)))


def fp64_moduli(s: int, q: int) -> list:
    """Reading F1: the s largest primes below 2^b (Eqs. 19-21)."""
    out = np.zeros(s, np.int64)
    _check(lib().oz2f_moduli(s, int(q), _p(out)))
    return [int(v) for v in out]


def _limbs_to_int_wl(limbs) -> int:
    v = 0
    for i, x in enumerate(limbs):
        v |= int(x) << (64 * i)
    nb = 64 * len(limbs)
    return v - (1 << nb) if v >> (nb - 1) else v


def fp64_constants(s: int, q: int) -> dict:
    m = np.zeros(s, np.int64)
    y = np.zeros(s, np.int64)
    M = np.zeros(FP64_WL, np.uint64)
    w = np.zeros(s * FP64_WL, np.uint64)
    L, T = ctypes.c_int32(), ctypes.c_int32()
    _check(lib().oz2f_constants(s, int(q), _p(m), _p(y), _p(M), _p(w), ctypes.byref(L), ctypes.byref(T)))
    return {"moduli": [int(v) for v in m], "y": [int(v) for v in y], "M": _limbs_to_int_wl(M),
            "w": [_limbs_to_int_wl(w[t * FP64_WL:(t + 1) * FP64_WL]) for t in range(s)], "L": L.value, "T": T.value}


def fp64_crt_scalar(s: int, q: int, residues) -> int:
    c = np.asarray(residues, np.int64)
    X = np.zeros(FP64_WL, np.uint64)
    _check(lib().oz2f_crt_scalar(s, int(q), _p(c), _p(X)))
    return _limbs_to_int_wl(X)


def fp64_dgemm(A, B, s: int, v: int = 2, want_exponents: bool = False, A2=None, B2=None):
    """C ~= A B in the FP64 prime regime with s primes for q = k: v binary64
    words per entry, returned as [v][m][n] (most significant first, F3).
    A2 / B2: second words of double-word inputs (A = A + A2, reading F6)."""
    A = _as_f64(A)
    B = _as_f64(B)
    m, k = A.shape
    n = B.shape[1]
    C = np.zeros((v, m, n), np.float64)
    e = np.zeros(max(m, 1), np.int32)
    f = np.zeros(max(n, 1), np.int32)
    if A2 is None and B2 is None:
        _check(lib().oz2f_dgemm(m, n, k, _p(A), k, _p(B), n, s, v, _p(C), n, _p(e), _p(f)))
    else:
        A2 = _as_f64(A2) if A2 is not None else None
        B2 = _as_f64(B2) if B2 is not None else None
        _check(lib().oz2f_dgemm_mw(m, n, k, _p(A), _p(A2) if A2 is not None else None, k, _p(B),
                                   _p(B2) if B2 is not None else None, n, s, v, _p(C), n, _p(e), _p(f)))
    if want_exponents:
        return C, e[:m], f[:n]
    return C


def fp64_scaled_trunc_mw(a1: float, a2: float, e: int) -> int:
    """Reading F6 for one element: trunc(2^e (a1 + a2))."""
    out = np.zeros(FP64_WL, np.uint64)
    lib().oz2f_scaled_trunc_mw(float(a1), float(a2), int(e), _p(out))
    return _limbs_to_int_wl(out)
