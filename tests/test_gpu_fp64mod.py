"""GPU parity of the FP64 prime-modulus regime (Sec. 3.2;
include/oz2.h oz2_dgemm_fp64mod) against the oracle (oracle/oz2_fp64_oracle.c):
every output word bitwise, for s = 2..22 primes, 1..4 words, ragged shapes,
k on both sides of a prime-width change (F1: b = 22 for k <= 2048, 21 above),
and special rows / columns (zero, non-finite, subnormal, huge)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2504_08009_b200.inputs import phi_matrix_np, integer_matrix_np

DEV = "cuda:0"


@pytest.fixture(scope="module")
def oz2():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2504_08009_b200 import build, oz2 as o
    build.build()
    return o


def _bitwise(got, ref, what):
    got = np.ascontiguousarray(got)
    ref = np.ascontiguousarray(ref)
    assert got.shape == ref.shape, (what, got.shape, ref.shape)
    diff = got.view(np.int64) != ref.view(np.int64)
    diff &= ~(np.isnan(got) & np.isnan(ref))
    n = int(diff.sum())
    if n:
        idx = np.argwhere(diff)[:5]
        raise AssertionError(f"{what}: {n} of {diff.size} differ, e.g. "
                             f"{[(tuple(i), got[tuple(i)], ref[tuple(i)]) for i in idx]}")


def test_tables_match_oracle(oz2, oracle):
    for s, q in ((2, 1), (16, 1024), (16, 2049), (22, 65536)):
        t = oz2.fp64mod_tables(s, q)
        o = oracle.fp64_constants(s, q)
        assert t["moduli"] == o["moduli"] and t["M"] == o["M"] and t["L"] == o["L"] and t["T"] == o["T"]


@pytest.mark.parametrize("m,n,k,s,v,phi", [
    (70, 90, 300, 16, 3, 0.5),
    (129, 257, 1024, 16, 2, 1.0),
    (33, 40, 2048, 8, 2, 2.0),      # b = 22 at the Eq. 19 boundary k m^2 <= 2^55
    (33, 40, 2049, 12, 2, 2.0),     # b = 21 above it
    (64, 64, 64, 2, 1, 0.5),
    (50, 61, 777, 22, 4, 4.0),
    (17, 300, 129, 5, 1, 1.0),
])
def test_fp64mod_vs_oracle(oz2, oracle, m, n, k, s, v, phi):
    A = phi_matrix_np(m, k, phi, seed=900 + m)
    B = phi_matrix_np(k, n, phi, seed=901 + n)
    C = oz2.dgemm_fp64mod(torch.from_numpy(A).to(DEV), torch.from_numpy(B).to(DEV), s, v).cpu().numpy()
    _bitwise(C, oracle.fp64_dgemm(A, B, s, v), f"fp64mod m={m} n={n} k={k} s={s} v={v}")


def test_fp64mod_special_values(oz2, oracle):
    m, n, k = 40, 36, 500
    A = phi_matrix_np(m, k, 1.0, seed=911)
    B = phi_matrix_np(k, n, 1.0, seed=912)
    A[3] = 0.0
    B[:, 5] = 0.0
    A[6, 7] = np.nan
    B[8, 9] = np.inf
    A[10] *= 2.0 ** -1060
    B[:, 11] *= 2.0 ** 800
    for s, v in ((10, 2), (16, 3)):
        C = oz2.dgemm_fp64mod(torch.from_numpy(A).to(DEV), torch.from_numpy(B).to(DEV), s, v).cpu().numpy()
        _bitwise(C, oracle.fp64_dgemm(A, B, s, v), f"special values s={s}")


def test_fp64mod_integer_inputs_exact(oz2):
    """Integer inputs within the budget: the words sum to AB exactly."""
    A = integer_matrix_np(30, 200, 2**25, seed=913)
    B = integer_matrix_np(200, 20, 2**25, seed=914)
    C = oz2.dgemm_fp64mod(torch.from_numpy(A).to(DEV), torch.from_numpy(B).to(DEV), 12, 3).cpu().numpy()
    exact = [[sum(int(a) * int(b) for a, b in zip(A[i], B[:, j])) for j in range(20)] for i in range(30)]
    from fractions import Fraction
    for i in range(30):
        for j in range(20):
            assert sum(Fraction(x) for x in C[:, i, j]) == exact[i][j]


def test_fp64mod_errors(oz2):
    A = torch.ones((4, 4), dtype=torch.float64, device=DEV)
    with pytest.raises(oz2.Oz2Error):
        oz2.dgemm_fp64mod(A, A, 23, 2)
    with pytest.raises(oz2.Oz2Error):
        oz2.dgemm_fp64mod(A, A, 1, 2)
    with pytest.raises(oz2.Oz2Error):
        oz2.dgemm_fp64mod(A, A, 16, 5)


def test_fp64mod_products_exact_at_the_eq20_bound(oz2, oracle):
    """Eq. (20): |C'_t| <= q (m_t/2)^2 <= 2^53 keeps the FP64 residue GEMMs
    exact.  Constant A (value c) and B (value d) rows give C'_t = k r_t(a') r_t(b')
    with every term of one sign; c, d are chosen (Python integers, from the
    oracle's exponents) so that some |C'_t| exceeds 2^52.9 at k = 2048, the
    largest k with 22-bit primes (k m^2 <= 2^55).  The GPU words must equal
    the oracle's, whose products are int64."""
    k, s, v = 2048, 16, 2
    mods = oracle.fp64_moduli(s, k)
    best = None
    for c in range(3, 4000, 2):
        A = np.full((1, k), float(c))
        C, e, f = oracle.fp64_dgemm(A, A.T.copy(), s, 1, want_exponents=True)
        ap = c * 2 ** int(e[0])
        rs = []
        for m in mods:
            r = ap % m
            rs.append(r - m if r > (m - 1) // 2 else r)
        worst = max(k * r * r for r in rs)
        if best is None or worst > best[0]:
            best = (worst, c)
        if worst > 2.0 ** 52.9:
            break
    worst, c = best
    assert worst > 2.0 ** 52.9 and worst <= 2 ** 53, (worst, c)
    A = np.full((64, k), float(c))
    A[1::2] *= -1.0                       # mixed signs across rows, one sign within a row
    B = A[:48].T.copy()
    got = oz2.dgemm_fp64mod(torch.from_numpy(A).to(DEV), torch.from_numpy(B).to(DEV), s, v).cpu().numpy()
    _bitwise(got, oracle.fp64_dgemm(A, B, s, v), "fp64mod at the Eq. 20 bound")


@pytest.mark.parametrize("m,n,k,s,v", [(40, 50, 300, 16, 3), (65, 33, 1024, 22, 4), (20, 20, 64, 8, 2)])
def test_fp64mod_double_word_inputs(oz2, oracle, m, n, k, s, v):
    """Double-word inputs (Eqs. 22-23, reading F6): A + A2, B + B2 with |A2| <=
    u |A|; every output word bitwise vs the oracle, which truncates the exact
    sum on a 2^-128 grid (the GPU uses trunc(x1) + an exact TwoSum adjustment).
    Includes integral first words with tiny second words of the other sign and
    second words that underflow when scaled."""
    rng = np.random.Generator(np.random.PCG64(m + n + k))
    A = phi_matrix_np(m, k, 1.0, seed=931 + m)
    B = phi_matrix_np(k, n, 1.0, seed=932 + n)
    A2 = A * 2.0 ** -53 * rng.uniform(-1, 1, A.shape)
    B2 = B * 2.0 ** -53 * rng.uniform(-1, 1, B.shape)
    A[0, :8] = np.round(A[0, :8] * 2.0 ** 40)          # integral after scaling, tiny opposite second words
    A2[0, :8] = -np.sign(A[0, :8]) * 1e-300
    A2[1, :4] = 5e-324 * np.sign(A[1, :4])
    B2[:, 0] = 0.0
    Ad, Bd = torch.from_numpy(A).to(DEV), torch.from_numpy(B).to(DEV)
    got = oz2.dgemm_fp64mod(Ad, Bd, s, v, A2=torch.from_numpy(A2).to(DEV), B2=torch.from_numpy(B2).to(DEV))
    _bitwise(got.cpu().numpy(), oracle.fp64_dgemm(A, B, s, v, A2=A2, B2=B2), f"double-word s={s} v={v}")
    one = oz2.dgemm_fp64mod(Ad, Bd, s, v, A2=torch.zeros_like(Ad))         # A2 = 0: the single-word result
    _bitwise(one.cpu().numpy(), oracle.fp64_dgemm(A, B, s, v), "A2 = 0")
