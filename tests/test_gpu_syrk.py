"""oz2_dsyrk on the GPU, bitwise against the oracle (tests/test_oracle_syrk.py
pins the oracle): one conversion of op(A), the triangle's tiles of the fused
GEMM, and only the requested triangle of C read or written."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from paper_2504_08009_b200.inputs import phi_matrix_np

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


@pytest.fixture(scope="module")
def oz2():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2504_08009_b200 import build, oz2 as o
    build.build()
    return o


def _check(oz2, oracle, A, N, uplo, trans, alpha=1.0, beta=0.0, C0=None, mode="fast"):
    n = A.shape[1] if trans else A.shape[0]
    mo = {"fast": oracle.MODE_FAST, "eq17": oracle.MODE_EQ17, "accu": oracle.MODE_ACCU}[mode]
    Cin = phi_matrix_np(n, n, 1.0, seed=99) if C0 is None else C0
    Cd = torch.from_numpy(Cin.copy()).to(DEV)
    got = oz2.syrk(torch.from_numpy(A).to(DEV), N, uplo, trans, alpha, beta, Cd, mode).cpu().numpy()
    ref = oracle.syrk(A, N, uplo, trans, alpha, beta, Cin, mo)
    bad = int((got.view(np.int64) != ref.view(np.int64)).sum())
    assert bad == 0, f"syrk n={n} N={N} uplo={uplo} trans={trans} mode={mode}: {bad} entries differ"


@pytest.mark.parametrize("uplo", ["L", "U"])
@pytest.mark.parametrize("trans", [False, True])
def test_syrk_tiles_and_triangles(oz2, oracle, uplo, trans):
    # n = 700: 3 x 2 tiles of 256 x 512, diagonal tiles cut by the triangle, ragged edges
    n, k = 700, 333
    A = phi_matrix_np(k, n, 1.0, seed=11) if trans else phi_matrix_np(n, k, 1.0, seed=11)
    _check(oz2, oracle, A, 14, uplo, trans)


def test_syrk_alpha_beta_modes_and_N(oz2, oracle):
    A = phi_matrix_np(300, 257, 0.5, seed=12)
    _check(oz2, oracle, A, 14, "L", False, alpha=-2.0, beta=0.5)
    _check(oz2, oracle, A, 20, "U", False)                       # 96-bit residue path
    _check(oz2, oracle, A, 9, "L", False, mode="eq17")
    _check(oz2, oracle, A, 14, "U", False, mode="accu")


def test_syrk_special_values_and_degenerate(oz2, oracle):
    A = phi_matrix_np(150, 90, 1.0, seed=13)
    A[3] = 0.0
    A[7, 5] = np.nan                                              # non-finite row: NaN row and column
    A[9] *= 2.0 ** -1060
    _check(oz2, oracle, A, 14, "L", False)
    n = 40                                                        # alpha = 0 and k = 0: C := beta C on the triangle
    C0 = phi_matrix_np(n, n, 1.0, seed=14)
    _check(oz2, oracle, phi_matrix_np(n, 10, 1.0, seed=15), 14, "U", False, alpha=0.0, beta=3.0, C0=C0)
    _check(oz2, oracle, np.zeros((n, 0)), 14, "L", False, beta=0.0, C0=C0)


def test_syrk_many_tiles(oz2, oracle):
    # n = 2100: 9 x 5 tiles, about half of them skipped
    A = phi_matrix_np(2100, 200, 1.0, seed=16)
    _check(oz2, oracle, A, 14, "L", False)


@pytest.mark.parametrize("side", ["L", "R"])
@pytest.mark.parametrize("uplo", ["L", "U"])
@pytest.mark.parametrize("transA", [False, True])
def test_trmm(oz2, oracle, side, uplo, transA):
    # 600 x 700 B: several tiles, ragged edges; the per-tile K skipping of the zero
    # triangle must not change a bit against the oracle (which multiplies the zeros)
    m, n = 600, 700
    na = m if side == "L" else n
    A = phi_matrix_np(na, na, 1.0, seed=31)
    B = phi_matrix_np(m, n, 1.0, seed=32)
    for unit, alpha in ((False, 1.0), (True, -0.75)):
        Bd = torch.from_numpy(B.copy()).to(DEV)
        got = oz2.trmm(torch.from_numpy(A).to(DEV), Bd, 14, side, uplo, transA, unit, alpha).cpu().numpy()
        ref = oracle.trmm(A, B, 14, side, uplo, transA, unit, alpha)
        bad = int((got.view(np.int64) != ref.view(np.int64)).sum())
        assert bad == 0, f"trmm side={side} uplo={uplo} transA={transA} unit={unit}: {bad} entries differ"


def test_trmm_k_blocking_and_N20(oz2, oracle, monkeypatch):
    # forced K chunks (2 k-blocks each) inside the per-tile K ranges, and the 96-bit residue path
    monkeypatch.setenv("OZ2_KB_CHUNK", "2")
    A = phi_matrix_np(900, 900, 0.5, seed=33)
    B = phi_matrix_np(900, 300, 0.5, seed=34)
    for N in (14, 20):
        Bd = torch.from_numpy(B.copy()).to(DEV)
        got = oz2.trmm(torch.from_numpy(A).to(DEV), Bd, N, "L", "U").cpu().numpy()
        ref = oracle.trmm(A, B, N, "L", "U")
        assert int((got.view(np.int64) != ref.view(np.int64)).sum()) == 0, f"N={N}"
