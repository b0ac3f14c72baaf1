"""Accuracy of the CUDA path against the exact product (oracle's Kulisch
reference) on config c2-shaped inputs (n = 4096, phi-controlled).

North star: within 2^-50 (|A||B|)_ij componentwise at the N the paper reports
as DGEMM-equivalent for phi <= 1 ("14 or 15 moduli"); error falls
with N until the FP64 floor (Eqs. 15-17).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2504_08009_b200.inputs import phi_matrix_torch, SEED_A, SEED_B

DEV = "cuda:0"


@pytest.fixture(scope="module")
def oz2():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2504_08009_b200 import build, oz2 as o
    build.build()
    return o


def _compwise(C, A_np_rows, B_np_cols, ii, jj, oracle):
    ab, absab = oracle.exact_entries(A_np_rows, B_np_cols, np.arange(len(ii)), np.arange(len(jj)))
    return float(np.max(np.abs(C[ii, jj] - ab) / absab))


@pytest.mark.parametrize("phi", [0.5, 1.0, 2.0])
def test_error_vs_N_c2(oz2, oracle, phi):
    n = 4096
    A = phi_matrix_torch(n, n, phi, SEED_A, device=DEV)
    B = phi_matrix_torch(n, n, phi, SEED_B, device=DEV)
    rng = np.random.Generator(np.random.PCG64(3))
    ii = rng.integers(0, n, 128)
    jj = rng.integers(0, n, 128)
    Ar = A[torch.from_numpy(ii).to(DEV)].cpu().numpy()
    Bc = B[:, torch.from_numpy(jj).to(DEV)].cpu().numpy()
    # pair p uses row p of Ar and column p of Bc
    errs = {}
    for N in (8, 10, 12, 14, 15, 16, 18, 20):
        C = oz2.dgemm(A, B, N).cpu().numpy()
        errs[N] = _compwise(C, Ar, Bc, ii, jj, oracle)
    dg = torch.matmul(A, B).cpu().numpy()
    dgemm_err = _compwise(dg, Ar, Bc, ii, jj, oracle)
    for a, b in [(8, 10), (10, 12), (12, 14)]:
        assert errs[b] < errs[a] / 16, errs                    # ~4 bits per modulus pre-floor
    if phi <= 1.0:
        assert errs[15] <= 2.0 ** -50, errs                    # north-star gate
        assert errs[15] <= 2 * max(dgemm_err, 2.0 ** -53), (errs, dgemm_err)
    assert errs[20] <= 2.0 ** -50 * (4 if phi > 1 else 1), errs
