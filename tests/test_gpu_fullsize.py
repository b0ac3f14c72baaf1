"""BASELINE.json configs at full size, in the launch configuration bench.py
times (the default handle, oz2_dgemm on device-resident inputs): sampled
outputs bitwise against the oracle, computed entry block by entry block, and
the north-star accuracy gate on the same samples.

  configs[2]: m = n = k = 16384, N = 14, phi = 1 (the headline)
  configs[3]: m = n = k = 32768, N = 16 (one GPU's share of the sharded case
              is a row block of it; here the whole product on one GPU)
  configs[4]: m = n = 8192, k = 65536, phi = 4, N = 20 (large k, wide range)
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


def _check(oz2, oracle, m, n, k, N, phi, nrows, ncols, full_rows, mode="fast", full_cols=()):
    A = phi_matrix_torch(m, k, phi, SEED_A, device=DEV)
    B = phi_matrix_torch(k, n, phi, SEED_B, device=DEV)
    C = oz2.dgemm(A, B, N, mode)
    rng = np.random.Generator(np.random.PCG64(7))
    rows = np.sort(rng.choice(m, nrows, replace=False))
    cols = np.sort(rng.choice(n, ncols, replace=False))
    # the last rows / columns too (ragged last tile when m, n are not tile multiples)
    rows[-1], cols[-1] = m - 1, n - 1
    Ar = A[torch.from_numpy(rows).to(DEV)].cpu().numpy()
    Bc = B[:, torch.from_numpy(cols).to(DEV)].cpu().numpy()
    got = C[torch.from_numpy(rows).to(DEV)][:, torch.from_numpy(cols).to(DEV)].cpu().numpy()
    ref = oracle.dgemm(Ar, Bc, N, {"fast": oracle.MODE_FAST, "accu": oracle.MODE_ACCU}[mode])
    if mode == "fast":
        # FAST exponents are per row / per column: a sub-block of A and B gives the same bits
        bad = int((got.view(np.int64) != ref.view(np.int64)).sum())
        assert bad == 0, f"{bad} sampled entries differ"
        for i in full_rows:
            row = C[i].cpu().numpy()
            ref_row = oracle.dgemm(A[i:i + 1].cpu().numpy(), B.cpu().numpy(), N)[0]
            assert np.array_equal(row.view(np.int64), ref_row.view(np.int64)), f"row {i}"
        for j in full_cols:
            col = C[:, j].cpu().numpy()
            ref_col = oracle.dgemm(A.cpu().numpy(), B[:, j:j + 1].cpu().numpy(), N)[:, 0]
            assert np.array_equal(col.view(np.int64), ref_col.view(np.int64)), f"column {j}"
    ii, jj = np.meshgrid(np.arange(nrows), np.arange(ncols), indexing="ij")
    ab, absab = oracle.exact_entries(Ar, Bc, ii.ravel(), jj.ravel())
    return float(np.max(np.abs(got.ravel() - ab) / absab))


def test_config2_headline(oz2, oracle):
    # sampled 32 x 32 block + 2 full rows (first / last: ragged-free edge tiles)
    # and 2 full columns, every entry bitwise
    err = _check(oz2, oracle, 16384, 16384, 16384, 14, 1.0, 32, 32, full_rows=[0, 16383],
                 full_cols=[0, 16383])
    assert err < 2.0 ** -48, err                            # N = 14 at phi = 1: ~2^-50 (DESIGN R14)


def test_config2_gate_n15(oz2, oracle):
    err = _check(oz2, oracle, 16384, 16384, 16384, 15, 1.0, 24, 24, full_rows=[])
    assert err <= 2.0 ** -50, err                           # north-star accuracy gate


def test_config3_32768(oz2, oracle):
    _check(oz2, oracle, 32768, 32768, 32768, 16, 1.0, 12, 12, full_rows=[])


def test_config4_large_k_wide_range(oz2, oracle):
    err = _check(oz2, oracle, 8192, 8192, 65536, 20, 4.0, 12, 12, full_rows=[])
    assert err <= 2.0 ** -48, err
