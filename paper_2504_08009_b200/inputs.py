"""Seeded synthetic inputs shared by the tests, the oracle runs and bench.py.

This module holds no arithmetic of the method: it only draws the paper's test
matrices (Sec. 4.1)

    a_ij, b_ij = (rand - 0.5) * exp(phi * randn),   rand in (0, 1], randn ~ N(0, 1)

(reading R15: rand = 1 - U with U ~ U[0, 1)), plus a few structured special
cases used as edge tests.  phi controls the spread of exponents; phi = 0.5 is
"comparable to" HPL.

Device generation is blocked by 1024 rows so that a matrix is identical for
any sharding across GPUs: block b of a matrix with base seed s uses the seed
s * 2**20 + b, drawing U before Z.
"""
from __future__ import annotations

import numpy as np

ROW_BLOCK = 1024
SEED_A = 1
SEED_B = 2


def phi_matrix_np(rows: int, cols: int, phi: float, seed: int) -> np.ndarray:
    """Host (numpy PCG64) version, used for oracle-sized cases."""
    g = np.random.Generator(np.random.PCG64(seed))
    u = 1.0 - g.random((rows, cols))          # (0, 1]
    z = g.standard_normal((rows, cols))
    return (u - 0.5) * np.exp(phi * z)


def phi_matrix_torch(rows: int, cols: int, phi: float, seed: int, device="cuda",
                     row_offset: int = 0, out=None):
    """Device version (torch.Generator on `device`), blocked by ROW_BLOCK rows.

    Produces rows [row_offset, row_offset + rows) of the matrix with base seed
    `seed`; any row range gives the same values as the full matrix.
    """
    import torch

    if out is None:
        out = torch.empty((rows, cols), dtype=torch.float64, device=device)
    g = torch.Generator(device=device)
    r = 0
    while r < rows:
        gr = row_offset + r
        blk = gr // ROW_BLOCK
        g.manual_seed(seed * 2**20 + blk)       # every block draws ROW_BLOCK full rows
        u = torch.rand((ROW_BLOCK, cols), generator=g, dtype=torch.float64, device=device)
        z = torch.randn((ROW_BLOCK, cols), generator=g, dtype=torch.float64, device=device)
        lo = gr - blk * ROW_BLOCK
        take = min(ROW_BLOCK - lo, rows - r)
        u = u[lo:lo + take]
        z = z[lo:lo + take]
        out[r:r + take].copy_((1.0 - u - 0.5) * torch.exp(phi * z))
        r += take
    return out


def integer_matrix_np(rows: int, cols: int, bound: int, seed: int) -> np.ndarray:
    """Integer-valued FP64 matrix with entries in [-bound, bound]."""
    g = np.random.Generator(np.random.PCG64(seed))
    return g.integers(-bound, bound + 1, size=(rows, cols)).astype(np.float64)


def dyadic_matrix_np(rows: int, cols: int, mant_bits: int, exp_range: int, seed: int) -> np.ndarray:
    """Entries +-m * 2^x with m < 2^mant_bits and |x| <= exp_range: short
    mantissas, so a modest power-of-two scaling makes them integers."""
    g = np.random.Generator(np.random.PCG64(seed))
    m = g.integers(0, 2**mant_bits, size=(rows, cols)).astype(np.float64)
    s = g.choice([-1.0, 1.0], size=(rows, cols))
    x = g.integers(-exp_range, exp_range + 1, size=(rows, cols))
    return s * np.ldexp(m, x)
