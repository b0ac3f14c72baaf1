#!/usr/bin/env python
"""One small product through the library for compute-sanitizer runs
(tools/gpu/r02_sanitize.sh): oz2_dgemm (the fused path or the unit-parallel
path by shape), the OS II-accu rule, the split API and the FP64 prime regime,
each checked bitwise against the oracle.

    python tools/sanitize_case.py M N K [N_moduli]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
from paper_2504_08009_b200 import oz2  # noqa: E402
from paper_2504_08009_b200.inputs import phi_matrix_np  # noqa: E402


def main():
    m, n, k = (int(x) for x in sys.argv[1:4])
    N = int(sys.argv[4]) if len(sys.argv) > 4 else 14
    A = phi_matrix_np(m, k, 1.0, seed=1)
    B = phi_matrix_np(k, n, 1.0, seed=2)
    Ad, Bd = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    bad = 0
    C = oz2.dgemm(Ad, Bd, N).cpu().numpy()
    bad += int((C.view(np.int64) != oracle.dgemm(A, B, N).view(np.int64)).sum())
    if k < 2**17:
        Ca = oz2.dgemm(Ad, Bd, N, mode="accu").cpu().numpy()
        bad += int((Ca.view(np.int64) != oracle.dgemm(A, B, N, oracle.MODE_ACCU).view(np.int64)).sum())
        e = oz2.scale_rows(Ad, N)
        f = oz2.scale_cols(Bd, N)
        Cp = oz2.modmul(oz2.residues_rows(Ad, e, N), oz2.residues_cols(Bd, f, N), k)
        Cc = oz2.crt(Cp, e, f, beta=oz2.certify(Ad, Bd, e, f, N)).cpu().numpy()
        bad += int((Cc.view(np.int64) != C.view(np.int64)).sum())
        oz2.status()
    if m * k < 2**22 and k * n < 2**22:
        F = oz2.dgemm_fp64mod(Ad, Bd, 16, 2).cpu().numpy()
        bad += int((F.view(np.int64) != oracle.fp64_dgemm(A, B, 16, 2).view(np.int64)).sum())
    torch.cuda.synchronize()
    print(f"sanitize case {m}x{n}x{k} N={N}: {bad} mismatches")
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
