#!/usr/bin/env python
"""Throughput and accuracy of the FP64 prime-modulus regime (oz2_dgemm_fp64mod,
PAPER.md:508-557) against native cuBLAS DGEMM on the same inputs: emulated
TFLOPS (2mnk/t) per (s, v), and the componentwise error of the v-word result
against the exact product (Fractions, sampled entries).  Context for DESIGN.md
section 7 / profiles (not the headline bench).

    python tools/fp64mod_bench.py [n] [phi]
"""
import json
import os
import sys
from fractions import Fraction

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2504_08009_b200 import oz2  # noqa: E402
from paper_2504_08009_b200.inputs import SEED_A, SEED_B, phi_matrix_torch  # noqa: E402


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
    phi = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
    A = phi_matrix_torch(n, n, phi, SEED_A)
    B = phi_matrix_torch(n, n, phi, SEED_B)
    flops = 2.0 * n ** 3
    out = {"n": n, "phi": phi, "rows": []}
    ms = timed(lambda: torch.matmul(A, B))
    out["cublas_dgemm_tflops"] = flops / (ms * 1e-3) / 1e12
    Cd = torch.matmul(A, B)
    rng = np.random.Generator(np.random.PCG64(3))
    ii, jj = rng.integers(0, n, 12), rng.integers(0, n, 12)
    An, Bn = A.cpu().numpy(), B.cpu().numpy()
    exact = [sum(Fraction(a) * Fraction(b) for a, b in zip(An[i], Bn[:, j])) for i, j in zip(ii, jj)]
    absab = [float(np.abs(An[i]) @ np.abs(Bn[:, j])) for i, j in zip(ii, jj)]
    cd = Cd.cpu().numpy()
    out["cublas_dgemm_compwise"] = max(abs(float(Fraction(cd[i, j]) - x)) / w
                                       for (i, j), x, w in zip(zip(ii, jj), exact, absab))
    for s, v in ((8, 1), (12, 2), (16, 2), (16, 3), (20, 3), (22, 4)):
        C = oz2.dgemm_fp64mod(A, B, s, v)
        ms = timed(lambda: oz2.dgemm_fp64mod(A, B, s, v, out=C))
        Cn = C.cpu().numpy()
        err = max(abs(float(sum(Fraction(Cn[w, i, j]) for w in range(v)) - x)) / wgt
                  for (i, j), x, wgt in zip(zip(ii, jj), exact, absab))
        out["rows"].append({"s": s, "v": v, "ms": ms, "emulated_tflops": flops / (ms * 1e-3) / 1e12,
                            "compwise_err": err, "compwise_log2": float(np.log2(err)) if err > 0 else None})
        print(json.dumps(out["rows"][-1]), file=sys.stderr)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
