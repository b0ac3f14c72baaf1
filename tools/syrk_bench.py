#!/usr/bin/env python
"""oz2_dsyrk vs oz2_dgemm_op on the same product at n = k (default 16384), N = 14:
time per call (CUDA events), DSYRK flop count k n (n + 1), and the written
triangle checked bitwise against the full GEMM's (both are Algorithm 1)."""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2504_08009_b200 import oz2
from paper_2504_08009_b200.inputs import phi_matrix_torch, SEED_A


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


p = argparse.ArgumentParser()
p.add_argument("--n", type=int, default=16384)
p.add_argument("--k", type=int, default=0)
p.add_argument("--N", type=int, default=14)
a = p.parse_args()
n, k = a.n, a.k or a.n
A = phi_matrix_torch(n, k, 1.0, SEED_A, device="cuda")
C1 = torch.zeros((n, n), dtype=torch.float64, device="cuda")
C2 = torch.zeros((n, n), dtype=torch.float64, device="cuda")
t_syrk = timed(lambda: oz2.syrk(A, a.N, "L", C=C1))
t_gemm = timed(lambda: oz2.gemm(A, A, a.N, transB=True, C=C2))
tri = torch.ones((n, n), dtype=torch.bool, device="cuda").tril()
same = torch.equal(C1.view(torch.int64)[tri], C2.view(torch.int64)[tri])
fl = k * n * (n + 1)
print(f"n={n} k={k} N={a.N}: syrk {t_syrk:.2f} ms ({fl / t_syrk / 1e9:.1f} TFLOPS, k n (n+1) flops), "
      f"gemm A A^T {t_gemm:.2f} ms ({2 * n * n * k / t_gemm / 1e9:.1f} TFLOPS); speed-up {t_gemm / t_syrk:.2f}x; "
      f"triangle bitwise equal: {same}")

# TRMM: B := op(tri(A)) B at m = n = k, against the full product with the masked matrix
from paper_2504_08009_b200.inputs import SEED_B
B = phi_matrix_torch(n, n, 1.0, SEED_B, device="cuda")
An = phi_matrix_torch(n, n, 1.0, SEED_A, device="cuda")
T = An.tril()
Bw = B.clone()
t_trmm = timed(lambda: (Bw.copy_(B), oz2.trmm(An, Bw, a.N, "L", "L")))
t_copy = timed(lambda: Bw.copy_(B))
Bw.copy_(B)
oz2.trmm(An, Bw, a.N, "L", "L")
C3 = oz2.gemm(T, B, a.N)
t_g = timed(lambda: oz2.gemm(T, B, a.N, C=C3))
same = torch.equal(Bw.view(torch.int64), C3.view(torch.int64))
t_trmm -= t_copy
print(f"n={n} N={a.N}: trmm {t_trmm:.2f} ms ({n * n * n / t_trmm / 1e9:.1f} TFLOPS, n^3 flops), "
      f"gemm tri(A) B {t_g:.2f} ms; speed-up {t_g / t_trmm:.2f}x; bitwise equal: {same}")
