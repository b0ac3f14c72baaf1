#!/usr/bin/env python
"""Throughput and accuracy vs the number of moduli N (the metric's "vs moduli N"):
emulated FP64 TFLOPS at m = n = k = --n (default 16384) for N = 8..20, OS II-fast and
OS II-accu, plus the componentwise / relative error on sampled entries against an
exact reference, next to cuBLAS DGEMM's error on the same entries (BASELINE configs
[1]-[2]; PAPER.md:634-640 for the accuracy claims).  Prints a markdown table.

    python tools/sweep.py [--n 16384] [--phis 0.5,1,2] [--moduli 8..20]
"""
import argparse
import math
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from bench import exact_entries                       # bench-local exact reference (error-free products + fsum)
from paper_2504_08009_b200 import oz2
from paper_2504_08009_b200.inputs import phi_matrix_torch, SEED_A, SEED_B


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
    p = argparse.ArgumentParser()
    p.add_argument("--n", type=int, default=16384)
    p.add_argument("--phis", default="0.5,1,2")
    p.add_argument("--moduli", default="8..20")
    p.add_argument("--samples", type=int, default=128)
    p.add_argument("--modes", default="fast,accu")
    a = p.parse_args()
    lo, hi = (int(v) for v in a.moduli.split(".."))
    n = a.n
    flops = 2.0 * n ** 3
    print(f"| phi | N | mode | TFLOPS | compwise err (log2) | max rel err (log2) | cuBLAS DGEMM compwise (log2) |")
    print("|---|---|---|---|---|---|---|")
    for phi in (float(v) for v in a.phis.split(",")):
        A = phi_matrix_torch(n, n, phi, SEED_A, device="cuda")
        B = phi_matrix_torch(n, n, phi, SEED_B, device="cuda")
        rng = np.random.Generator(np.random.PCG64(3))
        ii = rng.integers(0, n, a.samples)
        jj = rng.integers(0, n, a.samples)
        it, jt = torch.from_numpy(ii).cuda(), torch.from_numpy(jj).cuda()
        ab, absab = exact_entries(A[it].cpu().numpy(), B[:, jt].cpu().numpy())
        Cd = torch.matmul(A, B)
        dg = Cd[it, jt].cpu().numpy()
        dg_err = math.log2(float(np.max(np.abs(dg - ab) / absab)))
        del Cd
        C = torch.empty((n, n), dtype=torch.float64, device="cuda")
        for N in range(lo, hi + 1):
            for mode in a.modes.split(","):
                ms = timed(lambda: oz2.dgemm(A, B, N, mode, out=C))
                c = C[it, jt].cpu().numpy()
                err = np.abs(c - ab)
                cw = float(np.max(err / absab))
                nz = ab != 0
                rel = float(np.max(err[nz] / np.abs(ab[nz])))
                l2 = lambda x: f"{math.log2(x):.1f}" if x > 0 else "exact"
                print(f"| {phi:g} | {N} | {mode} | {flops / ms / 1e9:.1f} | {l2(cw)} | {l2(rel)} | {dg_err:.1f} |",
                      flush=True)
        del A, B, C
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
