#!/usr/bin/env python
"""Latency of small emulated DGEMMs (config c1 and neighbours): eager calls vs a
CUDA-graph replay of the same call (the launch-bound regime).

    python tools/latency.py
"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2504_08009_b200 import oz2
from paper_2504_08009_b200.inputs import phi_matrix_torch, SEED_A, SEED_B


def us(fn, reps=200):
    for _ in range(10):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


print("| m = n = k | N | eager (us) | CUDA graph (us) | native DGEMM (us) |")
print("|---|---|---|---|---|")
for n in (64, 256, 1024, 2048):
    A = phi_matrix_torch(n, n, 0.5, SEED_A, device="cuda")
    B = phi_matrix_torch(n, n, 0.5, SEED_B, device="cuda")
    C = torch.empty((n, n), dtype=torch.float64, device="cuda")
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        oz2.dgemm(A, B, 14, out=C)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            oz2.dgemm(A, B, 14, out=C)
    torch.cuda.current_stream().wait_stream(s)
    t_e = us(lambda: oz2.dgemm(A, B, 14, out=C))
    t_g = us(lambda: g.replay())
    t_d = us(lambda: torch.matmul(A, B))
    print(f"| {n} | 14 | {t_e:.1f} | {t_g:.1f} | {t_d:.1f} |", flush=True)
