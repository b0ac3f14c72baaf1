#!/usr/bin/env python
"""The oracle timed as SURVEY.md section 8(d) specifies ("Oracle timing beside
it"): c1 (64^3, N = 14, phi = 0.5) in full on 1 thread and on all cores; c2
(4096^3, N = 14, phi = 1) in full; c3 (16384^3, N = 14, phi = 1) on 16 full rows
of C, extrapolated x1024 and labelled as such.  Reported as emulated GFLOPS =
2 rows n k / t with the host's CPU model and core count.  A baseline, not the
target.  Run on the GPU box's host (tools/gpu/r02_oracle.sh) and summarised in
profiles/r02_oracle_timing.md.

    python tools/oracle_timing.py [--skip-c2] [--skip-c3]
"""
from __future__ import annotations

import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import oracle  # noqa: E402
from paper_2504_08009_b200.inputs import SEED_A, SEED_B, phi_matrix_np  # noqa: E402


def cpu_model() -> str:
    with open("/proc/cpuinfo") as fh:
        for line in fh:
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    return "unknown"


def timed(A, B, N):
    t0 = time.perf_counter()
    oracle.dgemm(A, B, N)
    return time.perf_counter() - t0


def main():
    skip_c2 = "--skip-c2" in sys.argv
    skip_c3 = "--skip-c3" in sys.argv
    cores = len(os.sched_getaffinity(0))
    out = {"cpu_model": cpu_model(), "cores": cores, "oracle_build": "gcc -O2 -fopenmp -ffp-contract=off"}
    # c1: full, 1 thread and all cores
    A = phi_matrix_np(64, 64, 0.5, seed=SEED_A)
    B = phi_matrix_np(64, 64, 0.5, seed=SEED_B)
    for thr in (1, cores):
        oracle.set_threads(thr)
        timed(A, B, 14)                                   # warm-up
        dt = min(timed(A, B, 14) for _ in range(5))
        out[f"c1_full_{thr}thr"] = {"s": dt, "gflops": 2 * 64 ** 3 / dt / 1e9, "threads": thr}
    oracle.set_threads(cores)
    if not skip_c2:
        n = 4096
        A = phi_matrix_np(n, n, 1.0, seed=SEED_A)
        B = phi_matrix_np(n, n, 1.0, seed=SEED_B)
        dt = timed(A, B, 14)
        out["c2_full"] = {"s": dt, "gflops": 2 * n ** 3 / dt / 1e9, "threads": cores}
    if not skip_c3:
        n = 16384
        B = phi_matrix_np(n, n, 1.0, seed=SEED_B)
        A = phi_matrix_np(32, n, 1.0, seed=SEED_A)
        t16 = timed(A[:16], B, 14)
        t32 = timed(A, B, 14)
        per_row = max(0.0, (t32 - t16) / 16)
        full = t16 + per_row * (n - 16)
        out["c3_16rows"] = {"s": t16, "gflops": 2 * 16 * n * n / t16 / 1e9, "threads": cores,
                            "s_32rows": t32, "per_row_s": per_row,
                            "extrapolated_full_s": full, "extrapolated_full_gflops": 2 * n ** 3 / full / 1e9,
                            "extrapolated_x1024_s": t16 * 1024,
                            "note": "16 full rows of C measured (the oracle converts all of B once per "
                                    "call); EXTRAPOLATED to the full product from the 16- and 32-row "
                                    "times (B's conversion once + the per-row cost), and x1024"}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
