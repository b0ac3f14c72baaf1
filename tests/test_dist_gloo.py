"""Host-side logic of the row-block multi-GPU path, on CPU with gloo, world size 2.

The local block product is the oracle (a CPU stand-in injected by the test;
the product path itself has no CPU fallback).  Checks: the partition, the B
broadcast, the ragged gather, and that the gathered result equals the
single-process result bit for bit (e_i depends only on row i, f_j only on
column j of B).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2504_08009_b200.dist import row_partition, dgemm_rowblock
from paper_2504_08009_b200.inputs import phi_matrix_np


def test_row_partition():
    for m in (0, 1, 7, 64, 1000):
        for world in (1, 2, 3, 8):
            parts = [row_partition(m, world, r) for r in range(world)]
            assert parts[0][0] == 0 and parts[-1][1] == m
            for (a0, a1), (b0, b1) in zip(parts, parts[1:]):
                assert a1 == b0
            sizes = [b - a for a, b in parts]
            assert max(sizes) - min(sizes) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _oracle_local(A_local, B, N, mode):
    import oracle
    C = oracle.dgemm(A_local.numpy(), B.numpy(), N, oracle.MODE_FAST if mode == "fast" else oracle.MODE_EQ17)
    return torch.from_numpy(C)


def _worker(rank, world, port, m, n, k, N, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        A = phi_matrix_np(m, k, 1.0, seed=5)
        r0, r1 = row_partition(m, world, rank)
        A_local = torch.from_numpy(A[r0:r1].copy())
        B = torch.from_numpy(phi_matrix_np(k, n, 1.0, seed=6)) if rank == 0 else torch.empty((k, n), dtype=torch.float64)
        C_local, C_full = dgemm_rowblock(A_local, B, N, "fast", local_fn=_oracle_local, m_total=m)
        if rank == 0:
            np.save(out_path, C_full.numpy())
        # the broadcast delivered B everywhere
        Bref = phi_matrix_np(k, n, 1.0, seed=6)
        assert np.array_equal(B.numpy(), Bref)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("m", [37, 64])
def test_rowblock_gloo_world2(tmp_path, oracle, m):
    n, k, N = 29, 300, 14
    out = str(tmp_path / "C.npy")
    mp.spawn(_worker, args=(2, _free_port(), m, n, k, N, out), nprocs=2, join=True)
    C = np.load(out)
    A = phi_matrix_np(m, k, 1.0, seed=5)
    B = phi_matrix_np(k, n, 1.0, seed=6)
    ref = oracle.dgemm(A, B, N)
    assert C.shape == (m, n)
    assert np.array_equal(C.view(np.int64), ref.view(np.int64))
