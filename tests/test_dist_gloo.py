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


def _oracle_scale_accu(A_local, B, N):
    import oracle
    e, f, _, _ = oracle.scale_accu(A_local.numpy(), B.numpy(), N)
    return torch.from_numpy(e), torch.from_numpy(f)


def _oracle_scaled(A_local, B, e, f, N):
    import oracle
    e, f = e.numpy(), f.numpy()
    Ap = oracle.trunc_rows(A_local.numpy(), e)
    BpT = oracle.trunc_cols(B.numpy(), f)
    Cp = oracle.modmul(oracle.residues(Ap, N), oracle.residues(BpT, N))
    return torch.from_numpy(oracle.crt(Cp, e, f))


def _worker_accu(rank, world, port, m, n, k, N, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        A = phi_matrix_np(m, k, 4.0, seed=7)
        r0, r1 = row_partition(m, world, rank)
        A_local = torch.from_numpy(A[r0:r1].copy())
        B = torch.from_numpy(phi_matrix_np(k, n, 4.0, seed=8)) if rank == 0 else torch.empty((k, n), dtype=torch.float64)
        _, C_full = dgemm_rowblock(A_local, B, N, "accu", m_total=m, accu_fns=(_oracle_scale_accu, _oracle_scaled))
        if rank == 0:
            np.save(out_path, C_full.numpy())
    finally:
        dist.destroy_process_group()


def test_rowblock_accu_gloo_world2(tmp_path, oracle):
    """OS II-accu sharded by rows: the MIN all-reduce of the partial f reproduces
    the single-process accu exponents, so C is bit-identical (reading R18)."""
    m, n, k, N = 40, 23, 200, 16
    out = str(tmp_path / "Ca.npy")
    mp.spawn(_worker_accu, args=(2, _free_port(), m, n, k, N, out), nprocs=2, join=True)
    C = np.load(out)
    A = phi_matrix_np(m, k, 4.0, seed=7)
    B = phi_matrix_np(k, n, 4.0, seed=8)
    ref = oracle.dgemm(A, B, N, oracle.MODE_ACCU)
    assert np.array_equal(C.view(np.int64), ref.view(np.int64))
    # and the sharding matters: rank 0's rows alone give a different (larger) f somewhere
    _, f_full, _, _ = oracle.scale_accu(A, B, N)
    _, f_half, _, _ = oracle.scale_accu(A[:20], B, N)
    assert np.all(f_half >= f_full)


def _worker(rank, world, port, m, n, k, N, out_path, chunks=1):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        A = phi_matrix_np(m, k, 1.0, seed=5)
        r0, r1 = row_partition(m, world, rank)
        A_local = torch.from_numpy(A[r0:r1].copy())
        B = torch.from_numpy(phi_matrix_np(k, n, 1.0, seed=6)) if rank == 0 else torch.empty((k, n), dtype=torch.float64)
        C_local, C_full = dgemm_rowblock(A_local, B, N, "fast", local_fn=_oracle_local, m_total=m, chunks=chunks)
        if rank == 0:
            np.save(out_path, C_full.numpy())
        # the broadcast delivered B everywhere
        Bref = phi_matrix_np(k, n, 1.0, seed=6)
        assert np.array_equal(B.numpy(), Bref)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("m,chunks", [(37, 1), (64, 1), (37, 3), (64, 4)])
def test_rowblock_gloo_world2(tmp_path, oracle, m, chunks):
    """chunks > 1: the pipelined gather (piece c transfers while c + 1 computes)
    reassembles the rows in order, ragged pieces included."""
    n, k, N = 29, 300, 14
    out = str(tmp_path / "C.npy")
    mp.spawn(_worker, args=(2, _free_port(), m, n, k, N, out, chunks), nprocs=2, join=True)
    C = np.load(out)
    A = phi_matrix_np(m, k, 1.0, seed=5)
    B = phi_matrix_np(k, n, 1.0, seed=6)
    ref = oracle.dgemm(A, B, N)
    assert C.shape == (m, n)
    assert np.array_equal(C.view(np.int64), ref.view(np.int64))


class _OraclePanelOps:
    """CPU stand-in for dist.Oz2PanelOps: 'prepared' operands are the matrices,
    the product is the oracle (FAST): the host logic of the panel pipeline
    (panel packing, broadcast, per-panel gather, reassembly) is what is tested."""

    def __init__(self, N):
        self.N = N

    def prepare_a(self, A):
        return A.clone()

    def prepare_b(self, Bp, slot):
        return Bp.clone()

    def product(self, pa, pb, out):
        import oracle
        out.copy_(torch.from_numpy(oracle.dgemm(pa.numpy(), pb.numpy(), self.N)))


def _worker_panels(rank, world, port, m, n, k, N, panels, out_path):
    from paper_2504_08009_b200.dist import dgemm_rowblock_panels
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        A = phi_matrix_np(m, k, 1.0, seed=17)
        r0, r1 = row_partition(m, world, rank)
        A_local = torch.from_numpy(A[r0:r1].copy())
        B = torch.from_numpy(phi_matrix_np(k, n, 1.0, seed=18)) if rank == 0 else None
        _, C_full = dgemm_rowblock_panels(A_local, B, N, m_total=m, panels=panels, ops=_OraclePanelOps(N), n=n)
        if rank == 0:
            np.save(out_path, C_full.numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("m,n,panels", [(37, 1300, 3), (8, 700, 4), (5, 1030, 1)])
def test_rowblock_panels_gloo_world2(tmp_path, oracle, m, n, panels):
    """B broadcast in 512-column-aligned panels (ragged last panel), C gathered
    per panel and reassembled on rank 0 (ragged row blocks): bit-identical to
    the single-process product (f_j depends on column j only, reading R4)."""
    from paper_2504_08009_b200.dist import panel_partition
    k, N = 300, 14
    pl = panel_partition(n, panels)
    assert pl[0][0] == 0 and pl[-1][1] == n and all(c0 % 512 == 0 for c0, _ in pl)
    out = str(tmp_path / "c.npy")
    mp.spawn(_worker_panels, args=(2, _free_port(), m, n, k, N, panels, out), nprocs=2, join=True)
    C = np.load(out)
    ref = oracle.dgemm(phi_matrix_np(m, k, 1.0, seed=17), phi_matrix_np(k, n, 1.0, seed=18), N)
    assert np.array_equal(C.view(np.int64), ref.view(np.int64))
