"""K-split (2-D multi-GPU) pieces on one GPU: the inner dimension is cut into
slices on the 256-chunk grid, each slice goes through the kslice statistics
phases, its own residues and reduced products, and oz2_crt_sum combines the
slices -- bitwise equal to the one-call product (the slice combination the
ranks would do with all-reduces is done here in the test).  Then the real
dist.dgemm_ksplit / dgemm_rowblock paths with two gloo ranks on cuda:0."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2504_08009_b200.inputs import phi_matrix_np

DEV = "cuda:0"


@pytest.fixture(scope="module")
def oz2():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2504_08009_b200 import build, oz2 as o
    build.build()
    return o


@pytest.mark.parametrize("mode,N", [("fast", 14), ("fast", 18), ("eq17", 14)])
def test_kslices_combine_bitwise(oz2, oracle, mode, N):
    from paper_2504_08009_b200.dist import kslice_partition
    m, n, k = 333, 290, 1500                               # slices 512 / 512 / 476 (ragged)
    A = phi_matrix_np(m, k, 2.0, seed=111)
    B = phi_matrix_np(k, n, 2.0, seed=112)
    A[4] = 0.0
    A[6, 1200] = np.inf                                    # non-finite entry in the last slice
    B[:, 9] *= 1e-300
    Ad, Bd = torch.from_numpy(A).to(DEV), torch.from_numpy(B).to(DEV)
    G = 3
    sl = [kslice_partition(k, G, r) for r in range(G)]
    EA = [oz2.kslice_stats_rows(Ad[:, a:b], mode=mode) for a, b in sl]
    EB = [oz2.kslice_stats_cols(Bd[a:b], mode=mode) for a, b in sl]
    EAg = torch.stack(EA).max(0).values
    EBg = torch.stack(EB).max(0).values
    SA = sum(oz2.kslice_stats_rows(Ad[:, a:b], EAg, mode=mode) for a, b in sl)
    SB = sum(oz2.kslice_stats_cols(Bd[a:b], EBg, mode=mode) for a, b in sl)
    e = oz2.exponents_from_stats(EAg, SA, k, N, mode)
    f = oz2.exponents_from_stats(EBg, SB, k, N, mode)
    mo = {"fast": oracle.MODE_FAST, "eq17": oracle.MODE_EQ17}[mode]
    assert np.array_equal(e.cpu().numpy(), oracle.scale_rows(A, N, mo)), "e from slice statistics"
    assert np.array_equal(f.cpu().numpy(), oracle.scale_cols(B, N, mo)), "f from slice statistics"
    parts = []
    for a, b in sl:
        Ar = oz2.residues_rows(Ad[:, a:b].contiguous(), e, N)
        Br = oz2.residues_cols(Bd[a:b].contiguous(), f, N)
        parts.append(oz2.modmul_residues(Ar, Br, b - a))
    R = torch.cat(parts)                                   # [G][N][m][n]
    C = oz2.crt_sum(R, G, N * m * n, m, n, e, f, N).cpu().numpy()
    ref = oz2.dgemm(Ad, Bd, N, mode).cpu().numpy()
    assert np.array_equal(C.view(np.int64), ref.view(np.int64)), "K-split combination"
    assert np.array_equal(ref.view(np.int64), oracle.dgemm(A, B, N, mo).view(np.int64))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    import torch.distributed as dist
    from paper_2504_08009_b200 import oz2
    from paper_2504_08009_b200.dist import dgemm_ksplit, dgemm_rowblock, kslice_partition, row_partition
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        m, n, k, N = 700, 650, 2300, 15
        A = torch.from_numpy(phi_matrix_np(m, k, 1.0, seed=121)).to(DEV)
        B = torch.from_numpy(phi_matrix_np(k, n, 1.0, seed=122)).to(DEV)
        a, b = kslice_partition(k, world, rank)
        _, Ck = dgemm_ksplit(A[:, a:b].contiguous(), B[a:b].contiguous(), k, N)
        r0, r1 = row_partition(m, world, rank)
        Bb = B.clone() if rank == 0 else torch.empty_like(B)
        _, Cr = dgemm_rowblock(A[r0:r1].contiguous(), Bb, N, m_total=m, chunks=2)
        from paper_2504_08009_b200.dist import dgemm_rowblock_panels
        # B in 2 column panels (512-aligned: 512 + 138 columns), C gathered per panel
        _, Cp = dgemm_rowblock_panels(A[r0:r1].contiguous(), B if rank == 0 else None, N, m_total=m, panels=2,
                                      n=n)
        if rank == 0:
            ref = oz2.dgemm(A, B, N)
            np.save(out, np.stack([Ck.cpu().numpy(), Cr.cpu().numpy(), Cp.cpu().numpy(), ref.cpu().numpy()]))
    finally:
        dist.destroy_process_group()


def test_dist_ksplit_and_rowblock_two_ranks_one_gpu(oz2, tmp_path):
    import torch.multiprocessing as mp
    out = str(tmp_path / "k.npy")
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    Ck, Cr, Cp, ref = np.load(out)
    assert np.array_equal(Ck.view(np.int64), ref.view(np.int64)), "dgemm_ksplit"
    assert np.array_equal(Cr.view(np.int64), ref.view(np.int64)), "dgemm_rowblock (prepared B, pieces)"
    assert np.array_equal(Cp.view(np.int64), ref.view(np.int64)), "dgemm_rowblock_panels (prepared A, B panels)"
