"""Multi-GPU Ozaki scheme II: output row-blocks of A per rank (north star:
"partitioned across the 8 B200s of one box by output row-blocks of A, with B
broadcast and C gathered over NVLink by NCCL").

Why row blocks need no other exchange: the exponent e_i of Alg. 1 line 1
depends only on row i of A and f_j only on column j of B (reading R4), so a
rank holding rows [r0, r1) of A and all of B computes exactly rows [r0, r1) of
the single-GPU result -- bit for bit.  One process per GPU, torch.distributed
(NCCL over NVLink / NVSwitch) for the two collectives.
"""
from __future__ import annotations

from typing import Callable, Optional


def row_partition(m: int, world: int, rank: int) -> tuple[int, int]:
    """Balanced contiguous row range [r0, r1) of rank `rank` (first m % world ranks get one more)."""
    base, extra = divmod(m, world)
    r0 = rank * base + min(rank, extra)
    return r0, r0 + base + (1 if rank < extra else 0)


def dgemm_rowblock(A_local, B, num_moduli: int = 14, mode: str = "fast", group=None, src: int = 0,
                   gather_to: Optional[int] = 0, m_total: Optional[int] = None,
                   local_fn: Optional[Callable] = None, accu_fns: Optional[tuple] = None,
                   chunks: int = 1, C_local=None):
    """C = A B with A sharded by rows.

    A_local: this rank's rows of A (rows `row_partition(m_total, world, rank)`).
    B:       the full k x n matrix on rank `src`; on the other ranks a tensor of
             the same shape and dtype to receive the broadcast into.
    Returns (C_local, C_full): C_full is the gathered m_total x n result on rank
    `gather_to` (None elsewhere, or everywhere when gather_to is None).

    local_fn(A_rows, B, num_moduli, mode) computes a block of rows; the default
    is the CUDA library: B is converted once (oz2.PreparedB, B-stationary) and
    every chunk of rows is one oz2_dgemm_prepared call.

    chunks > 1 pipelines the gather: the rows of every rank are cut into
    `chunks` pieces; piece c's gather (an asynchronous NCCL collective) runs
    while piece c + 1 computes, so only the last piece's transfer is exposed.
    (The caller leaves SMs to NCCL with oz2.set_sm_limit; results are
    bit-identical for any chunking.)

    mode "accu" (OS II-accu, reading R18): e_i needs row i and all of B (local),
    but f_j needs the bound P over ALL rows.  Each rank computes its partial f
    from its rows; since f_j = h_j - F_j with F_j common to all ranks and h_j
    non-increasing in max_i P_ij, the global f is the element-wise MIN over the
    ranks (one n-element int32 all-reduce) -- bit-identical to one GPU.
    accu_fns = (scale_fn(A_local, B, N) -> (e, f_partial), scaled_fn(A_local, B,
    e, f, N) -> C_local) replaces the CUDA library (oz2.scale_accu / dgemm_scaled).
    """
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    # gloo (CPU tests, or several ranks on one GPU as a functional check) moves
    # CUDA tensors through host copies; NCCL takes them directly
    host_coll = dist.get_backend(group) == "gloo" and B.is_cuda
    if host_coll:
        Bh = B.cpu()
        dist.broadcast(Bh, src=src, group=group)
        B.copy_(Bh)
    else:
        dist.broadcast(B, src=src, group=group)
    if m_total is None:
        sizes = torch.tensor([A_local.shape[0]], dtype=torch.int64, device=A_local.device)
        all_sizes = [torch.zeros_like(sizes) for _ in range(world)]
        dist.all_gather(all_sizes, sizes, group=group)
        rows = [int(v.item()) for v in all_sizes]
    else:
        rows = [row_partition(m_total, world, r)[1] - row_partition(m_total, world, r)[0] for r in range(world)]
    n = B.shape[1]
    if mode == "accu":
        if accu_fns is None:
            from . import oz2
            accu_fns = (oz2.scale_accu, oz2.dgemm_scaled)
        scale_fn, scaled_fn = accu_fns
        e, f = scale_fn(A_local, B, num_moduli)
        if host_coll:
            fh = f.cpu()
            dist.all_reduce(fh, op=dist.ReduceOp.MIN, group=group)
            f.copy_(fh)
        else:
            dist.all_reduce(f, op=dist.ReduceOp.MIN, group=group)
        res = scaled_fn(A_local, B, e, f, num_moduli)
        if C_local is None:
            C_local = res
        else:
            C_local.copy_(res)
        chunks = 1
        pieces = [C_local]
    else:
        if local_fn is None:
            from . import oz2
            prep = oz2.PreparedB(B, num_moduli, mode)
            block_fn = lambda a, out: prep.dgemm(a, out=out)
        else:
            def block_fn(a, out):
                out.copy_(local_fn(a, B, num_moduli, mode))
                return out
        if C_local is None:
            C_local = torch.empty((A_local.shape[0], n), dtype=torch.float64, device=A_local.device)
        chunks = max(1, int(chunks))
        pieces = []
    works, recv = [], []
    # the gathered result: pieces land directly in their rows of C_full when no
    # padding is needed (every rank's piece c has the same size)
    C_full = None
    rstart = [sum(rows[:r]) for r in range(world)]
    if gather_to is not None and rank == gather_to:
        C_full = torch.empty((sum(rows), n), dtype=torch.float64, device="cpu" if host_coll else B.device)
    for c in range(chunks):
        # piece c of every rank: rows row_partition(rows[r], chunks, c) of that rank's block
        pr = [row_partition(rr, chunks, c) for rr in rows]
        p0, p1 = pr[rank]
        if mode != "accu":
            if p1 > p0:
                block_fn(A_local[p0:p1], C_local[p0:p1])
            piece = C_local[p0:p1]
        else:
            piece = pieces[0]
        if gather_to is None:
            continue
        mr = max(b - a for a, b in pr)
        if piece.shape[0] < mr:
            send = torch.zeros((mr, n), dtype=C_local.dtype, device=C_local.device)
            send[:piece.shape[0]] = piece
        else:
            send = piece.contiguous()
        cdev = "cpu" if host_coll else C_local.device
        if host_coll:
            send = send.cpu()
        bufs, direct = None, all(b - a == mr for a, b in pr)
        if rank == gather_to:
            if direct:
                bufs = [C_full[rstart[r] + pr[r][0]: rstart[r] + pr[r][1]] for r in range(world)]
            else:
                bufs = [torch.empty((mr, n), dtype=C_local.dtype, device=cdev) for _ in range(world)]
        works.append(dist.gather(send, bufs, dst=gather_to, group=group, async_op=True))
        recv.append((bufs, pr, send, direct))
    for w in works:
        w.wait()
    if gather_to is None or rank != gather_to:
        return C_local, None
    for bufs, pr, _, direct in recv:                 # padded pieces: copy into place
        if not direct:
            for r in range(world):
                a, b = pr[r]
                C_full[rstart[r] + a: rstart[r] + b] = bufs[r][:b - a]
    return C_local, C_full.to(C_local.device)
