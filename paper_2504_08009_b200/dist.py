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
                   local_fn: Optional[Callable] = None, accu_fns: Optional[tuple] = None):
    """C = A B with A sharded by rows.

    A_local: this rank's rows of A (rows `row_partition(m_total, world, rank)`).
    B:       the full k x n matrix on rank `src`; on the other ranks a tensor of
             the same shape and dtype to receive the broadcast into.
    Returns (C_local, C_full): C_full is the gathered m_total x n result on rank
    `gather_to` (None elsewhere, or everywhere when gather_to is None).

    local_fn(A_local, B, num_moduli, mode) computes the local block; the default
    is the CUDA library (paper_2504_08009_b200.oz2.dgemm).

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
    if local_fn is None:
        from . import oz2
        local_fn = oz2.dgemm
    dist.broadcast(B, src=src, group=group)
    if mode == "accu":
        if accu_fns is None:
            from . import oz2
            accu_fns = (oz2.scale_accu, oz2.dgemm_scaled)
        scale_fn, scaled_fn = accu_fns
        e, f = scale_fn(A_local, B, num_moduli)
        dist.all_reduce(f, op=dist.ReduceOp.MIN, group=group)
        C_local = scaled_fn(A_local, B, e, f, num_moduli)
    else:
        C_local = local_fn(A_local, B, num_moduli, mode)
    if gather_to is None:
        return C_local, None
    if m_total is None:
        sizes = torch.tensor([A_local.shape[0]], dtype=torch.int64, device=C_local.device)
        all_sizes = [torch.zeros_like(sizes) for _ in range(world)]
        dist.all_gather(all_sizes, sizes, group=group)
        rows = [int(s.item()) for s in all_sizes]
    else:
        rows = [row_partition(m_total, world, r)[1] - row_partition(m_total, world, r)[0] for r in range(world)]
    # dist.gather needs equal shapes: pad every block to the largest
    mr = max(rows)
    n = C_local.shape[1]
    if C_local.shape[0] < mr:
        pad = torch.zeros((mr, n), dtype=C_local.dtype, device=C_local.device)
        pad[:C_local.shape[0]] = C_local
        send = pad
    else:
        send = C_local.contiguous()
    if rank == gather_to:
        bufs = [torch.empty((mr, n), dtype=C_local.dtype, device=C_local.device) for _ in range(world)]
        dist.gather(send, bufs, dst=gather_to, group=group)
        C_full = torch.cat([b[:r] for b, r in zip(bufs, rows)], dim=0)
        return C_local, C_full
    dist.gather(send, None, dst=gather_to, group=group)
    return C_local, None
