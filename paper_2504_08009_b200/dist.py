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


def kslice_partition(k: int, world: int, rank: int, chunk: int = 256) -> tuple[int, int]:
    """Balanced K range [l0, l1) of rank `rank`, boundaries on the FAST rule's
    256-element chunk grid (reading R4) -- the last range takes the ragged tail."""
    nch = (k + chunk - 1) // chunk
    c0, c1 = row_partition(nch, world, rank)
    return min(k, c0 * chunk), min(k, c1 * chunk)


def dgemm_ksplit(A_ks, B_ks, k_total: int, num_moduli: int = 14, mode: str = "fast", group=None,
                 gather_to: Optional[int] = 0):
    """C = A B with the inner dimension split across the ranks (2-D / K-split
    multi-GPU): rank r holds A[:, K_r] (m x k_r) and B[K_r, :]
    (k_r x n), K_r = kslice_partition(k_total, world, r).  No operand is
    broadcast; the exchange is
      1. two all-reduces of the per-row / per-column statistics (int32 MAX, then
         uint64 SUM; m + n values each) that give the exponents of the whole
         product, bit-identical to one GPU (reading R4 is built from per-chunk
         integer statistics);
      2. one all-to-all of the rank's reduced partial residues c''_t (uint8,
         N bytes per element of C) so that every rank receives, for its own
         row block, the partial residues of all K slices;
    then oz2_crt_sum adds them mod m_t and runs lines 8-10.  Returns (C_local,
    C_full) like dgemm_rowblock: rank r's rows are row_partition(m, world, r)
    padded to equal blocks of ceil(m / world).  FAST / EQ17."""
    import torch
    import torch.distributed as dist
    from . import oz2

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    m, n = A_ks.shape[0], B_ks.shape[1]
    N = num_moduli
    host_coll = dist.get_backend(group) == "gloo" and A_ks.is_cuda

    def allreduce(t, op):
        if host_coll:
            th = t.cpu()
            dist.all_reduce(th, op=op, group=group)
            t.copy_(th)
        else:
            dist.all_reduce(t, op=op, group=group)

    # exponents of the whole product (phase 1: MAX of chunk exponents, phase 2: SUM)
    E = torch.cat([oz2.kslice_stats_rows(A_ks, mode=mode), oz2.kslice_stats_cols(B_ks, mode=mode)])
    allreduce(E, dist.ReduceOp.MAX)
    EA, EB = E[:m], E[m:]
    S = torch.cat([oz2.kslice_stats_rows(A_ks, EA, mode=mode), oz2.kslice_stats_cols(B_ks, EB, mode=mode)])
    allreduce(S, dist.ReduceOp.SUM)
    e = oz2.exponents_from_stats(EA, S[:m], k_total, N, mode)
    f = oz2.exponents_from_stats(EB.contiguous(), S[m:].contiguous(), k_total, N, mode)
    # residues of the local slices and their reduced products, laid out by destination row block
    k_loc = A_ks.shape[1]
    Ar = oz2.residues_rows(A_ks, e, N)
    Br = oz2.residues_cols(B_ks, f, N)
    rpb = (m + world - 1) // world
    if k_loc > 0:
        R = oz2.modmul_residues(Ar, Br, k_loc, rows_per_block=rpb)          # [ceil(m/rpb)][N][rpb][n]
    else:
        R = torch.zeros(((m + rpb - 1) // rpb, N, rpb, n), dtype=torch.uint8, device=A_ks.device)
    if R.shape[0] < world:                                                 # fewer rows than ranks
        R = torch.cat([R, torch.zeros((world - R.shape[0], N, rpb, n), dtype=torch.uint8, device=R.device)])
    recv = torch.empty_like(R)
    if host_coll:
        rh = torch.empty_like(R, device="cpu")
        dist.all_to_all_single(rh, R.cpu(), group=group)
        recv.copy_(rh)
    else:
        dist.all_to_all_single(recv, R, group=group)
    r0 = min(m, rank * rpb)
    r1 = min(m, r0 + rpb)
    C_local = torch.empty((r1 - r0, n), dtype=torch.float64, device=A_ks.device)
    if r1 > r0:
        oz2.crt_sum(recv, world, N * rpb * n, r1 - r0, n, e[r0:r1], f, N, out=C_local)
    if gather_to is None:
        return C_local, None
    send = torch.zeros((rpb, n), dtype=torch.float64, device=A_ks.device)
    send[:r1 - r0] = C_local
    if host_coll:
        send = send.cpu()
    bufs = [torch.empty_like(send) for _ in range(world)] if rank == gather_to else None
    dist.gather(send, bufs, dst=gather_to, group=group)
    if rank != gather_to:
        return C_local, None
    return C_local, torch.cat(bufs, dim=0)[:m].to(A_ks.device)


def panel_partition(n: int, panels: int, align: int = 512) -> list[tuple[int, int]]:
    """Column panels [c0, c1) of n columns, boundaries on multiples of `align`
    (the GEMM's 512-column pair tile), as even as that allows; empty panels dropped."""
    units = (n + align - 1) // align
    out = []
    for p in range(panels):
        a, b = row_partition(units, panels, p)
        c0, c1 = min(n, a * align), min(n, b * align)
        if c1 > c0:
            out.append((c0, c1))
    return out


class Oz2PanelOps:
    """The CUDA library behind dgemm_rowblock_panels: A converted once
    (oz2_prepare_a), each B panel converted into one of two reused objects
    (oz2_prepare_b / oz2_reprepare), lines 6-10 by oz2_dgemm_prep2."""

    def __init__(self, num_moduli: int, mode: str):
        from . import oz2
        self.oz2 = oz2
        self.N, self.mode = num_moduli, mode
        self.slots = {}

    def prepare_a(self, A):
        return self.oz2.PreparedA(A, self.N, self.mode)

    def prepare_b(self, Bp, slot: int):
        s = self.slots.get(slot)
        if s is not None and (s.k, s.n) == tuple(Bp.shape):
            return s.reprepare(Bp)
        s = self.oz2.PreparedB(Bp, self.N, self.mode)
        self.slots[slot] = s
        return s

    def product(self, pa, pb, out):
        self.oz2.dgemm_prep2(pa, pb, out=out)

    def close(self):
        for s in self.slots.values():
            s.release()
        self.slots.clear()


def dgemm_rowblock_panels(A_local, B, num_moduli: int = 14, mode: str = "fast", group=None, src: int = 0,
                          gather_to: Optional[int] = 0, m_total: Optional[int] = None, panels: int = 4,
                          C_local=None, C_full=None, ops=None, n: Optional[int] = None):
    """C = A B with A sharded by output rows and B broadcast from `src` in column
    panels ("Overlap mechanics" option 1), FAST / EQ17.

    Every rank converts its rows of A once; then for panel p (columns [c0, c1)
    on the 512-column tile grid) it waits for panel p's broadcast, converts it
    (f and the B planes of those columns: f_j depends on column j only) and runs
    the fused GEMM into C_local[:, c0:c1].  Panel p + 1 is packed (on `src`: a
    contiguous copy of the strided column block) and broadcast while panel p is
    converted and multiplied, and panel p's C block is gathered to `gather_to`
    while panel p + 1 computes -- one collective stream, overlapped with the
    compute stream.  Results are bit-identical to one GPU for any panel count.

    A_local: this rank's rows (row_partition(m_total, world, rank)); B: k x n
    on `src` (None elsewhere, with n given: the panels arrive in local buffers).  C_full
    (gather_to only, optional): the m_total x n result, row-major.  ops: the
    local operations (tests inject a CPU stand-in).  Returns (C_local, C_full)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    host_coll = dist.get_backend(group) == "gloo" and A_local.is_cuda
    dev = A_local.device
    k = A_local.shape[1]
    if n is None:
        n = B.shape[1]
    if m_total is None:
        sizes = torch.tensor([A_local.shape[0]], dtype=torch.int64, device=dev if not host_coll else "cpu")
        all_sizes = [torch.zeros_like(sizes) for _ in range(world)]
        dist.all_gather(all_sizes, sizes, group=group)
        rows = [int(v.item()) for v in all_sizes]
        m_total = sum(rows)
    else:
        rows = [b - a for a, b in (row_partition(m_total, world, r) for r in range(world))]
    m_loc = A_local.shape[0]
    mr = max(rows)
    own_ops = ops is None
    if ops is None:
        ops = Oz2PanelOps(num_moduli, mode)
    if C_local is None:
        C_local = torch.empty((m_loc, n), dtype=torch.float64, device=dev)
    pl = panel_partition(n, panels)
    npmax = max(c1 - c0 for c0, c1 in pl) if pl else 0
    cdev = "cpu" if host_coll else dev
    # two flat panel buffers; panel p is a contiguous k x (c1 - c0) view (collectives need contiguity)
    bufs = [torch.empty(k * npmax, dtype=torch.float64, device=cdev) for _ in range(min(2, len(pl)))]
    do_gather = gather_to is not None and world > 1
    if gather_to is not None and rank == gather_to and C_full is None:
        C_full = torch.empty((m_total, n), dtype=torch.float64, device=dev)
    rstart = [sum(rows[:r]) for r in range(world)]

    def bcast(p):
        c0, c1 = pl[p]
        buf = bufs[p % 2][:k * (c1 - c0)].view(k, c1 - c0)
        if rank == src:
            buf.copy_(B[:, c0:c1])                        # strided column block -> contiguous
        return dist.broadcast(buf, src=src, group=group, async_op=True), buf

    pa = ops.prepare_a(A_local) if m_loc > 0 else None
    pending = bcast(0) if pl else None
    gathers = []
    for p, (c0, c1) in enumerate(pl):
        work, buf = pending
        work.wait()                                       # compute stream waits for panel p
        if host_coll:
            bdev = buf.to(dev)
        else:
            bdev = buf
        if p + 1 < len(pl):
            pending = bcast(p + 1)                        # overlaps panel p's conversion + GEMM
        if m_loc > 0:
            pb = ops.prepare_b(bdev, p % 2)
            ops.product(pa, pb, C_local[:, c0:c1])
        if do_gather:
            send = torch.zeros((mr, c1 - c0), dtype=torch.float64, device=cdev)
            send[:m_loc] = C_local[:, c0:c1]
            recv = ([torch.empty((mr, c1 - c0), dtype=torch.float64, device=cdev) for _ in range(world)]
                    if rank == gather_to else None)
            gathers.append((dist.gather(send, recv, dst=gather_to, group=group, async_op=True), recv, c0, c1, send))
        elif gather_to is not None and rank == gather_to:
            C_full[:, c0:c1] = C_local[:, c0:c1]
    for w, recv, c0, c1, _ in gathers:
        w.wait()
        if rank == gather_to:
            for r in range(world):
                C_full[rstart[r]:rstart[r] + rows[r], c0:c1] = recv[r][:rows[r]].to(dev)
    if own_ops:
        ops.close()
    return C_local, (C_full if gather_to is not None and rank == gather_to else None)
