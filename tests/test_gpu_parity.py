"""GPU parity: every stage of the CUDA path (through the C ABI) against the
oracle, element by element, bit for bit.

Sizes span several 128 x 256 output tiles and 128-byte K stages with ragged
tails; edge cases cover k = 1, single rows/columns, zero and non-finite rows,
the int32 exactness boundary k = 2^17 - 1, every N in 2..20 and both scaling
modes.  Large configurations are checked on sampled rows/columns: e_i depends
only on row i of A and f_j only on column j of B, so the oracle's result on a
row/column subset is exactly the corresponding block of C.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2504_08009_b200.inputs import phi_matrix_np, phi_matrix_torch, SEED_A, SEED_B

DEV = "cuda:0"


@pytest.fixture(scope="module")
def oz2():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2504_08009_b200 import build, oz2 as o
    build.build()
    return o


def _bits(x):
    x = np.ascontiguousarray(x, dtype=np.float64)
    return x.view(np.int64)


def assert_bitwise(got, ref, what):
    got = np.asarray(got)
    ref = np.asarray(ref)
    assert got.shape == ref.shape, (what, got.shape, ref.shape)
    if got.dtype == np.float64:
        diff = _bits(got) != _bits(ref)
        # NaN payloads may differ; NaN positions must not
        diff &= ~(np.isnan(got) & np.isnan(ref))
    else:
        diff = got != ref
    nbad = int(diff.sum())
    if nbad:
        idx = np.argwhere(diff)[:5]
        detail = [(tuple(i), got[tuple(i)], ref[tuple(i)]) for i in idx]
        raise AssertionError(f"{what}: {nbad} of {diff.size} differ, e.g. {detail}")


def _stages(oz2, oracle, A, B, N, mode):
    m, k = A.shape
    n = B.shape[1]
    mo = oracle.MODE_FAST if mode == "fast" else oracle.MODE_EQ17
    dA = torch.from_numpy(A).to(DEV)
    dB = torch.from_numpy(B).to(DEV)
    e = oz2.scale_rows(dA, N, mode)
    f = oz2.scale_cols(dB, N, mode)
    e_ref = oracle.scale_rows(A, N, mo)
    f_ref = oracle.scale_cols(B, N, mo)
    assert_bitwise(e.cpu().numpy(), e_ref, "e (Alg.1 line 1, rows)")
    assert_bitwise(f.cpu().numpy(), f_ref, "f (Alg.1 line 1, cols)")
    Ap = oz2.trunc_rows(dA, e)
    BpT = oz2.trunc_cols(dB, f)
    Ap_ref = oracle.trunc_rows(A, e_ref)
    BpT_ref = oracle.trunc_cols(B, f_ref)
    assert_bitwise(Ap.cpu().numpy(), Ap_ref, "A' (line 2)")
    assert_bitwise(BpT.cpu().numpy(), BpT_ref, "B' (line 3)")
    Ar = oz2.residues_rows(dA, e, N)
    Br = oz2.residues_cols(dB, f, N)
    Ar_ref = oracle.residues(Ap_ref, N)
    Br_ref = oracle.residues(BpT_ref, N)
    assert_bitwise(Ar[:, :, :k].cpu().numpy(), Ar_ref, "A residues (line 4)")
    assert_bitwise(Br[:, :, :k].cpu().numpy(), Br_ref, "B residues (line 5)")
    Cp = oz2.modmul(Ar, Br, k)
    Cp_ref = oracle.modmul(Ar_ref, Br_ref)
    assert_bitwise(Cp.cpu().numpy(), Cp_ref, "C'_t (line 6, tcgen05)")
    C = oz2.crt(Cp, e, f)
    C_ref = oracle.crt(Cp_ref, e_ref, f_ref)
    assert_bitwise(C.cpu().numpy(), C_ref, "C (lines 7-10)")
    C2 = oz2.dgemm(dA, dB, N, mode)
    assert_bitwise(C2.cpu().numpy(), oracle.dgemm(A, B, N, mo), "C (oz2_dgemm end to end)")


@pytest.mark.parametrize("m,n,k,N,phi,mode", [
    (64, 64, 64, 14, 0.5, "fast"),          # config c1
    (130, 300, 333, 14, 1.0, "fast"),       # 2x2 tiles, ragged M, N, K
    (257, 513, 700, 8, 2.0, "fast"),        # 3x3 tiles, 3 K-chunks of the FAST rule
    (128, 256, 128, 16, 0.5, "fast"),       # exact tile
    (100, 200, 256, 17, 1.0, "fast"),       # 96-bit residue path
    (77, 90, 129, 20, 4.0, "fast"),
    (33, 47, 300, 2, 0.5, "fast"),
    (70, 80, 200, 5, 0.5, "fast"),          # P = 1 CRT
    (70, 80, 200, 11, 1.0, "fast"),
    (64, 64, 64, 14, 0.5, "eq17"),
    (150, 260, 400, 20, 1.0, "eq17"),
])
def test_stage_parity(oz2, oracle, m, n, k, N, phi, mode):
    A = phi_matrix_np(m, k, phi, seed=1000 + m)
    B = phi_matrix_np(k, n, phi, seed=2000 + n)
    _stages(oz2, oracle, A, B, N, mode)


@pytest.mark.parametrize("N", list(range(2, 21)))
def test_dgemm_every_N(oz2, oracle, N):
    m, n, k = 140, 270, 260
    A = phi_matrix_np(m, k, 1.0, seed=7 + N)
    B = phi_matrix_np(k, n, 1.0, seed=8 + N)
    C = oz2.dgemm(torch.from_numpy(A).to(DEV), torch.from_numpy(B).to(DEV), N)
    assert_bitwise(C.cpu().numpy(), oracle.dgemm(A, B, N), f"dgemm N={N}")


def test_edge_shapes_and_values(oz2, oracle):
    cases = [(1, 1, 1), (1, 300, 5), (300, 1, 17), (5, 7, 1), (129, 257, 31), (3, 3, 16)]
    for (m, n, k) in cases:
        A = phi_matrix_np(m, k, 1.0, seed=m * 7 + k)
        B = phi_matrix_np(k, n, 1.0, seed=n * 11 + k)
        _stages(oz2, oracle, A, B, 14, "fast")
    m, n, k = 90, 100, 300
    A = phi_matrix_np(m, k, 1.0, seed=5)
    B = phi_matrix_np(k, n, 1.0, seed=6)
    A[3] = 0.0                              # zero row
    B[:, 7] = 0.0                           # zero column
    A[5, 10] = np.nan                       # non-finite row
    B[20, 9] = -np.inf                      # non-finite column
    A[8] *= 2.0 ** -1070                    # subnormal row
    B[:, 11] *= 2.0 ** 900                  # huge column
    A[12, :] = 2.0 ** 60                    # constant row
    _stages(oz2, oracle, A, B, 14, "fast")
    _stages(oz2, oracle, A, B, 18, "fast")


def test_extreme_range_within_chunk(oz2, oracle):
    # FAST statistics (reading R4) where |x| 2^(15 - E_c) underflows: a chunk that
    # holds 2^1000 next to subnormals must still count u = 1 for every nonzero
    # element; chunks whose maximum is subnormal take the 64-bit ilogb path; a
    # ragged last chunk (k = 600 = 2 * 256 + 88)
    m, n, k = 40, 48, 600
    A = phi_matrix_np(m, k, 1.0, seed=31)
    B = phi_matrix_np(k, n, 1.0, seed=32)
    A[0, 0] = 2.0 ** 1000
    A[0, 1:200:3] = 2.0 ** -1070                 # underflows against 2^(15-1000)
    A[0, 5] = -5e-324
    A[1, 260] = 2.0 ** 1000
    A[1, 301:512] *= 2.0 ** -1060                # mixed normal / subnormal in one chunk
    A[2, :256] = 2.0 ** -1050                    # a chunk whose maximum is subnormal
    A[2, 256:] *= 2.0 ** -1100
    A[3, 520:600] = 3e-320                       # subnormal tail chunk, zeros before
    A[3, :520] = 0.0
    B[0, 0] = -2.0 ** 10
    B[1:250:7, 0] = 2.0 ** -1074
    B[256:512, 1] *= 2.0 ** -1060
    B[300, 1] = 2.0 ** 990
    B[:, 2] = 1e-315                             # subnormal column
    B[512:, 3] = 2.0 ** -1040
    B[:512, 3] = 0.0
    for N in (14, 20):
        _stages(oz2, oracle, A, B, N, "fast")


def test_int32_boundary_k(oz2, oracle):
    # k = 2^17 - 1 with all residues -128 gives 2^31 - 16384
    k = 2**17 - 1
    m, n, N = 8, 8, 3
    ldr = (k + 15) // 16 * 16
    Ar = torch.full((N, m, ldr), -128, dtype=torch.int8, device=DEV)
    Br = torch.full((N, n, ldr), -128, dtype=torch.int8, device=DEV)
    Cp = oz2.modmul(Ar, Br, k).cpu().numpy()
    assert (Cp == 2**31 - 16384).all()
    rng = np.random.Generator(np.random.PCG64(3))
    Ar_np = rng.integers(-128, 128, size=(N, m, k)).astype(np.int8)
    Br_np = rng.integers(-128, 128, size=(N, n, k)).astype(np.int8)
    Ar = torch.zeros((N, m, ldr), dtype=torch.int8, device=DEV)
    Br = torch.zeros((N, n, ldr), dtype=torch.int8, device=DEV)
    Ar[:, :, :k] = torch.from_numpy(Ar_np).to(DEV)
    Br[:, :, :k] = torch.from_numpy(Br_np).to(DEV)
    assert_bitwise(oz2.modmul(Ar, Br, k).cpu().numpy(), oracle.modmul(Ar_np, Br_np), "modmul k=2^17-1")


def test_errors_fail_loudly(oz2):
    A = torch.ones((4, 4), dtype=torch.float64, device=DEV)
    with pytest.raises(oz2.Oz2Error):
        oz2.dgemm(A, A, 21)
    with pytest.raises(oz2.Oz2Error):
        oz2.dgemm(A, A, 1)
    big = torch.ones((1, 2**20), dtype=torch.float64, device=DEV)
    with pytest.raises(oz2.Oz2Error):
        oz2.dgemm(big, big.T.contiguous(), 14)
    with pytest.raises(oz2.Oz2Error):        # EQ17 budget < 1 (N = 2, k = 20000)
        w = torch.ones((2, 20000), dtype=torch.float64, device=DEV)
        oz2.dgemm(w, w.T.contiguous(), 2, mode="eq17")
    Z = oz2.dgemm(torch.ones((3, 0), dtype=torch.float64, device=DEV),
                  torch.ones((0, 5), dtype=torch.float64, device=DEV), 14)
    assert (Z.cpu().numpy() == 0).all()


def test_host_entry_point(oz2, oracle):
    A = phi_matrix_np(100, 200, 0.5, seed=1)
    B = phi_matrix_np(200, 150, 0.5, seed=2)
    C = oz2.dgemm_host(A, B, 14)
    assert_bitwise(C, oracle.dgemm(A, B, 14), "oz2_dgemm_host")


def test_host_entry_point_pipelined(oz2, oracle):
    """m = 9000: two row blocks (4608 + 4392 rows) on the copy/compute pipeline."""
    A = phi_matrix_np(9000, 700, 1.0, seed=21)
    B = phi_matrix_np(700, 600, 1.0, seed=22)
    Ah = torch.from_numpy(A).pin_memory().numpy()
    Bh = torch.from_numpy(B).pin_memory().numpy()
    Ch = torch.empty((9000, 600), dtype=torch.float64).pin_memory().numpy()
    oz2.dgemm_host(Ah, Bh, 14, out=Ch)
    Cd = oz2.dgemm(torch.from_numpy(A).to(DEV), torch.from_numpy(B).to(DEV), 14).cpu().numpy()
    assert_bitwise(Ch, Cd, "pipelined host path vs device path")
    rows = np.array([0, 4607, 4608, 8999])                    # both sides of the block boundary
    assert_bitwise(Ch[rows], oracle.dgemm(A[rows], B, 14), "pipelined host path vs oracle")


def test_host_entry_point_2d(oz2, oracle):
    """m, n >= 8192: the 2-D host pipeline (panels of B x blocks of A, ragged
    last panel 520 columns and last block 2088 rows), bitwise vs the device path."""
    m, n, k = 9000, 8200, 300
    A = phi_matrix_np(m, k, 1.0, seed=23)
    B = phi_matrix_np(k, n, 1.0, seed=24)
    Ah = torch.from_numpy(A).pin_memory().numpy()
    Bh = torch.from_numpy(B).pin_memory().numpy()
    Ch = torch.empty((m, n), dtype=torch.float64).pin_memory().numpy()
    oz2.dgemm_host(Ah, Bh, 14, out=Ch)
    Cd = oz2.dgemm(torch.from_numpy(A).to(DEV), torch.from_numpy(B).to(DEV), 14).cpu().numpy()
    assert_bitwise(Ch, Cd, "2-D host pipeline vs device path")
    rows = np.array([0, 2303, 2304, 8999])
    assert_bitwise(Ch[rows], oracle.dgemm(A[rows], B, 14), "2-D host pipeline vs oracle")


def test_k_blocking_forced(oz2, oracle, monkeypatch):
    """K blocking exercised at small k: OZ2_KB_CHUNK=2 splits the
    8 k-blocks of k = 1000 into 4 int32 accumulations whose residues are added."""
    monkeypatch.setenv("OZ2_KB_CHUNK", "2")
    A = phi_matrix_np(300, 1000, 1.0, seed=41)
    B = phi_matrix_np(1000, 530, 1.0, seed=42)
    for N in (3, 14, 20):
        C = oz2.dgemm(torch.from_numpy(A).to(DEV), torch.from_numpy(B).to(DEV), N).cpu().numpy()
        assert_bitwise(C, oracle.dgemm(A, B, N), f"k-blocked N={N}")


def test_k_beyond_int32_range(oz2, oracle):
    """k = 2^17 + 3000 > 2^17: two K blocks of <= 1023 k-blocks (ragged tail)."""
    k = 2**17 + 3000
    A = phi_matrix_np(96, k, 0.5, seed=43)
    B = phi_matrix_np(k, 200, 0.5, seed=44)
    C = oz2.dgemm(torch.from_numpy(A).to(DEV), torch.from_numpy(B).to(DEV), 14).cpu().numpy()
    assert_bitwise(C, oracle.dgemm(A, B, 14), "k = 2^17 + 3000")


def test_strided_operands(oz2, oracle):
    A = phi_matrix_np(70, 300, 1.0, seed=11)
    B = phi_matrix_np(300, 90, 1.0, seed=12)
    Abig = torch.zeros((70, 333), dtype=torch.float64, device=DEV)
    Bbig = torch.zeros((300, 101), dtype=torch.float64, device=DEV)
    Abig[:, :300] = torch.from_numpy(A).to(DEV)
    Bbig[:, :90] = torch.from_numpy(B).to(DEV)
    C = oz2.dgemm(Abig[:, :300], Bbig[:, :90], 14)           # lda = 333, ldb = 101 (odd: unaligned rows)
    assert_bitwise(C.cpu().numpy(), oracle.dgemm(A, B, 14), "strided dgemm")


@pytest.mark.parametrize("n,N", [(4096, 14), (4096, 8), (4096, 20)])
def test_c2_sampled(oz2, oracle, n, N):
    """config c2 (4096^3): sampled 48 x 48 block + 2 full rows, bitwise."""
    A = phi_matrix_torch(n, n, 1.0, SEED_A, device=DEV)
    B = phi_matrix_torch(n, n, 1.0, SEED_B, device=DEV)
    C = oz2.dgemm(A, B, N).cpu().numpy()
    rng = np.random.Generator(np.random.PCG64(3))
    rows = np.sort(rng.choice(n, 48, replace=False))
    cols = np.sort(rng.choice(n, 48, replace=False))
    An = A[torch.from_numpy(rows).to(DEV)].cpu().numpy()
    Bn = B[:, torch.from_numpy(cols).to(DEV)].cpu().numpy()
    assert_bitwise(C[np.ix_(rows, cols)], oracle.dgemm(An, Bn, N), f"c2 sampled N={N}")
    full_rows = rows[:2]
    Ar = A[torch.from_numpy(full_rows).to(DEV)].cpu().numpy()
    assert_bitwise(C[full_rows], oracle.dgemm(Ar, B.cpu().numpy(), N), f"c2 full rows N={N}")


@pytest.mark.parametrize("ta,tb", [(False, False), (True, False), (False, True), (True, True)])
def test_gemm_surface_transposes_alpha_beta(oz2, oracle, ta, tb):
    """oz2_dgemm_op (reading R19): op(A), op(B) and C := alpha AB + beta C, bitwise."""
    m, n, k = 300, 270, 520
    Aop = phi_matrix_np(m, k, 1.0, seed=61)
    Bop = phi_matrix_np(k, n, 1.0, seed=62)
    A = Aop.T.copy() if ta else Aop
    B = Bop.T.copy() if tb else Bop
    Cold = phi_matrix_np(m, n, 1.0, seed=63)
    for alpha, beta in [(1.0, 0.0), (-1.5, 0.0), (0.75, -2.0)]:
        Cd = torch.from_numpy(Cold.copy()).to(DEV)
        oz2.gemm(torch.from_numpy(A).to(DEV), torch.from_numpy(B).to(DEV), 14, alpha, beta, Cd,
                 transA=ta, transB=tb)
        ref = oracle.gemm(A, B, 14, alpha, beta, Cold, transA=ta, transB=tb)
        assert_bitwise(Cd.cpu().numpy(), ref, f"gemm ta={ta} tb={tb} alpha={alpha} beta={beta}")


def test_gemm_surface_degenerate(oz2, oracle):
    A = torch.from_numpy(phi_matrix_np(40, 50, 1.0, seed=64)).to(DEV)
    B = torch.from_numpy(phi_matrix_np(50, 30, 1.0, seed=65)).to(DEV)
    C0 = phi_matrix_np(40, 30, 1.0, seed=66)
    # beta = 0: C is not read (NaN must not propagate)
    Cn = torch.full((40, 30), float("nan"), dtype=torch.float64, device=DEV)
    oz2.gemm(A, B, 14, 2.0, 0.0, Cn)
    assert_bitwise(Cn.cpu().numpy(), 2.0 * oracle.dgemm(A.cpu().numpy(), B.cpu().numpy(), 14), "beta=0")
    # alpha = 0: C := beta C, no product
    Cd = torch.from_numpy(C0.copy()).to(DEV)
    oz2.gemm(A, B, 14, 0.0, -3.0, Cd)
    assert_bitwise(Cd.cpu().numpy(), -3.0 * C0, "alpha=0")
    # k = 0
    Cd = torch.from_numpy(C0.copy()).to(DEV)
    oz2.gemm(A[:, :0], B[:0, :], 14, 1.0, 0.5, Cd)
    assert_bitwise(Cd.cpu().numpy(), 0.5 * C0, "k=0")


def test_gemm_strided_batched(oz2, oracle):
    rng_seeds = [(71, 72), (73, 74), (75, 76)]
    A = np.stack([phi_matrix_np(90, 130, 1.0, seed=a) for a, _ in rng_seeds])
    B = np.stack([phi_matrix_np(110, 130, 1.0, seed=b) for _, b in rng_seeds])    # stored n x k (transB)
    C = oz2.gemm_strided_batched(torch.from_numpy(A).to(DEV), torch.from_numpy(B).to(DEV), 13,
                                 transB=True).cpu().numpy()
    for i in range(3):
        assert_bitwise(C[i], oracle.gemm(A[i], B[i], 13, transB=True), f"batch item {i}")


@pytest.mark.parametrize("N", [2, 8, 14, 16, 17, 20])
def test_accu_exponents_and_dgemm(oz2, oracle, N):
    """OS II-accu (reading R18): the line-1 exponents (bound GEMM on the tensor
    cores, row/column maxima) and the whole product, bitwise vs the oracle."""
    A = phi_matrix_np(301, 257, 4.0, seed=91)
    B = phi_matrix_np(257, 515, 4.0, seed=92)
    A[5, :] = 0.0
    A[7, 3] = np.inf
    B[:, 9] = 0.0
    B[:, 11] *= 1e-310                                   # a subnormal column
    e_ref, f_ref, _, _ = oracle.scale_accu(A, B, N)
    e, f = oz2.scale_accu(torch.from_numpy(A).to(DEV), torch.from_numpy(B).to(DEV), N)
    assert np.array_equal(e.cpu().numpy(), e_ref), "accu e"
    assert np.array_equal(f.cpu().numpy(), f_ref), "accu f"
    C = oz2.dgemm(torch.from_numpy(A).to(DEV), torch.from_numpy(B).to(DEV), N, mode="accu").cpu().numpy()
    assert_bitwise(C, oracle.dgemm(A, B, N, oracle.MODE_ACCU), f"accu dgemm N={N}")


def test_accu_transposed_operands(oz2, oracle):
    Aop = phi_matrix_np(200, 300, 2.0, seed=93)
    Bop = phi_matrix_np(300, 260, 2.0, seed=94)
    C = oz2.gemm(torch.from_numpy(Aop.T.copy()).to(DEV), torch.from_numpy(Bop.T.copy()).to(DEV), 15,
                 transA=True, transB=True, mode="accu").cpu().numpy()
    assert_bitwise(C, oracle.dgemm(Aop, Bop, 15, oracle.MODE_ACCU), "accu transposed")
    Ch = oz2.dgemm_host(Aop, Bop, 15, mode="accu")
    assert_bitwise(Ch, C, "accu host path")


def test_dgemm_scaled_and_sharded_accu(oz2, oracle):
    """oz2_dgemm_scaled with given exponents, and the row-sharded accu recipe of
    dist.dgemm_rowblock (partial f, element-wise MIN) on one GPU, bitwise."""
    A = phi_matrix_np(400, 300, 4.0, seed=95)
    B = phi_matrix_np(300, 270, 4.0, seed=96)
    Ad, Bd = torch.from_numpy(A).to(DEV), torch.from_numpy(B).to(DEV)
    ref = oracle.dgemm(A, B, 16, oracle.MODE_ACCU)
    e, f, _, _ = oracle.scale_accu(A, B, 16)
    C = oz2.dgemm_scaled(Ad, Bd, torch.from_numpy(e), torch.from_numpy(f), 16).cpu().numpy()
    assert_bitwise(C, ref, "dgemm_scaled with oracle accu exponents")
    parts = [(0, 130), (130, 400)]
    ef = [oz2.scale_accu(Ad[a:b], Bd, 16) for a, b in parts]
    fmin = torch.minimum(ef[0][1], ef[1][1])
    Cs = torch.cat([oz2.dgemm_scaled(Ad[a:b], Bd, ef[i][0], fmin, 16) for i, (a, b) in enumerate(parts)])
    assert_bitwise(Cs.cpu().numpy(), ref, "row-sharded accu (MIN of partial f)")


def test_prepared_b_and_sm_limit(oz2, oracle):
    """B-stationary products (oz2_prepare_b / oz2_dgemm_prepared) and a reduced
    GEMM SM budget give the same bits as oz2_dgemm."""
    B = phi_matrix_np(700, 650, 1.0, seed=97)
    Bd = torch.from_numpy(B).to(DEV)
    pb = oz2.PreparedB(Bd, 14)
    for seed, m in ((98, 300), (99, 1030)):
        A = phi_matrix_np(m, 700, 1.0, seed=seed)
        Ad = torch.from_numpy(A).to(DEV)
        ref = oz2.dgemm(Ad, Bd, 14).cpu().numpy()
        assert_bitwise(pb.dgemm(Ad).cpu().numpy(), ref, f"prepared B m={m}")
        assert_bitwise(ref[:5], oracle.dgemm(A[:5], B, 14), "dgemm rows vs oracle")
    pb.release()
    oz2.set_sm_limit(100)
    try:
        A = phi_matrix_np(900, 700, 1.0, seed=100)
        Ad = torch.from_numpy(A).to(DEV)
        C = oz2.dgemm(Ad, Bd, 14).cpu().numpy()
    finally:
        oz2.set_sm_limit(0)
    assert_bitwise(C, oz2.dgemm(Ad, Bd, 14).cpu().numpy(), "sm limit 100")


def test_cuda_graph_capture(oz2, oracle):
    """oz2_dgemm is capturable (no host synchronisation, no allocation once the
    workspace exists): a CUDA graph of the whole Algorithm 1 replays bit-identically
    -- the launch-bound small sizes (config c1) are meant to run this way."""
    A = torch.from_numpy(phi_matrix_np(64, 64, 0.5, seed=131)).to(DEV)
    B = torch.from_numpy(phi_matrix_np(64, 64, 0.5, seed=132)).to(DEV)
    C = torch.empty((64, 64), dtype=torch.float64, device=DEV)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        oz2.dgemm(A, B, 14, out=C)                        # warm-up: workspace, TMA encode, attributes
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            oz2.dgemm(A, B, 14, out=C)
    torch.cuda.current_stream().wait_stream(s)
    C.zero_()
    g.replay()
    torch.cuda.synchronize()
    assert_bitwise(C.cpu().numpy(), oracle.dgemm(A.cpu().numpy(), B.cpu().numpy(), 14), "graph replay")
