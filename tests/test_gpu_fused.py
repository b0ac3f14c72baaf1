"""GPU parity of the FUSED path (the one bench.py and every large call take):
the persistent tcgen05 GEMM with lines 7-10 in its epilogue, whose CRT slice
schedule (s0 = t * SLICES / N per (tile, modulus) unit) and 4 x 4 byte
transposes (zero-padded when N is not a multiple of 4) depend on N.  Also the
boundary's safety properties: concurrent handles, stray environment variables,
the condition (13) certificate, prepared operands and
argument validation.
"""
import threading

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


def assert_bitwise(got, ref, what):
    got = np.ascontiguousarray(got)
    ref = np.ascontiguousarray(ref)
    assert got.shape == ref.shape, (what, got.shape, ref.shape)
    diff = got.view(np.int64) != ref.view(np.int64)
    diff &= ~(np.isnan(got) & np.isnan(ref))
    nbad = int(diff.sum())
    if nbad:
        idx = np.argwhere(diff)[:5]
        raise AssertionError(f"{what}: {nbad} of {diff.size} differ, e.g. "
                             f"{[(tuple(i), got[tuple(i)], ref[tuple(i)]) for i in idx]}")


def _fused_shape_ok(m, n):
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    tiles = ((m + 255) // 256) * ((n + 511) // 512)
    return tiles >= sms // 2                      # below this the unit-parallel path runs


@pytest.mark.parametrize("N", list(range(2, 21)))
def test_fused_every_N(oz2, oracle, monkeypatch, N):
    """80 pair tiles on the fused epilogue (OZ2_UNIT_PARALLEL=0: the default
    schedule picks unit-parallel for a badly filled second wave), ragged n = 3900
    (a partial last tile: 316 of 512 columns) and ragged k = 300 (3 k-blocks, the
    last partial), full matrix bitwise for every N."""
    monkeypatch.setenv("OZ2_UNIT_PARALLEL", "0")
    m, n, k = 2560, 3900, 300
    assert _fused_shape_ok(m, n)
    A = phi_matrix_np(m, k, 1.0, seed=300 + N)
    B = phi_matrix_np(k, n, 1.0, seed=400 + N)
    C = oz2.dgemm(torch.from_numpy(A).to(DEV), torch.from_numpy(B).to(DEV), N).cpu().numpy()
    assert_bitwise(C, oracle.dgemm(A, B, N), f"fused dgemm N={N}")


@pytest.mark.parametrize("N", [2, 3, 5, 9, 13, 14, 17, 20])
def test_fused_forced_small(oz2, oracle, monkeypatch, N):
    """OZ2_UNIT_PARALLEL=0: the fused epilogue on a 2 x 2-tile problem (most
    CTA pairs idle; the last tile finished by the tail loop)."""
    monkeypatch.setenv("OZ2_UNIT_PARALLEL", "0")
    A = phi_matrix_np(300, 333, 1.0, seed=500 + N)
    B = phi_matrix_np(333, 600, 1.0, seed=600 + N)
    C = oz2.dgemm(torch.from_numpy(A).to(DEV), torch.from_numpy(B).to(DEV), N).cpu().numpy()
    assert_bitwise(C, oracle.dgemm(A, B, N), f"fused (forced) N={N}")


def test_c2_full_matrix_n14(oz2, oracle):
    """config c2 (4096^3, N = 14, phi = 1): every entry of C bitwise."""
    n = 4096
    A = phi_matrix_torch(n, n, 1.0, SEED_A, device=DEV)
    B = phi_matrix_torch(n, n, 1.0, SEED_B, device=DEV)
    C = oz2.dgemm(A, B, 14).cpu().numpy()
    assert_bitwise(C, oracle.dgemm(A.cpu().numpy(), B.cpu().numpy(), 14), "c2 full N=14")


@pytest.mark.parametrize("N", list(range(8, 21)))
def test_c2_sampled_256(oz2, oracle, N):
    """config c2 (4096^3), N sweep 8..20: a 256 x 256 sample (random rows and
    columns, the last row and column included) bitwise."""
    n = 4096
    A = phi_matrix_torch(n, n, 1.0, SEED_A, device=DEV)
    B = phi_matrix_torch(n, n, 1.0, SEED_B, device=DEV)
    C = oz2.dgemm(A, B, N)
    rng = np.random.Generator(np.random.PCG64(100 + N))
    rows = np.sort(rng.choice(n - 1, 255, replace=False))
    cols = np.sort(rng.choice(n - 1, 255, replace=False))
    rows = np.append(rows, n - 1)
    cols = np.append(cols, n - 1)
    ri, ci = torch.from_numpy(rows).to(DEV), torch.from_numpy(cols).to(DEV)
    got = C[ri][:, ci].cpu().numpy()
    assert_bitwise(got, oracle.dgemm(A[ri].cpu().numpy(), B[:, ci].cpu().numpy(), N), f"c2 sampled N={N}")


def test_two_handles_concurrent(oz2):
    """Two handles on two streams running 8192^3 products at the same time: the
    persistent GEMMs compete for SMs, so not every CTA of the second grid is
    resident; the progress fence must not wait for a CTA that is not running
    (DESIGN.md section 7).  Both results equal the one-stream results."""
    n, N = 8192, 14
    A = phi_matrix_torch(n, n, 1.0, SEED_A, device=DEV)
    B = phi_matrix_torch(n, n, 1.0, SEED_B, device=DEV)
    A2 = phi_matrix_torch(n, n, 0.5, 11, device=DEV)
    ref1 = oz2.dgemm(A, B, N).cpu().numpy()
    ref2 = oz2.dgemm(A2, B, N).cpu().numpy()
    hs = [oz2.Handle(0), oz2.Handle(0)]
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    outs = [torch.empty((n, n), dtype=torch.float64, device=DEV) for _ in range(2)]
    torch.cuda.synchronize()
    for rep in range(3):
        for h, s, a, c in zip(hs, streams, (A, A2), outs):
            with torch.cuda.stream(s):
                h.prepare("fast", oz2.workspace_bytes(n, n, n, N))
                rc = oz2.lib().oz2_dgemm_ex(h.ptr, n, n, n, oz2._vp(a), n, oz2._vp(B), n, oz2._vp(c), n, N)
                assert rc == 0
        done = threading.Event()

        def wait():
            torch.cuda.synchronize()
            done.set()

        t = threading.Thread(target=wait, daemon=True)
        t.start()
        assert done.wait(120), "concurrent products did not finish (fence deadlock?)"
        assert_bitwise(outs[0].cpu().numpy(), ref1, f"handle 0, rep {rep}")
        assert_bitwise(outs[1].cpu().numpy(), ref2, f"handle 1, rep {rep}")


def test_stray_env_knobs_are_inert(oz2, oracle, monkeypatch):
    """The experiment knobs that would give wrong results (or stall the fence)
    are compiled out of the product library; the tuning knobs are clamped."""
    for k, v in [("OZ2_EPI_NOP", "1"), ("OZ2_EXP_NO_CRT", "1"), ("OZ2_EXP_SKIP_B1", "1"),
                 ("OZ2_SYNC_LAG", "-7"), ("OZ2_SYNC_KB", "-3"), ("OZ2_KB_CHUNK", "-1"), ("OZ2_GROUP_TM", "0")]:
        monkeypatch.setenv(k, v)
    A = phi_matrix_np(2560, 300, 1.0, seed=71)
    B = phi_matrix_np(300, 3900, 1.0, seed=72)
    C = oz2.dgemm(torch.from_numpy(A).to(DEV), torch.from_numpy(B).to(DEV), 14).cpu().numpy()
    assert_bitwise(C, oracle.dgemm(A, B, 14), "dgemm with stray env knobs")


def test_certificate_condition13(oz2, oracle):
    """oz2_certify / oz2_dgemm_scaled / oz2_crt: FAST and
    OS II-accu exponents are certified (beta <= L); exponents raised past the
    bound are refused -- C is all NaN and oz2_status reports OZ2_ERR_NOT_UNIQUE
    -- and nothing is reported when the certificate holds."""
    N = 14
    tab = oz2.tables(N)
    A = phi_matrix_np(300, 400, 1.0, seed=81)
    B = phi_matrix_np(400, 260, 1.0, seed=82)
    A[7] = 0.0                                              # zero rows / columns do not take part
    B[:, 3] = 0.0
    Ad, Bd = torch.from_numpy(A).to(DEV), torch.from_numpy(B).to(DEV)
    e = oz2.scale_rows(Ad, N)
    f = oz2.scale_cols(Bd, N)
    beta = int(oz2.certify(Ad, Bd, e, f, N).item())
    assert beta <= 2 * tab["T"] <= tab["L"], beta           # the Cauchy-Schwarz bound alone gives 2T
    oz2.status()                                            # clears anything earlier
    C = oz2.dgemm_scaled(Ad, Bd, e, f, N).cpu().numpy()
    oz2.status()                                            # no refusal
    assert_bitwise(C, oracle.dgemm(A, B, N), "dgemm_scaled, certified")
    ea, fa = oz2.scale_accu(Ad, Bd, N)                      # accu exponents: certified too
    assert int(oz2.certify(Ad, Bd, ea, fa, N).item()) <= tab["L"]
    # one row scaled 2^40 beyond: no bound certifies it
    e_bad = e.clone()
    e_bad[5] += 40
    assert int(oz2.certify(Ad, Bd, e_bad, f, N).item()) > tab["L"]
    Cb = oz2.dgemm_scaled(Ad, Bd, e_bad, f, N).cpu().numpy()
    assert np.isnan(Cb).all()
    with pytest.raises(oz2.Oz2Error) as ex:
        oz2.status()
    assert ex.value.code == oz2.ERR_NOT_UNIQUE
    oz2.status()                                            # cleared
    # the zero row may carry any exponent
    e_z = e.clone()
    e_z[7] += 1000
    assert int(oz2.certify(Ad, Bd, e_z, f, N).item()) == beta
    # split API: oz2_crt with a certificate
    Ar = oz2.residues_rows(Ad, e_bad, N)
    Br = oz2.residues_cols(Bd, f, N)
    Cp = oz2.modmul(Ar, Br, 400)
    Cc = oz2.crt(Cp, e_bad, f, beta=oz2.certify(Ad, Bd, e_bad, f, N)).cpu().numpy()
    assert np.isnan(Cc).all()
    with pytest.raises(oz2.Oz2Error):
        oz2.status()
    Cc = oz2.crt(Cp, e_bad, f).cpu().numpy()                # no certificate: no check
    assert not np.isnan(Cc).any()
    oz2.status()


def test_prepared_objects_independent(oz2, oracle):
    """Two prepared B operands on one device (and a prepared A) do not share
    memory: each product uses its own operand (one prepared B per
    handle was overwritten by the next oz2_prepare_b)."""
    N = 14
    A = phi_matrix_np(600, 500, 1.0, seed=91)
    B1 = phi_matrix_np(500, 700, 1.0, seed=92)
    B2 = phi_matrix_np(500, 700, 1.0, seed=93)
    Ad = torch.from_numpy(A).to(DEV)
    p1 = oz2.PreparedB(torch.from_numpy(B1).to(DEV), N)
    p2 = oz2.PreparedB(torch.from_numpy(B2).to(DEV), N)
    pa = oz2.PreparedA(Ad, N)
    r1 = oracle.dgemm(A, B1, N)
    r2 = oracle.dgemm(A, B2, N)
    assert_bitwise(p1.dgemm(Ad).cpu().numpy(), r1, "prepared B1")
    assert_bitwise(p2.dgemm(Ad).cpu().numpy(), r2, "prepared B2")
    assert_bitwise(oz2.dgemm_prep2(pa, p1).cpu().numpy(), r1, "prep2 A x B1")
    p2.release()
    assert_bitwise(p1.dgemm(Ad).cpu().numpy(), r1, "prepared B1 after releasing B2")
    with pytest.raises(ValueError):
        p2.dgemm(Ad)
    # column panels of B against one prepared A: C's column blocks
    C = torch.empty((600, 700), dtype=torch.float64, device=DEV)
    Bd = torch.from_numpy(B1).to(DEV)
    for c0, c1 in ((0, 256), (256, 512), (512, 700)):
        pb = oz2.PreparedB(Bd[:, c0:c1], N)
        oz2.dgemm_prep2(pa, pb, out=C[:, c0:c1])
    assert_bitwise(C.cpu().numpy(), r1, "prep2 over column panels")


def test_out_and_device_validation(oz2):
    A = torch.ones((8, 8), dtype=torch.float64, device=DEV)
    with pytest.raises(ValueError):
        oz2.dgemm(A, A, 14, out=torch.empty((8, 8), dtype=torch.float32, device=DEV))
    with pytest.raises(ValueError):
        oz2.dgemm(A, A, 14, out=torch.empty((4, 8), dtype=torch.float64, device=DEV))
    with pytest.raises(ValueError):
        oz2.dgemm(A, A, 14, out=torch.empty((8, 8), dtype=torch.float64))
    with pytest.raises(ValueError):
        oz2.dgemm_scaled(A, A, torch.zeros(7, dtype=torch.int32), torch.zeros(8, dtype=torch.int32), 14)


@pytest.mark.parametrize("shape", [(2, 1), (1, 1)])
@pytest.mark.parametrize("N", [9, 14, 17])
def test_alternative_tile_shapes(oz2, oracle, monkeypatch, shape, N):
    """The env-selectable GEMM shapes other than the default 256 x 512 pair tile:
    OZ2_CG=2 OZ2_NH=1 (256 x 256 pair tile, TMEM double buffer) and OZ2_CG=1
    (128 x 256 single-CTA tile), fused epilogue on several tiles with ragged
    edges, bitwise against the oracle."""
    cg, nh = shape
    monkeypatch.setenv("OZ2_CG", str(cg))
    monkeypatch.setenv("OZ2_NH", str(nh))
    monkeypatch.setenv("OZ2_UNIT_PARALLEL", "0")
    A = phi_matrix_np(700, 500, 1.0, seed=700 + N)
    B = phi_matrix_np(500, 1300, 1.0, seed=800 + N)
    C = oz2.dgemm(torch.from_numpy(A).to(DEV), torch.from_numpy(B).to(DEV), N).cpu().numpy()
    assert_bitwise(C, oracle.dgemm(A, B, N), f"shape cg={cg} nh={nh} N={N}")


@pytest.mark.parametrize("N", [8, 14, 20])
def test_unit_parallel_midsize_default(oz2, oracle, N):
    """The default schedule on 98 pair tiles (3584 x 3584 output: a 0.66-full
    second wave) takes the unit-parallel path (units spread, lines 8-10 in the
    CRT kernel); full matrix bitwise with k = 257."""
    m = n = 3584
    k = 257
    assert oz2.lib().oz2_version() > 0
    A = phi_matrix_np(m, k, 1.0, seed=900 + N)
    B = phi_matrix_np(k, n, 1.0, seed=950 + N)
    C = oz2.dgemm(torch.from_numpy(A).to(DEV), torch.from_numpy(B).to(DEV), N).cpu().numpy()
    assert_bitwise(C, oracle.dgemm(A, B, N), f"unit-parallel (default) N={N}")
