"""Thin ctypes binding of liboz2.so (include/oz2.h) for torch tensors.

Argument marshalling only: every stage of the path runs in the library's
sm_100a kernels.  torch provides device memory (outputs and the workspace, via
its caching allocator) and the stream (torch.cuda.current_stream()).  If the
library is missing, every call raises -- there is no CPU fallback.
"""
from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# OZ2_LIB: an alternative in-tree build of the same library (A/B experiments only)
LIB_PATH = os.environ.get("OZ2_LIB") or os.path.join(_HERE, "liboz2.so")

OK = 0
MODE_FAST = 0
MODE_EQ17 = 1
MODE_ACCU = 2
EXP_NONFINITE = -(2**31)
ERR_NOT_UNIQUE = 8
MAX_K = 2**20          # oz2_modmul (raw int32 products): 2**17

# every symbol include/oz2.h declares (checked by tests/test_abi.py)
SYMBOLS = [
    "oz2_create", "oz2_destroy", "oz2_set_stream", "oz2_set_mode", "oz2_set_workspace",
    "oz2_workspace_bytes", "oz2_dgemm", "oz2_dgemm_ex", "oz2_dgemm_host", "oz2_scale_rows",
    "oz2_scale_cols", "oz2_trunc_rows", "oz2_trunc_cols", "oz2_residues_rows", "oz2_residues_cols",
    "oz2_modmul", "oz2_crt", "oz2_tables", "oz2_eq17_k", "oz2_strerror", "oz2_version",
    "oz2_set_profiling", "oz2_stage_times", "oz2_dgemm_op", "oz2_dgemm_strided_batched",
    "oz2_scale_accu", "oz2_dgemm_scaled", "oz2_prepare_a", "oz2_prepare_b", "oz2_dgemm_prepared",
    "oz2_dgemm_prep2", "oz2_reprepare", "oz2_release", "oz2_certify", "oz2_set_certify", "oz2_status",
    "oz2_set_sm_limit", "oz2_kslice_stats_rows", "oz2_kslice_stats_cols", "oz2_exponents_from_stats",
    "oz2_modmul_residues", "oz2_crt_sum", "oz2_dsyrk", "oz2_dtrmm", "oz2_kernel_launches",
    "oz2_dgemm_fp64mod", "oz2_dgemm_fp64mod_dw", "oz2_fp64mod_workspace_bytes", "oz2_fp64mod_tables",
]
OP_N, OP_T = 0, 1
# stage 0 times A's conversion (and B's too with OZ2_CONV_OVERLAP=1; the two column
# stages then read 0); the host pipeline (oz2_dgemm_host) times rows of A inside "gemm"
STAGES = ["rows_A", "colstats_B", "colres_B", "gemm", "crt"]


class Oz2Error(RuntimeError):
    def __init__(self, code: int, what: str = ""):
        msg = lib().oz2_strerror(code).decode() if _lib is not None else str(code)
        super().__init__(f"{what}: liboz2 error {code} ({msg})")
        self.code = code


_lib = None
_lock = threading.Lock()


def lib() -> ctypes.CDLL:
    """Load liboz2.so (raises OSError if it has not been built)."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not os.path.exists(LIB_PATH):
                    raise OSError(f"{LIB_PATH} not found: build it with "
                                  "`python -m paper_2504_08009_b200.build` (no CPU fallback)")
                L = ctypes.CDLL(LIB_PATH)
                P, i64, i32, sz = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_size_t
                L.oz2_create.argtypes = [ctypes.POINTER(P), i32]
                L.oz2_destroy.argtypes = [P]
                L.oz2_set_stream.argtypes = [P, P]
                L.oz2_set_mode.argtypes = [P, i32]
                L.oz2_set_workspace.argtypes = [P, P, sz]
                L.oz2_workspace_bytes.argtypes = [i64, i64, i64, i32]
                L.oz2_workspace_bytes.restype = sz
                L.oz2_dgemm.argtypes = [i64, i64, i64, P, i64, P, i64, P, i64, i32]
                L.oz2_dgemm_ex.argtypes = [P, i64, i64, i64, P, i64, P, i64, P, i64, i32]
                L.oz2_dgemm_host.argtypes = [P, i64, i64, i64, P, i64, P, i64, P, i64, i32]
                d = ctypes.c_double
                L.oz2_dgemm_op.argtypes = [P, i32, i32, i64, i64, i64, d, P, i64, P, i64, d, P, i64, i32]
                L.oz2_dsyrk.argtypes = [P, i32, i32, i64, i64, d, P, i64, d, P, i64, i32]
                L.oz2_dtrmm.argtypes = [P, i32, i32, i32, i32, i64, i64, d, P, i64, P, i64, i32]
                L.oz2_dgemm_strided_batched.argtypes = [P, i32, i32, i64, i64, i64, d, P, i64, i64, P, i64, i64,
                                                        d, P, i64, i64, i64, i32]
                L.oz2_scale_rows.argtypes = [P, i64, i64, P, i64, i32, P]
                L.oz2_scale_cols.argtypes = [P, i64, i64, P, i64, i32, P]
                L.oz2_scale_accu.argtypes = [P, i64, i64, i64, P, i64, P, i64, i32, P, P]
                L.oz2_prepare_a.argtypes = [P, i64, i64, P, i64, i32, ctypes.POINTER(P)]
                L.oz2_prepare_b.argtypes = [P, i64, i64, P, i64, i32, ctypes.POINTER(P)]
                L.oz2_dgemm_prepared.argtypes = [P, P, i64, P, i64, P, i64]
                L.oz2_dgemm_prep2.argtypes = [P, P, P, P, i64]
                L.oz2_release.argtypes = [P]
                L.oz2_reprepare.argtypes = [P, P, P, i64]
                L.oz2_certify.argtypes = [P, i64, i64, i64, P, i64, P, i64, P, P, i32, P]
                L.oz2_set_certify.argtypes = [P, i32]
                L.oz2_status.argtypes = [P]
                L.oz2_set_sm_limit.argtypes = [P, i32]
                L.oz2_kslice_stats_rows.argtypes = [P, i64, i64, P, i64, P, P, P]
                L.oz2_kslice_stats_cols.argtypes = [P, i64, i64, P, i64, P, P, P]
                L.oz2_exponents_from_stats.argtypes = [P, i64, P, P, i64, i32, P]
                L.oz2_modmul_residues.argtypes = [P, i64, i64, i64, P, P, i64, i32, P, i64]
                L.oz2_crt_sum.argtypes = [P, i32, i64, i64, P, i64, P, P, i32, P, i64, P]
                L.oz2_dgemm_scaled.argtypes = [P, i64, i64, i64, P, i64, P, i64, P, P, P, i64, i32]
                L.oz2_trunc_rows.argtypes = [P, i64, i64, P, i64, P, P]
                L.oz2_trunc_cols.argtypes = [P, i64, i64, P, i64, P, P]
                L.oz2_residues_rows.argtypes = [P, i64, i64, P, i64, P, i32, P, i64]
                L.oz2_residues_cols.argtypes = [P, i64, i64, P, i64, P, i32, P, i64]
                L.oz2_modmul.argtypes = [P, i64, i64, i64, P, P, i64, i32, P]
                L.oz2_crt.argtypes = [P, i64, i64, P, P, P, i32, P, i64, P]
                L.oz2_tables.argtypes = [i32, P, P, P, P, P, P, P]
                L.oz2_eq17_k.argtypes = [i32, i64]
                L.oz2_strerror.argtypes = [i32]
                L.oz2_strerror.restype = ctypes.c_char_p
                L.oz2_version.argtypes = []
                L.oz2_set_profiling.argtypes = [P, i32]
                L.oz2_stage_times.argtypes = [P, P, P]
                L.oz2_dgemm_fp64mod.argtypes = [P, i64, i64, i64, P, i64, P, i64, i32, i32, P, i64, i64]
                L.oz2_dgemm_fp64mod_dw.argtypes = [P, i64, i64, i64, P, P, i64, P, P, i64, i32, i32, P, i64, i64]
                L.oz2_fp64mod_workspace_bytes.argtypes = [i64, i64, i64, i32]
                L.oz2_fp64mod_workspace_bytes.restype = sz
                L.oz2_fp64mod_tables.argtypes = [i32, i64, P, P, P, P]
                L.oz2_kernel_launches.argtypes = []
                L.oz2_kernel_launches.restype = ctypes.c_ulonglong
                _lib = L
    return _lib


def _check(rc: int, what: str):
    if rc != OK:
        raise Oz2Error(rc, what)


def _mode_id(mode) -> int:
    if isinstance(mode, int):
        return mode
    return {"fast": MODE_FAST, "eq17": MODE_EQ17, "accu": MODE_ACCU}[mode.lower()]


# ---------------------------------------------------------------------------
# constants (host only, no GPU)
# ---------------------------------------------------------------------------
def tables(N: int) -> dict:
    m = np.zeros(N, np.int32)
    y = np.zeros(N, np.int32)
    w = np.zeros(5 * N, np.uint32)
    Mw = np.zeros(5, np.uint32)
    nb, L, T = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
    c = lambda a: a.ctypes.data_as(ctypes.c_void_p)
    _check(lib().oz2_tables(N, c(m), c(y), c(w), c(Mw), ctypes.byref(nb), ctypes.byref(L),
                            ctypes.byref(T)), "oz2_tables")
    words = lambda ws: sum(int(v) << (32 * i) for i, v in enumerate(ws))
    return {"moduli": [int(v) for v in m], "y": [int(v) for v in y],
            "w": [words(w[5 * t:5 * t + 5]) for t in range(N)], "M": words(Mw),
            "nbytes": nb.value, "L": L.value, "T": T.value}


def kernel_launches() -> int:
    """liboz2 kernels launched since the library was loaded (oz2_kernel_launches)."""
    return int(lib().oz2_kernel_launches())


def eq17_k(N: int, q: int) -> int:
    return int(lib().oz2_eq17_k(N, int(q)))


def workspace_bytes(m: int, n: int, k: int, N: int) -> int:
    return int(lib().oz2_workspace_bytes(m, n, k, N))


# ---------------------------------------------------------------------------
# handles (one per device), workspace from torch
# ---------------------------------------------------------------------------
class Handle:
    def __init__(self, device: int):
        import torch

        self.device = int(device)
        h = ctypes.c_void_p()
        _check(lib().oz2_create(ctypes.byref(h), self.device), "oz2_create")
        self._h = h
        self._ws = None
        self._torch = torch

    @property
    def ptr(self):
        return self._h

    def prepare(self, mode, ws_bytes: int = 0):
        torch = self._torch
        _check(lib().oz2_set_mode(self._h, _mode_id(mode)), "oz2_set_mode")
        stream = torch.cuda.current_stream(self.device).cuda_stream
        _check(lib().oz2_set_stream(self._h, ctypes.c_void_p(stream)), "oz2_set_stream")
        if ws_bytes:
            if self._ws is None or self._ws.numel() < ws_bytes:
                self._ws = None
                self._ws = torch.empty(ws_bytes, dtype=torch.uint8, device=f"cuda:{self.device}")
            self._ws.record_stream(torch.cuda.current_stream(self.device))
            _check(lib().oz2_set_workspace(self._h, ctypes.c_void_p(self._ws.data_ptr()), self._ws.numel()),
                   "oz2_set_workspace")
        else:
            _check(lib().oz2_set_workspace(self._h, None, 0), "oz2_set_workspace")

    def set_profiling(self, on: bool):
        _check(lib().oz2_set_profiling(self._h, 1 if on else 0), "oz2_set_profiling")

    def stage_times(self) -> tuple[dict, int]:
        """Summed device ms per stage since the last read, and the call count."""
        ms = np.zeros(len(STAGES), np.float64)
        calls = ctypes.c_int64()
        _check(lib().oz2_stage_times(self._h, ms.ctypes.data_as(ctypes.c_void_p), ctypes.byref(calls)),
               "oz2_stage_times")
        return dict(zip(STAGES, ms.tolist())), calls.value

    def __del__(self):
        try:
            if getattr(self, "_h", None) is not None and _lib is not None:
                _lib.oz2_destroy(self._h)
        except Exception:
            pass


_handles: dict = {}


def handle(device=None) -> Handle:
    import torch

    dev = torch.cuda.current_device() if device is None else int(device)
    if dev not in _handles:
        _handles[dev] = Handle(dev)
    return _handles[dev]


def _vp(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


def _rowmajor(x, dtype):
    import torch

    assert x.is_cuda, "liboz2 takes CUDA tensors (no CPU fallback)"
    assert x.dim() == 2 and x.dtype == dtype, (x.shape, x.dtype)
    if x.stride(1) != 1 or x.stride(0) < max(1, x.shape[1]):
        x = x.contiguous()
    return x


def _ld(x):
    return max(int(x.stride(0)), max(1, int(x.shape[1])))


def _same_device(dev, *xs):
    for x in xs:
        if x is not None and x.device != dev:
            raise ValueError(f"tensor on {x.device}, expected {dev}")


def _out(out, m: int, n: int, dev):
    """The output matrix: a new (m, n) float64 tensor, or `out` validated (the
    library writes m*n doubles with leading dimension out.stride(0))."""
    import torch

    if out is None:
        return torch.empty((m, n), dtype=torch.float64, device=dev)
    if not (out.dtype == torch.float64 and out.device == dev and out.dim() == 2 and tuple(out.shape) == (m, n)
            and out.stride(1) == 1 and out.stride(0) >= max(1, n)):
        raise ValueError(f"out must be a row-major float64 ({m}, {n}) tensor on {dev}; got "
                         f"{out.dtype} {tuple(out.shape)} strides {tuple(out.stride())} on {out.device}")
    return out


def _vec_i32(v, n: int, dev, name: str):
    import torch

    v = v.to(device=dev, dtype=torch.int32).contiguous()
    if v.numel() != n:
        raise ValueError(f"{name}: {v.numel()} entries, expected {n}")
    return v


def ld_res_for(k: int) -> int:
    return max(16, (k + 15) // 16 * 16)


# ---------------------------------------------------------------------------
# main entry point
# ---------------------------------------------------------------------------
def dgemm(A, B, num_moduli: int = 14, mode="fast", out=None):
    """C = A @ B (float64, CUDA) by Ozaki scheme II with `num_moduli` INT8 GEMMs."""
    import torch

    A = _rowmajor(A, torch.float64)
    B = _rowmajor(B, torch.float64)
    m, k = A.shape
    k2, n = B.shape
    if k != k2:
        raise ValueError(f"inner dimensions differ: {A.shape} @ {B.shape}")
    _same_device(A.device, B)
    C = _out(out, m, n, A.device)
    h = handle(A.device.index)
    h.prepare(mode, workspace_bytes(m, n, k, num_moduli))
    _check(lib().oz2_dgemm_ex(h.ptr, m, n, k, _vp(A), _ld(A), _vp(B), _ld(B), _vp(C), _ld(C),
                              num_moduli), "oz2_dgemm_ex")
    return C


class Prepared:
    """A converted operand (oz2_prepare_a / oz2_prepare_b): its exponents and
    its N residue planes in device memory owned by this object (one object, one
    allocation; released by release() or garbage collection)."""

    def __init__(self, X, side: str, num_moduli: int = 14, mode="fast"):
        import torch

        X = _rowmajor(X, torch.float64)
        self.side = side
        self.N = num_moduli
        self.mode = mode
        self.device = X.device
        self.h = handle(X.device.index)
        self.h.prepare(mode)
        self._p = ctypes.c_void_p()
        if side == "A":
            self.rows, self.k = X.shape
            _check(lib().oz2_prepare_a(self.h.ptr, self.rows, self.k, _vp(X), _ld(X), num_moduli,
                                       ctypes.byref(self._p)), "oz2_prepare_a")
        else:
            self.k, self.rows = X.shape
            _check(lib().oz2_prepare_b(self.h.ptr, self.k, self.rows, _vp(X), _ld(X), num_moduli,
                                       ctypes.byref(self._p)), "oz2_prepare_b")

    @property
    def ptr(self):
        if self._p is None or not self._p.value:
            raise ValueError("prepared operand already released")
        return self._p

    def reprepare(self, X):
        """Convert another matrix of the same shape into this object's memory
        (oz2_reprepare; stream-ordered after work already queued that reads it)."""
        import torch

        X = _rowmajor(X, torch.float64)
        _same_device(self.device, X)
        shape = (self.rows, self.k) if self.side == "A" else (self.k, self.rows)
        if tuple(X.shape) != shape:
            raise ValueError(f"reprepare: shape {tuple(X.shape)}, prepared with {shape}")
        self.h.prepare(self.mode)
        _check(lib().oz2_reprepare(self.h.ptr, self.ptr, _vp(X), _ld(X)), "oz2_reprepare")
        return self

    def release(self):
        if self._p is not None and self._p.value:
            # the object's memory may still be read by queued work: wait first
            self.h._torch.cuda.current_stream(self.device).synchronize()
            _check(lib().oz2_release(self._p), "oz2_release")
        self._p = None

    def __del__(self):
        try:
            self.release()
        except Exception:
            pass


class PreparedB(Prepared):
    """B-stationary products: B (k x n) converted once, then any number of row
    blocks of A (oz2_dgemm_prepared), or prepared A blocks (oz2_dgemm_prep2)."""

    def __init__(self, B, num_moduli: int = 14, mode="fast"):
        super().__init__(B, "B", num_moduli, mode)
        self.n = self.rows

    def dgemm(self, A, out=None):
        import torch

        A = _rowmajor(A, torch.float64)
        _same_device(self.device, A)
        m = A.shape[0]
        if A.shape[1] != self.k:
            raise ValueError(f"A has {A.shape[1]} columns, B was prepared with k = {self.k}")
        C = _out(out, m, self.n, self.device)
        self.h.prepare(self.mode, workspace_bytes(m, self.n, self.k, self.N))
        _check(lib().oz2_dgemm_prepared(self.h.ptr, self.ptr, m, _vp(A), _ld(A), _vp(C), _ld(C)),
               "oz2_dgemm_prepared")
        return C


class PreparedA(Prepared):
    def __init__(self, A, num_moduli: int = 14, mode="fast"):
        super().__init__(A, "A", num_moduli, mode)
        self.m = self.rows


def dgemm_prep2(pa: PreparedA, pb: PreparedB, out=None):
    """Lines 6-10 on two prepared operands (oz2_dgemm_prep2)."""
    if pa.k != pb.k or pa.N != pb.N or pa.device != pb.device:
        raise ValueError("prepared operands do not match (k, N, device)")
    C = _out(out, pa.m, pb.n, pa.device)
    h = pa.h
    h.prepare(pa.mode, workspace_bytes(pa.m, pb.n, 0, pa.N))
    _check(lib().oz2_dgemm_prep2(h.ptr, pa.ptr, pb.ptr, _vp(C), _ld(C)), "oz2_dgemm_prep2")
    return C


def set_sm_limit(sms: int, device=None):
    """Persistent-GEMM SM budget on this device's handle (0 = all)."""
    _check(lib().oz2_set_sm_limit(handle(device).ptr, int(sms)), "oz2_set_sm_limit")


# ---------------------------------------------------------------------------
# K-split (2-D multi-GPU) pieces: see include/oz2.h
# ---------------------------------------------------------------------------
def kslice_stats_rows(A, E_global=None, mode="fast"):
    """Phase 1 (E_global None): max chunk exponents of the rows of this K slice
    (int32; INT32_MIN none, INT32_MAX non-finite).  Phase 2: the uint64 partial
    sums (returned as int64) relative to the global exponents."""
    import torch

    A = _rowmajor(A, torch.float64)
    m, k = A.shape
    h = handle(A.device.index)
    h.prepare(mode)
    if E_global is None:
        E = torch.empty(m, dtype=torch.int32, device=A.device)
        _check(lib().oz2_kslice_stats_rows(h.ptr, m, k, _vp(A), _ld(A), None, _vp(E), None), "oz2_kslice_stats_rows")
        return E
    S = torch.empty(m, dtype=torch.int64, device=A.device)
    _check(lib().oz2_kslice_stats_rows(h.ptr, m, k, _vp(A), _ld(A), _vp(E_global.contiguous()), None, _vp(S)),
           "oz2_kslice_stats_rows")
    return S


def kslice_stats_cols(B, E_global=None, mode="fast"):
    import torch

    B = _rowmajor(B, torch.float64)
    k, n = B.shape
    h = handle(B.device.index)
    h.prepare(mode, 16 * n * ((k + 255) // 256) + 4 * n + 4096)
    if E_global is None:
        E = torch.empty(n, dtype=torch.int32, device=B.device)
        _check(lib().oz2_kslice_stats_cols(h.ptr, k, n, _vp(B), _ld(B), None, _vp(E), None), "oz2_kslice_stats_cols")
        return E
    S = torch.empty(n, dtype=torch.int64, device=B.device)
    _check(lib().oz2_kslice_stats_cols(h.ptr, k, n, _vp(B), _ld(B), _vp(E_global.contiguous()), None, _vp(S)),
           "oz2_kslice_stats_cols")
    return S


def exponents_from_stats(E, S, k_total: int, N: int, mode="fast"):
    import torch

    cnt = E.numel()
    e = torch.empty(cnt, dtype=torch.int32, device=E.device)
    h = handle(E.device.index)
    h.prepare(mode)
    _check(lib().oz2_exponents_from_stats(h.ptr, cnt, _vp(E.contiguous()), _vp(S.contiguous()), int(k_total), N,
                                          _vp(e)), "oz2_exponents_from_stats")
    return e


def modmul_residues(Ares, Bres, k: int, rows_per_block: int = 0):
    """Lines 6-7: uint8 c''_t planes, [ceil(m/rpb)][N][rpb][n] (rpb = m: [1][N][m][n])."""
    import torch

    N, m, ldr = Ares.shape
    n = Bres.shape[1]
    rpb = rows_per_block or m
    nblk = (m + rpb - 1) // rpb
    R = torch.empty((nblk, N, rpb, n), dtype=torch.uint8, device=Ares.device)
    h = handle(Ares.device.index)
    h.prepare("fast", workspace_bytes(m, n, k, N))
    _check(lib().oz2_modmul_residues(h.ptr, m, n, k, _vp(Ares), _vp(Bres), ldr, N, _vp(R), rpb),
           "oz2_modmul_residues")
    return R


def crt_sum(R, parts: int, part_stride: int, m: int, n: int, e, f, N: int, out=None, beta=None):
    """Lines 7-10 over `parts` partial residue planes: C = D^-1 X E^-1.
    beta: a certificate from certify() (refusal: C := NaN, status())."""
    import torch

    C = _out(out, m, n, R.device)
    e = _vec_i32(e, m, R.device, "e")
    f = _vec_i32(f, n, R.device, "f")
    _same_device(R.device, beta)
    h = handle(R.device.index)
    h.prepare("fast")
    _check(lib().oz2_crt_sum(h.ptr, parts, m, n, _vp(R), part_stride, _vp(e), _vp(f), N,
                             _vp(C), _ld(C), _vp(beta)), "oz2_crt_sum")
    return C


def dgemm_scaled(A, B, e, f, num_moduli: int = 14, out=None):
    """Alg. 1 lines 2-10 with given exponent vectors e (rows of A), f (columns of B).
    Condition (13) is certified on the device (oz2_certify): on refusal C is NaN
    and status() raises OZ2_ERR_NOT_UNIQUE."""
    import torch

    A = _rowmajor(A, torch.float64)
    B = _rowmajor(B, torch.float64)
    m, k = A.shape
    n = B.shape[1]
    _same_device(A.device, B)
    e = _vec_i32(e, m, A.device, "e")
    f = _vec_i32(f, n, A.device, "f")
    C = _out(out, m, n, A.device)
    h = handle(A.device.index)
    h.prepare("fast", workspace_bytes(m, n, k, num_moduli))
    _check(lib().oz2_dgemm_scaled(h.ptr, m, n, k, _vp(A), _ld(A), _vp(B), _ld(B), _vp(e), _vp(f), _vp(C), _ld(C),
                                  num_moduli), "oz2_dgemm_scaled")
    return C


def gemm(A, B, num_moduli: int = 14, alpha: float = 1.0, beta: float = 0.0, C=None,
         transA: bool = False, transB: bool = False, mode="fast"):
    """C := alpha op(A) op(B) + beta C (float64, CUDA, row-major; BLAS DGEMM semantics)
    through oz2_dgemm_op.  A, B are the STORED matrices: op(A) = A.T if transA."""
    import torch

    A = _rowmajor(A, torch.float64)
    B = _rowmajor(B, torch.float64)
    m, k = (A.shape[1], A.shape[0]) if transA else A.shape
    kb, n = (B.shape[1], B.shape[0]) if transB else B.shape
    if k != kb:
        raise ValueError(f"inner dimensions differ: op(A) {m}x{k}, op(B) {kb}x{n}")
    if C is None:
        C = torch.zeros((m, n), dtype=torch.float64, device=A.device)
    assert C.is_cuda and C.dtype == torch.float64 and C.shape == (m, n) and C.stride(1) == 1
    h = handle(A.device.index)
    h.prepare(mode, workspace_bytes(m, n, k, num_moduli))
    _check(lib().oz2_dgemm_op(h.ptr, OP_T if transA else OP_N, OP_T if transB else OP_N, m, n, k,
                              float(alpha), _vp(A), _ld(A), _vp(B), _ld(B), float(beta), _vp(C), _ld(C),
                              num_moduli), "oz2_dgemm_op")
    return C


LOWER, UPPER = 1, 2


def syrk(A, num_moduli: int = 14, uplo: str = "L", trans: bool = False, alpha: float = 1.0,
         beta: float = 0.0, C=None, mode="fast"):
    """C := alpha op(A) op(A)^T + beta C on the `uplo` triangle only (BLAS DSYRK
    semantics, row-major) through oz2_dsyrk; op(A) = A.T if trans.  The other
    triangle of C is left as it was (zeros when C is None)."""
    import torch

    A = _rowmajor(A, torch.float64)
    n, k = (A.shape[1], A.shape[0]) if trans else A.shape
    if C is None:
        C = torch.zeros((n, n), dtype=torch.float64, device=A.device)
    assert C.is_cuda and C.dtype == torch.float64 and C.shape == (n, n) and C.stride(1) == 1
    h = handle(A.device.index)
    h.prepare(mode, workspace_bytes(n, n, k, num_moduli))
    _check(lib().oz2_dsyrk(h.ptr, LOWER if uplo.upper() == "L" else UPPER, OP_T if trans else OP_N, n, k,
                           float(alpha), _vp(A), _ld(A), float(beta), _vp(C), _ld(C), num_moduli), "oz2_dsyrk")
    return C


def trmm(A, B, num_moduli: int = 14, side: str = "L", uplo: str = "L", transA: bool = False,
         unit: bool = False, alpha: float = 1.0, mode="fast"):
    """B := alpha op(tri(A)) B (side "L") or alpha B op(tri(A)) (side "R"), in
    place on the CUDA tensor B (BLAS DTRMM semantics, row-major) through oz2_dtrmm."""
    import torch

    A = _rowmajor(A, torch.float64)
    assert B.is_cuda and B.dtype == torch.float64 and B.dim() == 2 and B.stride(1) == 1
    m, n = B.shape
    na = m if side.upper() == "L" else n
    assert A.shape == (na, na)
    h = handle(A.device.index)
    h.prepare(mode, workspace_bytes(m, n, na, num_moduli))
    _check(lib().oz2_dtrmm(h.ptr, 0 if side.upper() == "L" else 1, LOWER if uplo.upper() == "L" else UPPER,
                           OP_T if transA else OP_N, 1 if unit else 0, m, n, float(alpha), _vp(A), _ld(A),
                           _vp(B), _ld(B), num_moduli), "oz2_dtrmm")
    return B


def gemm_strided_batched(A, B, num_moduli: int = 14, alpha: float = 1.0, beta: float = 0.0, C=None,
                         transA: bool = False, transB: bool = False, mode="fast"):
    """Batched gemm over the leading dimension of contiguous 3-D tensors (one
    oz2_dgemm_strided_batched call)."""
    import torch

    assert A.dim() == 3 and B.dim() == 3 and A.shape[0] == B.shape[0]
    A = A.contiguous()
    B = B.contiguous()
    batch = A.shape[0]
    m, k = (A.shape[2], A.shape[1]) if transA else A.shape[1:]
    kb, n = (B.shape[2], B.shape[1]) if transB else B.shape[1:]
    if k != kb:
        raise ValueError("inner dimensions differ")
    if C is None:
        C = torch.zeros((batch, m, n), dtype=torch.float64, device=A.device)
    assert C.is_contiguous() and C.shape == (batch, m, n)
    h = handle(A.device.index)
    h.prepare(mode, workspace_bytes(m, n, k, num_moduli))
    _check(lib().oz2_dgemm_strided_batched(
        h.ptr, OP_T if transA else OP_N, OP_T if transB else OP_N, m, n, k, float(alpha),
        _vp(A), max(1, A.shape[2]), A.shape[1] * A.shape[2], _vp(B), max(1, B.shape[2]), B.shape[1] * B.shape[2],
        float(beta), _vp(C), max(1, n), m * n, batch, num_moduli), "oz2_dgemm_strided_batched")
    return C


def dgemm_host(A: np.ndarray, B: np.ndarray, num_moduli: int = 14, mode="fast", out=None,
               device=None) -> np.ndarray:
    """End-to-end through oz2_dgemm_host: host (ideally pinned) buffers in and out."""
    A = np.ascontiguousarray(A, dtype=np.float64)
    B = np.ascontiguousarray(B, dtype=np.float64)
    m, k = A.shape
    n = B.shape[1]
    C = out if out is not None else np.empty((m, n), np.float64)
    h = handle(device)
    ws = workspace_bytes(m, n, k, num_moduli) + 8 * (m * max(k, 1) + max(k, 1) * n + m * n) + 4096
    h.prepare(mode, ws)
    p = lambda a: a.ctypes.data_as(ctypes.c_void_p)
    _check(lib().oz2_dgemm_host(h.ptr, m, n, k, p(A), max(k, 1), p(B), max(n, 1), p(C), max(n, 1),
                                num_moduli), "oz2_dgemm_host")
    return C


# ---------------------------------------------------------------------------
# split API (stage parity tests)
# ---------------------------------------------------------------------------
def scale_rows(A, N: int, mode="fast"):
    import torch

    A = _rowmajor(A, torch.float64)
    m, k = A.shape
    e = torch.empty(m, dtype=torch.int32, device=A.device)
    h = handle(A.device.index)
    h.prepare(mode)
    _check(lib().oz2_scale_rows(h.ptr, m, k, _vp(A), _ld(A), N, _vp(e)), "oz2_scale_rows")
    return e


def scale_accu(A, B, N: int):
    """OS II-accu exponents (reading R18) of the product A B: (e, f)."""
    import torch

    A = _rowmajor(A, torch.float64)
    B = _rowmajor(B, torch.float64)
    m, k = A.shape
    n = B.shape[1]
    e = torch.empty(m, dtype=torch.int32, device=A.device)
    f = torch.empty(n, dtype=torch.int32, device=A.device)
    h = handle(A.device.index)
    h.prepare("fast", workspace_bytes(m, n, k, 1))
    _check(lib().oz2_scale_accu(h.ptr, m, n, k, _vp(A), _ld(A), _vp(B), _ld(B), N, _vp(e), _vp(f)),
           "oz2_scale_accu")
    return e, f


def scale_cols(B, N: int, mode="fast"):
    import torch

    B = _rowmajor(B, torch.float64)
    k, n = B.shape
    f = torch.empty(n, dtype=torch.int32, device=B.device)
    h = handle(B.device.index)
    h.prepare(mode, 1 << 20 if k * n == 0 else 16 * n * ((k + 255) // 256) + 4 * n + 4096)
    _check(lib().oz2_scale_cols(h.ptr, k, n, _vp(B), _ld(B), N, _vp(f)), "oz2_scale_cols")
    return f


def trunc_rows(A, e):
    import torch

    A = _rowmajor(A, torch.float64)
    m, k = A.shape
    out = torch.empty((m, k), dtype=torch.float64, device=A.device)
    h = handle(A.device.index)
    h.prepare("fast")
    _check(lib().oz2_trunc_rows(h.ptr, m, k, _vp(A), _ld(A), _vp(e.contiguous()), _vp(out)), "oz2_trunc_rows")
    return out


def trunc_cols(B, f):
    import torch

    B = _rowmajor(B, torch.float64)
    k, n = B.shape
    out = torch.empty((n, k), dtype=torch.float64, device=B.device)
    h = handle(B.device.index)
    h.prepare("fast")
    _check(lib().oz2_trunc_cols(h.ptr, k, n, _vp(B), _ld(B), _vp(f.contiguous()), _vp(out)), "oz2_trunc_cols")
    return out


def residues_rows(A, e, N: int, ld_res: int | None = None):
    """int8 planes [N][m][ld_res]; entries [k, ld_res) of each row are unspecified."""
    import torch

    A = _rowmajor(A, torch.float64)
    m, k = A.shape
    ldr = ld_res or ld_res_for(k)
    out = torch.zeros((N, m, ldr), dtype=torch.int8, device=A.device)
    h = handle(A.device.index)
    h.prepare("fast")
    _check(lib().oz2_residues_rows(h.ptr, m, k, _vp(A), _ld(A), _vp(e.contiguous()), N, _vp(out), ldr),
           "oz2_residues_rows")
    return out


def residues_cols(B, f, N: int, ld_res: int | None = None):
    """int8 planes [N][n][ld_res] holding B'^T (K-major)."""
    import torch

    B = _rowmajor(B, torch.float64)
    k, n = B.shape
    ldr = ld_res or ld_res_for(k)
    out = torch.zeros((N, n, ldr), dtype=torch.int8, device=B.device)
    h = handle(B.device.index)
    h.prepare("fast")
    _check(lib().oz2_residues_cols(h.ptr, k, n, _vp(B), _ld(B), _vp(f.contiguous()), N, _vp(out), ldr),
           "oz2_residues_cols")
    return out


def modmul(Ares, Bres, k: int):
    """int32 [N][m][n] = Ares[t] @ Bres[t]^T over the first k columns, on tcgen05."""
    import torch

    N, m, ldr = Ares.shape
    n = Bres.shape[1]
    assert Bres.shape[0] == N and Bres.shape[2] == ldr and Ares.is_contiguous() and Bres.is_contiguous()
    out = torch.empty((N, m, n), dtype=torch.int32, device=Ares.device)
    h = handle(Ares.device.index)
    h.prepare("fast", 4096)
    _check(lib().oz2_modmul(h.ptr, m, n, k, _vp(Ares), _vp(Bres), ldr, N, _vp(out)), "oz2_modmul")
    return out


def crt(Cprod, e, f, out=None, beta=None):
    """Lines 7-10 on int32 products; beta: a certificate from certify()."""
    N, m, n = Cprod.shape
    C = _out(out, m, n, Cprod.device)
    e = _vec_i32(e, m, Cprod.device, "e")
    f = _vec_i32(f, n, Cprod.device, "f")
    _same_device(Cprod.device, beta)
    h = handle(Cprod.device.index)
    h.prepare("fast")
    _check(lib().oz2_crt(h.ptr, m, n, _vp(Cprod.contiguous()), _vp(e), _vp(f), N,
                         _vp(C), _ld(C), _vp(beta)), "oz2_crt")
    return C


def certify(A, B, e, f, N: int):
    """Device int32 tensor [beta]: c_max <= 2^beta for the product A B under the
    exponents e, f (oz2_certify; beta <= tables(N)["L"] certifies condition (13))."""
    import torch

    A = _rowmajor(A, torch.float64)
    B = _rowmajor(B, torch.float64)
    _same_device(A.device, B)
    m, k = A.shape
    n = B.shape[1]
    e = _vec_i32(e, m, A.device, "e")
    f = _vec_i32(f, n, A.device, "f")
    beta = torch.empty(1, dtype=torch.int32, device=A.device)
    h = handle(A.device.index)
    h.prepare("fast", 16 * n * ((k + 255) // 256) + 4 * n + 4096)
    _check(lib().oz2_certify(h.ptr, m, n, k, _vp(A), _ld(A), _vp(B), _ld(B), _vp(e), _vp(f), N, _vp(beta)),
           "oz2_certify")
    return beta


def status(device=None):
    """Waits for this device's handle and raises Oz2Error(OZ2_ERR_NOT_UNIQUE) if
    a certified call refused since the last status() (oz2_status)."""
    _check(lib().oz2_status(handle(device).ptr), "oz2_status")


def set_certify(on: bool, device=None):
    _check(lib().oz2_set_certify(handle(device).ptr, 1 if on else 0), "oz2_set_certify")


# ---------------------------------------------------------------------------
# the FP64 prime-modulus regime (include/oz2.h)
# ---------------------------------------------------------------------------
def fp64mod_tables(s: int, q: int) -> dict:
    m = np.zeros(s, np.int64)
    Mw = np.zeros(17, np.uint32)
    L, T = ctypes.c_int32(), ctypes.c_int32()
    c = lambda a: a.ctypes.data_as(ctypes.c_void_p)
    _check(lib().oz2_fp64mod_tables(s, int(q), c(m), c(Mw), ctypes.byref(L), ctypes.byref(T)), "oz2_fp64mod_tables")
    return {"moduli": [int(v) for v in m], "M": sum(int(v) << (32 * i) for i, v in enumerate(Mw)),
            "L": L.value, "T": T.value}


def dgemm_fp64mod(A, B, s: int = 16, v: int = 2, out=None, A2=None, B2=None):
    """C ~= A @ B in the FP64 prime-modulus regime with s primes: a (v, m, n)
    float64 tensor, word 0 the most significant (oz2_dgemm_fp64mod).  A2, B2:
    second words of double-word inputs (A + A2, B + B2; |A2| <= u |A|, Eq. 23)."""
    import torch

    A = _rowmajor(A, torch.float64).contiguous()
    B = _rowmajor(B, torch.float64).contiguous()
    _same_device(A.device, B, A2, B2)
    if A2 is not None:
        A2 = A2.to(torch.float64).contiguous()
        assert A2.shape == A.shape
    if B2 is not None:
        B2 = B2.to(torch.float64).contiguous()
        assert B2.shape == B.shape
    m, k = A.shape
    k2, n = B.shape
    if k != k2:
        raise ValueError(f"inner dimensions differ: {A.shape} @ {B.shape}")
    if out is None:
        out = torch.empty((v, m, n), dtype=torch.float64, device=A.device)
    if not (out.dtype == torch.float64 and out.device == A.device and tuple(out.shape) == (v, m, n)
            and out.is_contiguous()):
        raise ValueError(f"out must be a contiguous float64 ({v}, {m}, {n}) tensor on {A.device}")
    h = handle(A.device.index)
    h.prepare("fast", int(lib().oz2_fp64mod_workspace_bytes(m, n, max(k, 1), s)))
    _check(lib().oz2_dgemm_fp64mod_dw(h.ptr, m, n, k, _vp(A), _vp(A2), _ld(A), _vp(B), _vp(B2), _ld(B), s, v,
                                      _vp(out), max(1, n), m * max(1, n)), "oz2_dgemm_fp64mod_dw")
    return out
