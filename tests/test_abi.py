"""CPU-side checks of the C-ABI boundary (no GPU): the library loads, exports
every symbol include/oz2.h declares, and its host constants agree with the
oracle's (two independent implementations)."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def oz2():
    from paper_2504_08009_b200 import build, oz2 as o
    build.build()
    o.lib()
    return o


def _header_functions():
    src = open(os.path.join(ROOT, "include", "oz2.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(oz2_[a-z0-9_]+)\s*\(", src)))


def test_header_symbols_exported(oz2):
    declared = _header_functions()
    assert sorted(oz2.SYMBOLS) == declared
    out = subprocess.run(["nm", "-D", "--defined-only", oz2.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\sT\s(oz2_\w+)", out))
    for name in declared:
        assert name in exported, name
        getattr(oz2.lib(), name)


def test_plain_c_signatures():
    src = open(os.path.join(ROOT, "include", "oz2.h")).read()
    assert "torch" not in src.lower() and "at::" not in src and "Tensor" not in src
    assert 'extern "C"' in src


def test_library_is_sm100a(oz2):
    out = subprocess.run(["cuobjdump", "--list-elf", oz2.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", oz2.LIB_PATH], capture_output=True, text=True).stdout
    assert "UTCIMMA" in sass            # tcgen05.mma kind::i8
    assert "UTMALDG" in sass            # TMA tile loads
    assert "LDTM" in sass               # tcgen05.ld


@pytest.mark.parametrize("N", list(range(2, 21)))
def test_tables_match_oracle(oz2, oracle, N):
    t = oz2.tables(N)
    c = oracle.constants(N)
    assert t["moduli"] == c["moduli"]
    assert t["y"] == c["y"]
    assert t["L"] == c["L"] and t["T"] == c["T"]
    assert t["M"] == c["M"]
    assert t["nbytes"] == (c["M"].bit_length() + 7) // 8
    assert t["w"] == list(c["w"])
    assert all(0 < w < c["M"] for w in t["w"])


def test_eq17_matches_oracle(oz2, oracle):
    for N in (2, 3, 8, 14, 16, 20):
        for q in (1, 7, 1024, 4096, 16384, 65536, 131071):
            assert oz2.eq17_k(N, q) == oracle.eq17_k(N, q)


def test_errors_without_device(oz2):
    import ctypes
    L = oz2.lib()
    assert L.oz2_strerror(0) == b"ok"
    assert L.oz2_version() >= 100
    assert L.oz2_workspace_bytes(64, 64, 64, 14) > 14 * 2 * 64 * 64
    assert L.oz2_workspace_bytes(64, 64, 64, 21) == 0
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:
        has_gpu = False
    if not has_gpu:
        h = ctypes.c_void_p()
        assert L.oz2_create(ctypes.byref(h), 0) != 0       # fails loudly: no device, no fallback
