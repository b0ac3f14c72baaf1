"""Build liboz2.so (the product library) in-tree with nvcc for sm_100a.

    python -m paper_2504_08009_b200.build        # or __graft_entry__.build()

Two translation units compiled in parallel and linked into one shared library:
liboz2.cu (conversion, CRT, accu, K-split, certificate kernels, the C ABI) and
liboz2_gemm.cu (the persistent tcgen05 GEMM).  An object is rebuilt only when
one of its sources changed.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "liboz2.so")
ROOT = os.path.dirname(HERE)
OBJDIR = os.path.join(HERE, "build")

COMMON = ["oz2_device.cuh", "oz2_kernels.h", "oz2_tables.h", "crt_device.cuh"]
UNITS = {
    "liboz2.cu": COMMON + ["liboz2.cu", "scale.cu", "crt.cu", "accu.cu", "kslice.cu", "certify.cu", "fp64mod.cu", "api.cu"],
    "liboz2_gemm.cu": COMMON + ["liboz2_gemm.cu", "gemm.cu"],
    "tables.cpp": ["tables.cpp", "oz2_tables.h"],
}

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = [*ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-warn-spills"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.isabs(cand) and os.path.exists(cand) or not os.path.isabs(cand)):
            return cand
    return "nvcc"


def _obj(unit: str) -> str:
    return os.path.join(OBJDIR, unit.replace(".", "_") + ".o")


def _stale(unit: str) -> bool:
    o = _obj(unit)
    if not os.path.exists(o):
        return True
    t = os.path.getmtime(o)
    hdr = os.path.join(ROOT, "include", "oz2.h")
    return any(os.path.getmtime(os.path.join(CSRC, d)) > t for d in UNITS[unit]) or os.path.getmtime(hdr) > t


def needs_build() -> bool:
    return not os.path.exists(LIB) or any(_stale(u) for u in UNITS) or \
        any(os.path.getmtime(_obj(u)) > os.path.getmtime(LIB) for u in UNITS)


def build(force: bool = False, verbose: bool = False, extra_flags: list[str] | None = None,
          lib: str | None = None) -> str:
    """Compile the stale units in parallel and link.  extra_flags / lib: an
    alternative build (e.g. -DOZ2_EXPERIMENTS into another .so) for A/B runs."""
    out = lib or LIB
    objdir = OBJDIR if not extra_flags else OBJDIR + "_" + str(abs(hash(tuple(extra_flags))) % 10**8)
    os.makedirs(objdir, exist_ok=True)
    procs = []
    for unit in UNITS:
        o = os.path.join(objdir, os.path.basename(_obj(unit)))
        if not force and not extra_flags and not _stale(unit):
            continue
        cmd = [nvcc(), *NVCC_FLAGS, *(extra_flags or []), "-c", "-o", o + ".tmp", os.path.join(CSRC, unit)]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        procs.append((subprocess.Popen(cmd, cwd=CSRC), o))
    for p, o in procs:
        if p.wait() != 0:
            raise subprocess.CalledProcessError(p.returncode, "nvcc")
        os.replace(o + ".tmp", o)
    if procs or force or not os.path.exists(out) or needs_build():
        objs = [os.path.join(objdir, os.path.basename(_obj(u))) for u in UNITS]
        cmd = [nvcc(), *ARCH, "-shared", "-Xcompiler", "-fPIC", "-o", out + ".tmp", *objs]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.check_call(cmd, cwd=CSRC)
        os.replace(out + ".tmp", out)
    return out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
