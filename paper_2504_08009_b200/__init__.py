"""paper_2504_08009_b200 -- a B200-native Ozaki scheme II (INT8 moduli) DGEMM.

The compute path is the C-ABI library ``liboz2.so`` (hand-written sm_100a
CUDA kernels, declared in ``include/oz2.h``); ``oz2`` is its thin ctypes
binding.  Importing this package does not load the library: the first call
into ``oz2`` does, and fails loudly if it is missing.  There is no CPU
fallback.
"""
__all__ = ["oz2", "inputs", "dist"]
