"""CPU pins of the FP32-quotient steps the CUDA residue kernels (scale.cu,
residue_odd) and the GEMM drain (crt_device.cuh, reduce_line7_lowbyte) rely on
(DESIGN.md section 7).  Both form q = rint(f * RN_binary32(1/m) + 1.5 2^23) with
one binary32 FMA and claim it equals an exact integer quotient:

  residues (Eq. 1, odd m): f = y, 0 <= y < 2^20,
      q == floor((y + (m-1)/2) / m)   (so y - q m is the symmetric residue)
  line 7 (Alg. 1 line 7): f = y - (m-1)/2, 2^20 <= y < 2^22.2,
      q == floor(y / m)                (so y - q m = c'' in [0, m))

The FMA is emulated exactly in integers (binary32 1/m is an integer mantissa
times a power of two; the product and the 1.5 2^23 addend are summed exactly and
rounded once, ties to even), exhaustively over every y of both ranges and every
odd modulus of the table (reading R1).  Independent of the CUDA code: only the
arithmetic claim is checked, against Python integer division.
"""
import numpy as np
import pytest

MODULI = [256, 255, 253, 251, 247, 239, 233, 229, 227, 223, 217, 211, 199, 197, 193, 191, 241, 181, 179, 173]
ODD = [m for m in MODULI if m % 2]


def f32_recip(m):
    """RN_binary32(1/m) as (mantissa, exponent): value = mant * 2^exp exactly."""
    v = np.float32(1.0) / np.float32(m)            # IEEE division, correctly rounded
    mant, exp = np.frexp(np.float64(v))            # exact: binary32 fits binary64
    mi = int(mant * (1 << 24))
    assert mi * 2.0 ** (exp - 24) == float(v)
    return mi, exp - 24


def fma_round_to_int(f, m):
    """rint(f * RN(1/m)) for int64 arrays f, |f| < 2^23, as the binary32 FMA with
    the 1.5 2^23 addend computes it (result in [2^23, 2^24): ulp 1, ties to even)."""
    mi, e = f32_recip(m)
    assert e < 0
    s = -e
    P = f.astype(np.int64) * mi                   # exact: |f| < 2^23, mi < 2^24
    q = P >> s                                     # floor(P / 2^s)
    rem = P - (q << s)
    half = np.int64(1) << (s - 1)
    up = (rem > half) | ((rem == half) & ((q & 1) == 1))
    return q + up.astype(np.int64)


@pytest.mark.parametrize("m", ODD)
def test_residue_quotient_exhaustive(m):
    y = np.arange(0, 1 << 20, dtype=np.int64)
    q = fma_round_to_int(y, m)
    h = (m - 1) // 2
    assert np.array_equal(q, (y + h) // m)
    r = y - q * m
    assert r.min() >= -h and r.max() <= h          # the symmetric residue of Eq. (1)


@pytest.mark.parametrize("m", ODD)
def test_line7_quotient_exhaustive(m):
    lo, hi = 1 << 20, int(2 ** 22.2) + 1
    y = np.arange(lo, hi, dtype=np.int64)
    h = (m - 1) // 2
    q = fma_round_to_int(y - h, m)
    assert np.array_equal(q, y // m)
    r = y - q * m
    assert r.min() >= 0 and r.max() < m            # c'' in [0, m) (reading R8)


def test_line7_range_covers_every_int32():
    """The drain's y = hi k18s + lo + 2^21 - 8 k18s stays in [2^20, 2^22.2) for
    every int32 c' = hi 2^18 + lo and every modulus, and y == c' (mod m)."""
    for m in ODD:
        k18 = pow(2, 18, m)
        k18s = k18 - m if 2 * k18 > m else k18
        for c in (-(1 << 31), (1 << 31) - 1, -1, 0, 1, 123456789, -987654321, (1 << 18) - 1, -(1 << 18)):
            hi, lo = c >> 18, c & 0x3FFFF
            y = hi * k18s + lo + (1 << 21) - 8 * k18s
            assert (1 << 20) <= y < 2 ** 22.2
            assert (y - c) % m == 0


def test_bit_offsets_vanish_mod_256():
    """0x4B000000 and 0x4B400000 * m are multiples of 256: the low byte of
    y' + qb (2^32 - m) is y - q m mod 256 (residue kernels and line 7)."""
    for m in MODULI:
        assert 0x4B000000 % 256 == 0 and (0x4B400000 * m) % 256 == 0
        for y, q in ((5, 0), (1000, 3), ((1 << 20) - 1, 4000)):
            yb, qb = 0x4B000000 + y, 0x4B400000 + q
            assert ((yb + qb * ((1 << 32) - m)) % (1 << 32)) % 256 == (y - q * m) % 256
