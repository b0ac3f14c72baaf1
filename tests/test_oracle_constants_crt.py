"""Pins for the oracle's Eq. (1), moduli table, CRT constants and CRT.

Each check compares the oracle with something other than itself: the paper's
printed table, Python's own integer arithmetic (math.prod, pow(x, -1, m),
%, bit_length), or brute-force enumeration.
"""
import math
import random

import pytest

from conftest import golden


def test_smod_paper_and_spec_examples(oracle):
    # Eq. (1); examples SPEC.md:50-53; tie PAPER.md:455-456
    assert oracle.smod(7, 5) == 2
    assert oracle.smod(103, 5) == -2
    assert oracle.smod(128, 256) == -128
    assert oracle.smod(-128, 256) == -128
    assert oracle.smod(0, 17) == 0
    assert oracle.smod(300, 256) == 44
    assert oracle.smod(300, 255) == 45


def test_smod_bruteforce(oracle):
    # unique characterisation of Eq. (1): r == a (mod m) and -m/2 <= r < m/2
    ms = list(range(2, 40)) + [127, 128, 173, 191, 241, 253, 255, 256, 300]
    for m in ms:
        for a in range(-3 * m - 5, 3 * m + 6):
            r = oracle.smod(a, m)
            assert (r - a) % m == 0
            assert -m <= 2 * r < m, (a, m, r)
            assert oracle.smod_long(a, m) == r


def test_moduli_table_is_eq18(oracle):
    eq18 = [int(v) for v in golden("eq18_moduli.txt")[0]]
    c16 = oracle.constants(16)
    assert c16["moduli"] == eq18
    assert abs(c16["moduli"][15] / c16["moduli"][0] - 0.74) < 0.01
    for N in range(2, 21):
        assert oracle.constants(N)["moduli"] == oracle.constants(20)["moduli"][:N]


def test_moduli_extension_reading_R1(oracle):
    # R1: m_17..m_20 are, one at a time, the largest v <= 256 coprime to all earlier moduli
    mods = oracle.constants(20)["moduli"]
    for t in range(16, 20):
        cands = [v for v in range(256, 1, -1)
                 if v not in mods[:t] and all(math.gcd(v, u) == 1 for u in mods[:t])]
        assert mods[t] == cands[0]
    assert mods[16:] == [241, 181, 179, 173]
    for i in range(20):
        for j in range(i):
            assert math.gcd(mods[i], mods[j]) == 1


@pytest.mark.parametrize("N", list(range(2, 21)))
def test_crt_constants(oracle, N):
    c = oracle.constants(N)
    m = c["moduli"]
    M = math.prod(m)
    assert c["M"] == M
    for t in range(N):
        Mt = M // m[t]
        assert c["y"][t] == pow(Mt, -1, m[t])          # least positive inverse (R2)
        assert c["w"][t] == Mt * c["y"][t]
        assert c["w"][t] % m[t] == 1
        for s in range(N):
            if s != t:
                assert c["w"][t] % m[s] == 0
    L = (M // 2 - 1).bit_length() - 1                   # floor(log2(M/2 - 1))
    assert c["L"] == L and c["T"] == L // 2
    assert 4 ** c["T"] < M // 2                         # 2^(2T) <= 2^L < M/2


def test_crt_bruteforce_small_M(oracle):
    # N = 2: M = 65280; every x in [-M/2, M/2) is the unique value with its residues
    M = 256 * 255
    for x in range(-M // 2, M // 2, 7):
        assert oracle.crt_scalar(2, [x % 256, x % 255]) == x
    # Eq. (1) tie: S == M/2 (mod M) maps to -M/2
    assert oracle.crt_scalar(2, [(M // 2) % 256, (M // 2) % 255]) == -M // 2


@pytest.mark.parametrize("N", [3, 8, 14, 16, 17, 20])
def test_crt_roundtrip_random(oracle, N):
    mods = oracle.constants(N)["moduli"]
    M = math.prod(mods)
    rng = random.Random(N)
    for _ in range(300):
        x = rng.randrange(-(M // 2) + 1, M // 2)
        # any congruent representatives work (unreduced, shifted by multiples)
        c = [x % m + m * rng.randrange(-3, 4) for m in mods]
        assert oracle.crt_scalar(N, c) == x


def test_eq17_budget(oracle):
    for N in (2, 8, 14, 16, 20):
        M = math.prod(oracle.constants(N)["moduli"])
        for q in (1, 2, 1024, 4096, 16384, 65536):
            k = oracle.eq17_k(N, q)
            if k >= 0:
                assert q * 4 ** k <= M // 2 - 1 < q * 4 ** (k + 1)
    assert oracle.eq17_k(2, 1024) == 2
    # "For s = 16, k = 53 is expected" (reading R11: >= 53)
    for q in (1024, 4096, 16384):
        assert oracle.eq17_k(16, q) >= 53
    assert [oracle.eq17_k(16, q) for q in (1024, 4096, 16384)] == [57, 56, 55]
