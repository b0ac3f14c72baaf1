// tables.cpp -- host construction of the per-N constants (Oz2Table).
//
// Written independently of oracle/ (which uses a fixed 256-bit integer and a
// brute-force inverse search): here a little base-2^32 big natural number and
// the extended Euclidean algorithm.  tests/test_abi.py compares the exported
// tables with the oracle's.
//
//  moduli: Eq. (18), then 241, 181, 179, 173 (reading R1)
//  M = prod m_t (Eq. 7); M_t = M / m_t; y_t = M_t^-1 mod m_t
//  (least positive, reading R2); w_t = M_t y_t (Alg. 1 line 8,
//  "M y_t / m_t", stored in a table).
#include "oz2_tables.h"

#include <math.h>
#include <string.h>

#include <vector>

namespace {

const int32_t kModuli[OZ2_MAX_MODULI] = {256, 255, 253, 251, 247, 239, 233, 229, 227, 223,
                                         217, 211, 199, 197, 193, 191, 241, 181, 179, 173};

// non-negative big integer, little-endian base 2^32
struct Nat {
    std::vector<uint32_t> d;
    explicit Nat(uint64_t v = 0) {
        while (v) { d.push_back((uint32_t)v); v >>= 32; }
    }
    void trim() { while (!d.empty() && d.back() == 0) d.pop_back(); }
    int bits() const {
        if (d.empty()) return 0;
        return 32 * (int)(d.size() - 1) + (32 - __builtin_clz(d.back()));
    }
    bool bit(int i) const {
        size_t w = (size_t)i / 32;
        return w < d.size() && ((d[w] >> (i % 32)) & 1u);
    }
};

Nat mul_small(const Nat& a, uint32_t s) {
    Nat r; uint64_t carry = 0;
    for (uint32_t x : a.d) { uint64_t v = (uint64_t)x * s + carry; r.d.push_back((uint32_t)v); carry = v >> 32; }
    while (carry) { r.d.push_back((uint32_t)carry); carry >>= 32; }
    r.trim(); return r;
}
Nat divmod_small(const Nat& a, uint32_t s, uint32_t* rem) {
    Nat q; q.d.assign(a.d.size(), 0); uint64_t r = 0;
    for (size_t i = a.d.size(); i-- > 0;) { uint64_t cur = (r << 32) | a.d[i]; q.d[i] = (uint32_t)(cur / s); r = cur % s; }
    q.trim(); if (rem) *rem = (uint32_t)r; return q;
}
Nat sub_small(const Nat& a, uint32_t s) {            // a >= s
    Nat r = a; uint64_t borrow = s;
    for (size_t i = 0; i < r.d.size() && borrow; i++) {
        uint64_t v = r.d[i];
        if (v >= borrow) { r.d[i] = (uint32_t)(v - borrow); borrow = 0; }
        else { r.d[i] = (uint32_t)(v + (1ull << 32) - borrow); borrow = 1; }
    }
    r.trim(); return r;
}
Nat shr1(const Nat& a) {
    Nat r = a;
    for (size_t i = 0; i < r.d.size(); i++) r.d[i] = (r.d[i] >> 1) | (i + 1 < r.d.size() ? r.d[i + 1] << 31 : 0);
    r.trim(); return r;
}
int cmp(const Nat& a, const Nat& b) {
    if (a.d.size() != b.d.size()) return a.d.size() < b.d.size() ? -1 : 1;
    for (size_t i = a.d.size(); i-- > 0;) if (a.d[i] != b.d[i]) return a.d[i] < b.d[i] ? -1 : 1;
    return 0;
}
uint64_t bits_at(const Nat& a, int lo, int nbits) {   // bits [lo, lo+nbits), nbits <= 64
    uint64_t v = 0;
    for (int i = 0; i < nbits; i++) if (a.bit(lo + i)) v |= 1ull << i;
    return v;
}
double to_double(const Nat& a) {                      // nearest-ish (only used for 1/M)
    double v = 0;
    for (size_t i = a.d.size(); i-- > 0;) v = v * 4294967296.0 + a.d[i];
    return v;
}
// extended Euclid: inverse of a modulo m (gcd(a, m) = 1), least positive
int64_t inverse_mod(int64_t a, int64_t m) {
    int64_t r0 = m, r1 = ((a % m) + m) % m, s0 = 0, s1 = 1;
    while (r1) { int64_t q = r0 / r1, t = r0 - q * r1; r0 = r1; r1 = t; t = s0 - q * s1; s0 = s1; s1 = t; }
    if (r0 != 1) return -1;
    return ((s0 % m) + m) % m;
}
int64_t pow2_mod(int e, int64_t m) { int64_t r = 1 % m; for (int i = 0; i < e; i++) r = (r * 2) % m; return r; }

Nat product(int N) { Nat M(1); for (int t = 0; t < N; t++) M = mul_small(M, (uint32_t)kModuli[t]); return M; }

}  // namespace

int oz2_build_tables(Oz2Table tabs[OZ2_MAX_MODULI + 1]) {
    memset(tabs, 0, sizeof(Oz2Table) * (OZ2_MAX_MODULI + 1));
    for (int N = 2; N <= OZ2_MAX_MODULI; N++) {
        Oz2Table& T = tabs[N];
        T.N = N;
        Nat M = product(N);
        int Mbits = M.bits();
        T.JB = (Mbits + 7) / 8;
        T.WS = (Mbits + 13 + 31) / 32;                // S < 20 * 255 * M < 2^13 M
        T.WX = (Mbits + 2 + 31) / 32;                 // 3M/2 < 2^(Mbits + 1) fits 32 WX - 1 bits
        Nat half = shr1(M);                            // M is even (m_1 = 256)
        T.L = sub_small(half, 1).bits() - 1;
        T.T = T.L / 2;
        for (int w = 0; w < OZ2_MAX_WORDS; w++) {
            T.M32[w] = (uint32_t)bits_at(M, 32 * w, 32);
            T.Mh32[w] = (uint32_t)bits_at(half, 32 * w, 32);
        }
        T.qscale = (float)((T.WS >= 2 ? ldexp(1.0, 32 * (T.WS - 2)) : 1.0) / to_double(M));
        for (int t = 0; t < N; t++) {
            int64_t m = kModuli[t];
            T.m[t] = (int32_t)m;
            T.magic[t] = (uint32_t)(((1ull << 32) + (uint64_t)m - 1) / (uint64_t)m);
            T.h[t] = (int32_t)((m - 1) / 2);
            T.negm[t] = (uint32_t)(0x100000000ull - (uint64_t)m);
            for (int w = 0; w < 3; w++) {
                uint32_t packed = 0;
                for (int b = 0; b < 4; b++) packed |= (uint32_t)pow2_mod(8 * (4 * w + b), m) << (8 * b);
                T.cw[w][t] = packed;
            }
            T.k16[t] = (uint32_t)pow2_mod(16, m);
            T.k16s[t] = 2 * (int64_t)T.k16[t] > m ? (int32_t)T.k16[t] - (int32_t)m : (int32_t)T.k16[t];
            T.off7[t] = (uint32_t)(m * (((1 << 22) + m - 1) / m));
            T.g32[t] = (uint32_t)((m - pow2_mod(32, m)) % m);
            T.g64[t] = (int32_t)((m - pow2_mod(64, m)) % m);
            T.g96[t] = (int32_t)((m - pow2_mod(96, m)) % m);
            T.G63[t] = (uint32_t)((m - pow2_mod(63, m)) % m);
            T.G95[t] = (uint32_t)((m - pow2_mod(95, m)) % m);
            T.hmagic[t] = (uint64_t)T.h[t] * (uint64_t)T.magic[t];
            T.G63f[t] = 0x4B000000u + T.G63[t];
            T.G95f[t] = 0x4B000000u + T.G95[t];
            T.invm[t] = 1.0f / (float)m;                  // correctly rounded (IEEE division)
            {
                const int64_t k18 = (int64_t)pow2_mod(18, m);
                T.k18s[t] = (int32_t)(2 * k18 > m ? k18 - m : k18);
                T.k18k[t] = (uint32_t)(-8 * (int64_t)T.k18s[t]);
                T.h23f[t] = 8388608.0f + (float)((m - 1) / 2);
            }
            uint32_t rem;
            Nat Mt = divmod_small(M, (uint32_t)m, &rem);
            if (rem) return 1;
            uint32_t Mt_mod;
            divmod_small(Mt, (uint32_t)m, &Mt_mod);
            int64_t y = inverse_mod(Mt_mod, m);
            if (y <= 0) return 2;
            T.y[t] = (int32_t)y;
            Nat w = mul_small(Mt, (uint32_t)y);
            if (w.bits() > Mbits) return 3;
            for (int j = 0; j < OZ2_MAX_BYTES; j++)
                T.Wb[j][t / 4] |= (uint32_t)bits_at(w, 8 * j, 8) << (8 * (t % 4));
            for (int x = 0; x < OZ2_MAX_WORDS; x++) T.w32[t][x] = (uint32_t)bits_at(w, 32 * x, 32);
        }
    }
    return 0;
}

int oz2_host_eq17_k(int N, int64_t q) {
    if (N < 2 || N > OZ2_MAX_MODULI) return -2;
    if (q < 1) q = 1;
    Nat lim = sub_small(shr1(product(N)), 1);
    Nat v((uint64_t)q);
    int k = -1;
    for (int kap = 0; kap < 200; kap++) {
        if (cmp(v, lim) <= 0) k = kap; else break;
        v = mul_small(v, 4);
    }
    return k;
}
