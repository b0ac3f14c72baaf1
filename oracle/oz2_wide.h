/*
 * oz2_wide.h -- TEST INFRASTRUCTURE ONLY (part of the oracle, shared by the
 * oracle's two translation units, never by the CUDA path): fixed-width
 * two's-complement integers of WL 64-bit limbs and the exact operations the
 * oracle needs (add, multiply, shifts, long division, Eq. (1), round-to-nearest
 * conversion to binary64).  Every function is static: each oracle file
 * includes it with its own WL.
 */
#pragma once
#include <stdint.h>
#include <math.h>

/* ------------------------------------------------------------------------- */
/* WL x 64-bit two's-complement integers (WL = 4: 256 bits, the INT8-modulus  */
/* oracle; the FP64-prime-modulus oracle includes this with WL = 10)           */
/* ------------------------------------------------------------------------- */
#ifndef WL
#define WL 4
#endif
typedef struct { uint64_t l[WL]; } wide_t;
typedef unsigned __int128 u128;

static wide_t w_from_i64(int64_t v) {
    wide_t r; r.l[0] = (uint64_t)v;
    for (int i = 1; i < WL; i++) r.l[i] = v < 0 ? ~0ull : 0ull;
    return r;
}
static int w_is_neg(wide_t a) { return (int)(a.l[WL - 1] >> 63); }
static int w_is_zero(wide_t a) { for (int i = 0; i < WL; i++) if (a.l[i]) return 0; return 1; }
static wide_t w_add(wide_t a, wide_t b) {
    wide_t r; u128 c = 0;
    for (int i = 0; i < WL; i++) { c += (u128)a.l[i] + b.l[i]; r.l[i] = (uint64_t)c; c >>= 64; }
    return r;
}
static wide_t w_not(wide_t a) { for (int i = 0; i < WL; i++) a.l[i] = ~a.l[i]; return a; }
static wide_t w_neg(wide_t a) { return w_add(w_not(a), w_from_i64(1)); }
static wide_t w_sub(wide_t a, wide_t b) { return w_add(a, w_neg(b)); }
/* a * b mod 2^256; correct for signed operands when the true product fits */
static wide_t w_mul(wide_t a, wide_t b) {
    uint64_t r[WL] = {0};
    for (int i = 0; i < WL; i++) {
        u128 c = 0;
        for (int j = 0; i + j < WL; j++) {
            c += (u128)a.l[i] * b.l[j] + r[i + j];
            r[i + j] = (uint64_t)c; c >>= 64;
        }
    }
    wide_t o; memcpy(o.l, r, sizeof r); return o;
}
static int w_cmp(wide_t a, wide_t b) {           /* signed comparison */
    int na = w_is_neg(a), nb = w_is_neg(b);
    if (na != nb) return na ? -1 : 1;
    for (int i = WL - 1; i >= 0; i--) if (a.l[i] != b.l[i]) return a.l[i] < b.l[i] ? -1 : 1;
    return 0;
}
static int w_bitlen(wide_t a) {                  /* for a >= 0 */
    for (int i = WL - 1; i >= 0; i--) if (a.l[i]) return 64 * i + 64 - __builtin_clzll(a.l[i]);
    return 0;
}
static wide_t w_shl(wide_t a, int s) {           /* 0 <= s < 256 */
    wide_t r = {{0}}; int q = s / 64, b = s % 64;
    for (int i = WL - 1; i >= q; i--) {
        uint64_t v = a.l[i - q] << b;
        if (b && i - q - 1 >= 0) v |= a.l[i - q - 1] >> (64 - b);
        r.l[i] = v;
    }
    return r;
}
static wide_t w_shr(wide_t a, int s) {           /* logical, for a >= 0 */
    wide_t r = {{0}}; int q = s / 64, b = s % 64;
    for (int i = 0; i + q < WL; i++) {
        uint64_t v = a.l[i + q] >> b;
        if (b && i + q + 1 < WL) v |= a.l[i + q + 1] << (64 - b);
        r.l[i] = v;
    }
    return r;
}
/* schoolbook binary long division of num >= 0 by den > 0 */
static void w_udivmod(wide_t num, wide_t den, wide_t* q, wide_t* r) {
    wide_t qq = w_from_i64(0);
    int sh = w_bitlen(num) - w_bitlen(den);
    for (int s = sh; s >= 0; s--) {
        wide_t d = w_shl(den, s);
        if (w_cmp(num, d) >= 0) { num = w_sub(num, d); qq = w_add(qq, w_shl(w_from_i64(1), s)); }
    }
    *q = qq; *r = num;
}
/* floor(num / den) for any num, den > 0 */
static wide_t w_floordiv(wide_t num, wide_t den) {
    wide_t q, r;
    if (!w_is_neg(num)) { w_udivmod(num, den, &q, &r); return q; }
    w_udivmod(w_neg(num), den, &q, &r);
    q = w_neg(q);
    if (!w_is_zero(r)) q = w_sub(q, w_from_i64(1));
    return q;
}
/* schoolbook short division of num >= 0 by a one-limb den > 0 */
static void w_udivmod_small(wide_t num, uint64_t den, wide_t* q, uint64_t* r) {
    u128 rem = 0;
    for (int i = WL - 1; i >= 0; i--) {
        u128 cur = (rem << 64) | num.l[i];
        q->l[i] = (uint64_t)(cur / den);
        rem = cur % den;
    }
    *r = (uint64_t)rem;
}
/* floor(num / den) for any num and a one-limb den > 0 */
static wide_t w_floordiv_small(wide_t num, uint64_t den) {
    wide_t q; uint64_t r;
    if (!w_is_neg(num)) { w_udivmod_small(num, den, &q, &r); return q; }
    w_udivmod_small(w_neg(num), den, &q, &r);
    q = w_neg(q);
    if (r) q = w_sub(q, w_from_i64(1));
    return q;
}
/* Eq. (1) for a modulus that fits one limb (all m_t): same formula, short division */
static wide_t w_smod_small(wide_t a, int64_t m) {
    wide_t mm = w_from_i64(m);
    wide_t q = w_floordiv_small(w_add(w_add(a, a), mm), (uint64_t)(2 * m));
    return w_sub(a, w_mul(mm, q));
}
/* Eq. (1): r = a - m * floor(a/m + 1/2) = a - m * floor((2a + m) / (2m)) */
static wide_t w_smod(wide_t a, wide_t m) {
    wide_t two_a_plus_m = w_add(w_add(a, a), m);
    wide_t q = w_floordiv(two_a_plus_m, w_add(m, m));
    return w_sub(a, w_mul(m, q));
}
/* the integer value of an integral binary64 x, exactly */
static wide_t w_from_double(double x) {
    if (x == 0.0) return w_from_i64(0);
    int ex; double f = frexp(fabs(x), &ex);       /* |x| = f * 2^ex, f in [0.5, 1) */
    uint64_t mant = (uint64_t)ldexp(f, 53);         /* exact 53-bit integer        */
    int sh = ex - 53;
    wide_t r = w_from_i64((int64_t)mant);
    if (sh >= 0) r = w_shl(r, sh); else r = w_shr(r, -sh);   /* x integral: no bits lost */
    return x < 0 ? w_neg(r) : r;
}
/* round-to-nearest-even conversion to binary64 (Alg. 1 caption) */
static double w_to_double_rn(wide_t a) {
    int neg = w_is_neg(a);
    wide_t mag = neg ? w_neg(a) : a;
    int bl = w_bitlen(mag);
    double v;
    if (bl <= 53) {
        v = (double)mag.l[0];                          /* exact */
    } else {
        int drop = bl - 53;
        wide_t q = w_shr(mag, drop);
        wide_t rem = w_sub(mag, w_shl(q, drop));
        wide_t half = w_shl(w_from_i64(1), drop - 1);
        int c = w_cmp(rem, half);
        uint64_t qi = q.l[0];
        if (c > 0 || (c == 0 && (qi & 1))) qi += 1;  /* ties to even */
        v = ldexp((double)qi, drop);                   /* qi <= 2^53: exact */
    }
    return neg ? -v : v;
}

