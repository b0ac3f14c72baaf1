/*
 * oz2_fp64_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * The FP64 prime-modulus regime of Ozaki scheme II (Sec. 3.2,
 * Eqs. 19-21), plainly and exactly on the CPU: the residue products run in
 * binary64 on the GPU path, here in int64 (exact); every other step uses
 * WL = 10 limb (640-bit) integers, so A', the CRT sum S and M (up to 2^484 at
 * s = 22 primes of 22 bits) are held exactly.  Only tests/ may load it; it
 * shares no code with the CUDA path (paper_2504_08009_b200/).
 *
 * Readings (F1-F4):
 *  F1  moduli: the s largest primes below 2^b, b = floor((55 - ceil(log2 q))/2),
 *      so that q m^2 <= 2^55 = 4 u^-1 (Eq. 19).  For q = 1024 this is b = 22 and
 *      reproduces Eq. (21) verbatim ("m_1 ~ 2^22 <= sqrt(2^45)").
 *  F2  line 1: the OS II-fast rule (reading R4) with T = floor(L/2), L =
 *      floor(log2(M/2 - 1)) of this M ("k_A + k_B is obtained as in (easy_k)",
 *      PAPER.md:525, with the Cauchy-Schwarz form of the INT8 path).
 *  F3  output: X 2^-(e+f) as v unevaluated binary64 words, most significant
 *      first, each the nearest binary64 to the remaining integer (Eq. 22-23's
 *      multi-word format): w_1 = RN(X), w_2 = RN(X - w_1), ... then scaled.
 *  F4  s in [2, 22] (T <= 241 < 256 keeps A' in the 256-bit path of the
 *      residue code; M < 2^484 fits the 640-bit integers with room for S).
 *  F6  double-word inputs A = A1 + A2 with |A2| <= u |A1| (Eqs. 22-23): line 1
 *      on |A1| + |A2| rounded up; x' = trunc(2^e (a1 + a2)) exactly
 *      (scaled_trunc_mw).
 *
 * Build: compiled with oz2_oracle.c into liboz2_oracle.so (oracle/__init__.py).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>
#include <limits.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define WL 10
#define OZ2O_KC 256
#define OZ2O_EXP_NONFINITE INT32_MIN
#include "oz2_wide.h"
#include "oz2_fast_rule.h"

#define OZ2F_OK 0
#define OZ2F_ERR_ARG 1
#define OZ2F_ERR_NUM_MODULI 2
#define OZ2F_MAX_S 22

/* trial division: plainly the definition of a prime */
static int is_prime(int64_t v) {
    if (v < 2) return 0;
    for (int64_t d = 2; d * d <= v; d++)
        if (v % d == 0) return 0;
    return 1;
}

/* F1: b = floor((55 - ceil(log2 q)) / 2) */
int oz2f_prime_bits(int64_t q) {
    int lq = 0;
    while (((int64_t)1 << lq) < q) lq++;
    return (55 - lq) / 2;
}

/* Eq. (19)-(21), reading F1: the s largest primes below 2^b, descending */
int oz2f_moduli(int s, int64_t q, int64_t* m) {
    if (s < 1 || s > 64 || q < 1) return OZ2F_ERR_ARG;
    int b = oz2f_prime_bits(q);
    int64_t v = ((int64_t)1 << b) - 1;
    for (int t = 0; t < s; v--) {
        if (v < 2) return OZ2F_ERR_ARG;
        if (is_prime(v)) m[t++] = v;
    }
    return OZ2F_OK;
}

typedef struct {
    int s;
    int64_t m[OZ2F_MAX_S];
    int64_t y[OZ2F_MAX_S];
    wide_t M;
    wide_t w[OZ2F_MAX_S];
    int L, T;
} fconsts_t;

static int64_t mod_i64(int64_t a, int64_t m) { int64_t r = a % m; return r < 0 ? r + m : r; }

static int make_fconsts(int s, int64_t q, fconsts_t* c) {
    if (s < 2 || s > OZ2F_MAX_S) return OZ2F_ERR_NUM_MODULI;
    c->s = s;
    if (oz2f_moduli(s, q, c->m)) return OZ2F_ERR_ARG;
    /* Eq. (7): M = prod m_t */
    wide_t M = w_from_i64(1);
    for (int t = 0; t < s; t++) M = w_mul(M, w_from_i64(c->m[t]));
    c->M = M;
    for (int t = 0; t < s; t++) {
        /* M_t = M / m_t, y_t = M_t^-1 mod m_t (least positive, R2),
         * found by the extended Euclidean algorithm on (M_t mod m_t, m_t)       */
        wide_t Mt, rem;
        w_udivmod(M, w_from_i64(c->m[t]), &Mt, &rem);
        wide_t qq, r; w_udivmod(Mt, w_from_i64(c->m[t]), &qq, &r);
        int64_t a = (int64_t)r.l[0], mm = c->m[t];
        int64_t old_r = a, rr = mm, old_s = 1, ss = 0;
        while (rr) {
            int64_t quo = old_r / rr, tmp;
            tmp = old_r - quo * rr; old_r = rr; rr = tmp;
            tmp = old_s - quo * ss; old_s = ss; ss = tmp;
        }
        if (old_r != 1) return OZ2F_ERR_ARG;           /* not coprime: cannot happen */
        c->y[t] = mod_i64(old_s, mm);
        c->w[t] = w_mul(Mt, w_from_i64(c->y[t]));      /* Alg. 1 line 8: M y_t / m_t */
    }
    /* L = floor(log2(M/2 - 1)) as in Eq. (16); M is odd here, so
     * M/2 - 1 = (M - 2)/2 is a half-integer and floor(log2((M - 2)/2)) =
     * bitlen(floor(M/2) - 1) - 1.  T = floor(L/2) (F2).                         */
    wide_t half_minus_1 = w_sub(w_shr(M, 1), w_from_i64(1));
    c->L = w_bitlen(half_minus_1) - 1;
    c->T = c->L / 2;
    return OZ2F_OK;
}

/* constants for tests: moduli, y, M and w_t as WL limbs, L, T */
int oz2f_constants(int s, int64_t q, int64_t* moduli, int64_t* y, uint64_t* M_limbs, uint64_t* w_limbs,
                   int32_t* L, int32_t* T) {
    fconsts_t c; int rc = make_fconsts(s, q, &c); if (rc) return rc;
    for (int t = 0; t < s; t++) {
        if (moduli) moduli[t] = c.m[t];
        if (y) y[t] = c.y[t];
        if (w_limbs) for (int i = 0; i < WL; i++) w_limbs[t * WL + i] = c.w[t].l[i];
    }
    if (M_limbs) for (int i = 0; i < WL; i++) M_limbs[i] = c.M.l[i];
    if (L) *L = c.L;
    if (T) *T = c.T;
    return OZ2F_OK;
}

/* Alg. 1 lines 7-10 for one element in this regime:
 *   line 7:  c''_t = c'_t mod m_t in [0, m_t)
 *   line 8:  S = sum_t c''_t w_t              (exact)
 *   line 9:  X = S mod M                      (Eq. 1)
 *   line 10 + F3: v words of 2^-(e+f) X                                       */
static void crt_words(const fconsts_t* c, const int64_t* cp, int32_t e, int32_t f, int v, double* out,
                      int64_t ostride, wide_t* Xo) {
    wide_t S = w_from_i64(0);
    for (int t = 0; t < c->s; t++) S = w_add(S, w_mul(w_from_i64(mod_i64(cp[t], c->m[t])), c->w[t]));
    wide_t X = w_smod(S, c->M);
    if (Xo) *Xo = X;
    if (e == OZ2O_EXP_NONFINITE || f == OZ2O_EXP_NONFINITE) {
        for (int i = 0; i < v; i++) out[i * ostride] = NAN;
        return;
    }
    wide_t R = X;
    for (int i = 0; i < v; i++) {
        double w = w_to_double_rn(R);                  /* nearest binary64 to the remainder */
        out[i * ostride] = ldexp(w, -(e + f));
        R = w_sub(R, w_from_double(w));                /* exact: w is an integer here */
    }
}

/* |a1| + |a2| rounded upward (an upper bound of |a1 + a2|): TwoSum, then one
 * step up when the rounded sum fell below the exact one                       */
static double abs_sum_up(double a1, double a2) {
    const double x = fabs(a1), y = fabs(a2);
    const double s = x + y, bb = s - x, err = (x - (s - bb)) + (y - bb);
    return err > 0 ? nextafter(s, INFINITY) : s;
}

/* Reading F6 (multi-word inputs, Eqs. 22-23): x' = trunc(2^e (x1 + x2)) exactly,
 * for |x2| <= u |x1| (so the sum has the sign of x1).  Plainly: if |2^e x1| < 1
 * the truncation is 0; otherwise 2^e x1 has no bits below 2^-52, and
 * X = 2^128 (2^e x1) + R(2^128 2^e x2) is an exact integer with R = floor for
 * x1 > 0 and ceil for x1 < 0 -- rounding x2 on the 2^-128 grid toward the side
 * that keeps floor (resp. ceil) of the sum -- and x' = trunc(X / 2^128).  A
 * scaled second word of magnitude below 2^-64 (or underflowing) acts only
 * through its sign and is taken as +-2^-64.                                    */
static wide_t scaled_trunc_mw(double a1, double a2, int e) {
    const double x1 = ldexp(a1, e);
    if (fabs(x1) < 1.0) return w_from_i64(0);
    double x2 = ldexp(a2, e);
    if (a2 != 0.0 && fabs(x2) < 0x1p-64) x2 = copysign(0x1p-64, a2);
    const double g = ldexp(x2, 128);
    const double gr = x1 > 0 ? floor(g) : ceil(g);
    const wide_t X = w_add(w_from_double(ldexp(x1, 128)), w_from_double(gr));
    return w_is_neg(X) ? w_neg(w_shr(w_neg(X), 128)) : w_shr(X, 128);
}

/* The whole product in the FP64 prime regime: C (v words [v][m][n], word plane
 * stride m*ldc) ~= A B, A m x k (lda), B k x n (ldb), row-major, s primes for
 * q = k.  A2 / B2 (NULL or the second words of double-word inputs, same
 * layout, reading F6).  e_out / f_out optional.                               */
int oz2f_dgemm_mw(int64_t m, int64_t n, int64_t k, const double* A, const double* A2, int64_t lda,
                  const double* B, const double* B2, int64_t ldb, int s, int v, double* C, int64_t ldc,
                  int32_t* e_out, int32_t* f_out) {
    if (m < 0 || n < 0 || k < 1 || v < 1 || v > 4) return OZ2F_ERR_ARG;
    fconsts_t c; int rc = make_fconsts(s, k, &c); if (rc) return rc;
    int32_t* e = (int32_t*)malloc(sizeof(int32_t) * (m ? m : 1));
    int32_t* f = (int32_t*)malloc(sizeof(int32_t) * (n ? n : 1));
    /* line 1 (F2, F6): OS II-fast with this regime's T, on |x1| + |x2| rounded up */
    double* Ab = (double*)malloc(sizeof(double) * (size_t)(m * k ? m * k : 1));
    double* Bb = (double*)malloc(sizeof(double) * (size_t)(n * k ? n * k : 1));
    for (int64_t i = 0; i < m; i++)
        for (int64_t l = 0; l < k; l++)
            Ab[i * k + l] = A2 ? abs_sum_up(A[i * lda + l], A2[i * lda + l]) : A[i * lda + l];
    for (int64_t l = 0; l < k; l++)
        for (int64_t j = 0; j < n; j++)
            Bb[l * n + j] = B2 ? abs_sum_up(B[l * ldb + j], B2[l * ldb + j]) : B[l * ldb + j];
    #pragma omp parallel for schedule(dynamic, 16)
    for (int64_t i = 0; i < m; i++) e[i] = fast_exponent_one(k, Ab + i * k, 1, c.T);
    #pragma omp parallel for schedule(dynamic, 16)
    for (int64_t j = 0; j < n; j++) f[j] = fast_exponent_one(k, Bb + j, n, c.T);
    free(Ab); free(Bb);
    /* lines 2-5: A' = trunc(D A), residues A'_t = A' mod m_t (Eq. 1), as int64 */
    int64_t* Ar = (int64_t*)malloc(sizeof(int64_t) * (size_t)s * (size_t)(m * k ? m * k : 1));
    int64_t* Br = (int64_t*)malloc(sizeof(int64_t) * (size_t)s * (size_t)(n * k ? n * k : 1));
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < m; i++)
        for (int64_t l = 0; l < k; l++) {
            wide_t xw;
            if (e[i] == OZ2O_EXP_NONFINITE) xw = w_from_i64(0);
            else if (A2) xw = scaled_trunc_mw(A[i * lda + l], A2[i * lda + l], e[i]);
            else xw = w_from_double(trunc(ldexp(A[i * lda + l], e[i])));
            for (int t = 0; t < s; t++) Ar[((int64_t)t * m + i) * k + l] = (int64_t)w_smod_small(xw, c.m[t]).l[0];
        }
    #pragma omp parallel for schedule(static)
    for (int64_t j = 0; j < n; j++)
        for (int64_t l = 0; l < k; l++) {
            wide_t xw;
            if (f[j] == OZ2O_EXP_NONFINITE) xw = w_from_i64(0);
            else if (B2) xw = scaled_trunc_mw(B[l * ldb + j], B2[l * ldb + j], f[j]);
            else xw = w_from_double(trunc(ldexp(B[l * ldb + j], f[j])));
            for (int t = 0; t < s; t++) Br[((int64_t)t * n + j) * k + l] = (int64_t)w_smod_small(xw, c.m[t]).l[0];
        }
    /* line 6: C'_t = A'_t B'_t exactly (int64: |.| <= k (m_t/2)^2 <= 2^53, Eq. 20) */
    #pragma omp parallel for schedule(dynamic, 1)
    for (int64_t i = 0; i < m; i++) {
        int64_t cp[OZ2F_MAX_S];
        double words[4];
        for (int64_t j = 0; j < n; j++) {
            for (int t = 0; t < s; t++) {
                const int64_t* a = Ar + ((int64_t)t * m + i) * k;
                const int64_t* b = Br + ((int64_t)t * n + j) * k;
                int64_t acc = 0;
                for (int64_t l = 0; l < k; l++) acc += a[l] * b[l];
                cp[t] = acc;
            }
            crt_words(&c, cp, e[i], f[j], v, words, 1, NULL);
            for (int w = 0; w < v; w++) C[(int64_t)w * m * ldc + i * ldc + j] = words[w];
        }
    }
    if (e_out) memcpy(e_out, e, sizeof(int32_t) * m);
    if (f_out) memcpy(f_out, f, sizeof(int32_t) * n);
    free(e); free(f); free(Ar); free(Br);
    return OZ2F_OK;
}

int oz2f_dgemm(int64_t m, int64_t n, int64_t k, const double* A, int64_t lda, const double* B, int64_t ldb,
               int s, int v, double* C, int64_t ldc, int32_t* e_out, int32_t* f_out) {
    return oz2f_dgemm_mw(m, n, k, A, NULL, lda, B, NULL, ldb, s, v, C, ldc, e_out, f_out);
}

/* Eq. (8) + line 9 for one element (tests): X = (sum_t c_t w_t) mod M as WL limbs */
int oz2f_crt_scalar(int s, int64_t q, const int64_t* cres, uint64_t* X_limbs) {
    fconsts_t c; int rc = make_fconsts(s, q, &c); if (rc) return rc;
    wide_t S = w_from_i64(0);
    for (int t = 0; t < s; t++) S = w_add(S, w_mul(w_from_i64(mod_i64(cres[t], c.m[t])), c.w[t]));
    wide_t X = w_smod(S, c.M);
    for (int i = 0; i < WL; i++) X_limbs[i] = X.l[i];
    return OZ2F_OK;
}

/* reading F6 for one element (tests): trunc(2^e (a1 + a2)) as WL limbs */
void oz2f_scaled_trunc_mw(double a1, double a2, int e, uint64_t* limbs) {
    const wide_t x = scaled_trunc_mw(a1, a2, e);
    for (int i = 0; i < WL; i++) limbs[i] = x.l[i];
}
