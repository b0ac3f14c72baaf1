/*
 * oz2_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously-correct CPU implementation of Ozaki scheme II with
 * INT8 moduli (Ozaki, Uchino, Imamura, arXiv 2504.08009), written from PAPER.md.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
 * leg may load this library.  The product path (paper_2504_08009_b200/) never
 * links, imports or calls it, and this file shares no code with it.
 *
 * Every function cites the PAPER.md passage it follows.  Integer work uses a
 * fixed 256-bit two's-complement integer ("wide_t") so that A', the CRT sum
 * and M are held exactly (log2 M = 155.4 at N = 20).  Floating point is only
 * used where the paper's definition is a floating-point operation (ldexp,
 * trunc, the final round-to-nearest conversion).
 *
 * Readings of points where the paper is silent are labelled R1..R13 and are
 * listed in DESIGN.md section "Readings".  Parity status: every stage below
 * is pinned by tests/test_oracle_*.py (no "parity unpinned" functions).
 *
 * Build: gcc -O2 -fopenmp -ffp-contract=off -fPIC -shared (see oracle/build.py)
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>
#include <limits.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define OZ2O_OK 0
#define OZ2O_ERR_ARG 1
#define OZ2O_ERR_NUM_MODULI 2
#define OZ2O_ERR_K_TOO_LARGE 3
#define OZ2O_ERR_BUDGET 4
#define OZ2O_ERR_OVERFLOW 5

/* exponent sentinel for a row/column holding Inf or NaN (reading R13) */
#define OZ2O_EXP_NONFINITE INT32_MIN

#define OZ2O_MODE_FAST 0
#define OZ2O_MODE_EQ17 1
#define OZ2O_MODE_ACCU 2

/* R4/R5: chunk length of the FAST (Cauchy-Schwarz) rule */
#define OZ2O_KC 256
#define OZ2O_MAX_N 20

#include "oz2_wide.h"

/* ------------------------------------------------------------------------- */
/* Constants: moduli, M, M_t, y_t, w_t = M_t y_t, L, T                          */
/* ------------------------------------------------------------------------- */
/* Eq. (18), used verbatim for N <= 16 ("stored in a table for
 * s = 2, 3, ...").  Reading R1: for N = 17..20 append 241, 181,
 * 179, 173, the largest remaining values <= 256 coprime to all earlier ones. */
static const int32_t T20[20] = {256, 255, 253, 251, 247, 239, 233, 229, 227, 223,
                                217, 211, 199, 197, 193, 191, 241, 181, 179, 173};

typedef struct {
    int N;
    int32_t m[20];
    int32_t y[20];
    wide_t M;
    wide_t w[20];
    int L, T;
} consts_t;

static int make_consts(int N, consts_t* c) {
    if (N < 2 || N > 20) return OZ2O_ERR_NUM_MODULI;
    c->N = N;
    /* Eq. (7): M = prod m_i */
    wide_t M = w_from_i64(1);
    for (int t = 0; t < N; t++) { c->m[t] = T20[t]; M = w_mul(M, w_from_i64(T20[t])); }
    c->M = M;
    for (int t = 0; t < N; t++) {
        /* M_t = M / m_t, y_t with M_t y_t == 1 (mod m_t).
         * Reading R2: the least positive representative, found by search.   */
        wide_t mt = w_from_i64(c->m[t]), Mt, rem;
        w_udivmod(M, mt, &Mt, &rem);
        wide_t q, r; w_udivmod(Mt, mt, &q, &r);
        int64_t Mt_mod = (int64_t)r.l[0];
        int y = 0;
        for (int cand = 1; cand < c->m[t]; cand++)
            if ((Mt_mod * cand) % c->m[t] == 1) { y = cand; break; }
        if (!y) return OZ2O_ERR_ARG;                   /* not coprime: cannot happen */
        c->y[t] = y;
        c->w[t] = w_mul(Mt, w_from_i64(y));            /* Alg. 1 line 8: M y_t / m_t */
    }
    /* Eq. (16)-(17) with q dropped: L = floor(log2(M/2 - 1)), T = floor(L/2)
     * (reading R3: k_A = k_B).  M is even (m_1 = 256).      */
    wide_t half_minus_1 = w_sub(w_shr(M, 1), w_from_i64(1));
    c->L = w_bitlen(half_minus_1) - 1;
    c->T = c->L / 2;
    return OZ2O_OK;
}

/* ------------------------------------------------------------------------- */
/* Exported: constants                                                          */
/* ------------------------------------------------------------------------- */
int oz2o_constants(int N, int32_t* moduli, int32_t* y, uint64_t* M_limbs4,
                   uint64_t* w_limbs, int32_t* L, int32_t* T) {
    consts_t c; int rc = make_consts(N, &c); if (rc) return rc;
    for (int t = 0; t < N; t++) {
        if (moduli) moduli[t] = c.m[t];
        if (y) y[t] = c.y[t];
        if (w_limbs) for (int i = 0; i < WL; i++) w_limbs[t * WL + i] = c.w[t].l[i];
    }
    if (M_limbs4) for (int i = 0; i < WL; i++) M_limbs4[i] = c.M.l[i];
    if (L) *L = c.L;
    if (T) *T = c.T;
    return OZ2O_OK;
}

/* Eq. (1) on int64 inputs (for brute-force tests) */
int64_t oz2o_smod_i64(int64_t a, int64_t m) {
    wide_t r = w_smod_small(w_from_i64(a), m);
    return (int64_t)r.l[0];
}
/* the same through the general (long-division) path, used for the CRT */
int64_t oz2o_smod_i64_long(int64_t a, int64_t m) {
    wide_t r = w_smod(w_from_i64(a), w_from_i64(m));
    return (int64_t)r.l[0];
}

/* Eq. (8), PAPER.md:312-316 + Alg. 1 line 9: X = (sum_t c_t w_t) mod M (Eq. 1)
 * for one element; c_t are any integers congruent to the residues.           */
int oz2o_crt_scalar(int N, const int64_t* c, uint64_t* X_limbs4) {
    consts_t k; int rc = make_consts(N, &k); if (rc) return rc;
    wide_t S = w_from_i64(0);
    for (int t = 0; t < N; t++) S = w_add(S, w_mul(w_from_i64(c[t]), k.w[t]));
    wide_t X = w_smod(S, k.M);
    for (int i = 0; i < WL; i++) X_limbs4[i] = X.l[i];
    return OZ2O_OK;
}

/* Eq. (17), in exact integer form (used by mode EQ17):
 * k* = max{ kappa >= 0 : q * 4^kappa <= M/2 - 1 }, or -1 if none.             */
int oz2o_eq17_k(int N, int64_t q) {
    consts_t c; if (make_consts(N, &c)) return -2;
    if (q < 1) q = 1;
    wide_t lim = w_sub(w_shr(c.M, 1), w_from_i64(1));
    int k = -1;
    for (int kap = 0; kap < 200; kap++) {
        wide_t v = w_shl(w_from_i64(q), 2 * kap);
        if (w_cmp(v, lim) <= 0) k = kap; else break;
    }
    return k;
}

/* ------------------------------------------------------------------------- */
/* Part 1 / Alg. 1 line 1: the shift values (exponent vectors e, f)            */
/* ------------------------------------------------------------------------- */
/* x(r, l) = X[r * s_row + l * s_col]: rows of A use (lda, 1), columns of B use (1, ldb). */

#include "oz2_fast_rule.h"

int oz2o_scale_fast(int64_t rows, int64_t len, const double* X, int64_t s_row,
                    int64_t s_col, int N, int32_t* e) {
    consts_t c; int rc = make_consts(N, &c); if (rc) return rc;
    #pragma omp parallel for schedule(dynamic, 16)
    for (int64_t r = 0; r < rows; r++)
        e[r] = fast_exponent_one(len, X + r * s_row, s_col, c.T);
    return OZ2O_OK;
}

/* Mode EQ17 (Eqs. 15-17): k* from oz2o_eq17_k with q = the
 * inner dimension; reading R5: e = k* - 1 - ilogb(max|x|), so every scaled
 * entry has |2^e x| < 2^k*  ("a in Z_k means |a| <= 2^k").      */
int oz2o_scale_eq17(int64_t rows, int64_t len, const double* X, int64_t s_row,
                    int64_t s_col, int N, int64_t q, int32_t* e) {
    int ks = oz2o_eq17_k(N, q);
    if (ks == -2) return OZ2O_ERR_NUM_MODULI;
    if (ks < 1) return OZ2O_ERR_BUDGET;
    #pragma omp parallel for schedule(dynamic, 16)
    for (int64_t r = 0; r < rows; r++) {
        int Emax = INT_MIN, bad = 0;
        for (int64_t l = 0; l < len; l++) {
            double x = X[r * s_row + l * s_col];
            if (!isfinite(x)) { bad = 1; break; }
            if (x != 0.0) { int ex = ilogb(x); if (ex > Emax) Emax = ex; }
        }
        e[r] = bad ? OZ2O_EXP_NONFINITE : (Emax == INT_MIN ? 0 : ks - 1 - Emax);
    }
    return OZ2O_OK;
}

/* Mode ACCU (OS II-accu: "employing cublasGemmEx with CUDA_R_8I
 * for the line 1 to satisfy the condition (13)"; "low-precision
 * computation", 637-640).  Reading R18, step by step:
 *   1. E_i = ilogb(max_l |a_il|), F_j = ilogb(max_l |b_lj|)  (rows/cols of zeros: none);
 *   2. 7-bit upper approximations  ahat_il = ceil(|a_il| 2^(6 - E_i)) in [0, 128],
 *      bhat_lj = ceil(|b_lj| 2^(6 - F_j)), so |a_il| <= ahat_il 2^(E_i - 6);
 *   3. P = Ahat Bhat, the INT8 GEMM of the line-1 bound (unsigned, exact in int32
 *      for k < 2^17):  (|A||B|)_ij <= P_ij 2^(E_i + F_j - 12);
 *   4. with lambda(x) = ceil(log2 x):  g_i = min(G, floor((L + 12 - lambda(max_j P_ij)) / 2)),
 *      h_j = min(G, floor((L + 12 - lambda(max_i P_ij)) / 2))  (G where the maximum
 *      is 0);  e_i = g_i - E_i,  f_j = h_j - F_j.  G = 61 (N <= 16) or 93 (N > 16)
 *      keeps |a'| < 2^(g + 1) within 62 / 94 bits, the integer width of FAST's
 *      largest |a'| (2^T, T = 62 at N = 16, 77 at N = 20) rounded to whole words.
 * Then (|A'||B'|)_ij <= 2^(g_i + h_j - 12) P_ij <= 2^L < M/2 (condition (13)).
 * A zero row / column gets 0; one holding Inf / NaN the sentinel (R13).         */
static int ilogb_max(int64_t len, const double* X, int64_t s_col, int* bad) {
    int E = INT_MIN;
    *bad = 0;
    for (int64_t l = 0; l < len; l++) {
        double x = X[l * s_col];
        if (!isfinite(x)) { *bad = 1; return INT_MIN; }
        if (x != 0.0) { int ex = ilogb(x); if (ex > E) E = ex; }
    }
    return E;
}
static uint8_t hat7(double x, int E) {                   /* ceil(|x| 2^(6 - E)) */
    if (x == 0.0 || E == INT_MIN) return 0;
    /* exact whenever the result is >= 1 (values < 1 become 1); 2^(6-E) itself
     * overflows for E < -1017, hence two steps there                           */
    double v = 6 - E > 1000 ? ceil(ldexp(ldexp(fabs(x), 1000), 6 - E - 1000)) : ceil(ldexp(fabs(x), 6 - E));
    return (uint8_t)(v < 1.0 ? 1.0 : v);
}
static int lambda_ceil_log2(uint64_t x) {                /* ceil(log2 x), x >= 1 */
    int l = 0;
    while (l < 64 && (1ull << l) < x) l++;
    return l;
}
static int floor_half(int v) { return v >= 0 ? v / 2 : -((-v + 1) / 2); }

int oz2o_scale_accu(int64_t m, int64_t n, int64_t k, const double* A, int64_t lda, const double* B,
                    int64_t ldb, int N, int32_t* e, int32_t* f, uint32_t* P_rowmax, uint32_t* P_colmax) {
    consts_t c; int rc = make_consts(N, &c); if (rc) return rc;
    if (k >= (1 << 17)) return OZ2O_ERR_K_TOO_LARGE;     /* the bound GEMM is exact in int32 */
    int* E = (int*)malloc(sizeof(int) * (m ? m : 1));
    int* F = (int*)malloc(sizeof(int) * (n ? n : 1));
    int* badA = (int*)malloc(sizeof(int) * (m ? m : 1));
    int* badB = (int*)malloc(sizeof(int) * (n ? n : 1));
    uint8_t* Ah = (uint8_t*)malloc((size_t)(m * k > 0 ? m * k : 1));
    uint8_t* Bh = (uint8_t*)malloc((size_t)(n * k > 0 ? n * k : 1));   /* Bhat^T: n x k */
    uint32_t* rmax = (uint32_t*)calloc((size_t)(m ? m : 1), sizeof(uint32_t));
    uint32_t* cmax = (uint32_t*)calloc((size_t)(n ? n : 1), sizeof(uint32_t));
    for (int64_t i = 0; i < m; i++) {                    /* steps 1-2, rows of A */
        E[i] = ilogb_max(k, A + i * lda, 1, &badA[i]);
        for (int64_t l = 0; l < k; l++) Ah[i * k + l] = badA[i] ? 0 : hat7(A[i * lda + l], E[i]);
    }
    for (int64_t j = 0; j < n; j++) {                    /* steps 1-2, columns of B */
        F[j] = ilogb_max(k, B + j, ldb, &badB[j]);
        for (int64_t l = 0; l < k; l++) Bh[j * k + l] = badB[j] ? 0 : hat7(B[l * ldb + j], F[j]);
    }
    #pragma omp parallel for schedule(dynamic, 4)
    for (int64_t i = 0; i < m; i++)                      /* step 3 */
        for (int64_t j = 0; j < n; j++) {
            uint64_t p = 0;
            for (int64_t l = 0; l < k; l++) p += (uint64_t)Ah[i * k + l] * Bh[j * k + l];
            if (p > rmax[i]) rmax[i] = (uint32_t)p;
            #pragma omp critical
            { if (p > cmax[j]) cmax[j] = (uint32_t)p; }
        }
    const int G = N <= 16 ? 61 : 93;
    for (int64_t i = 0; i < m; i++) {                    /* step 4 */
        int g = rmax[i] ? floor_half(c.L + 12 - lambda_ceil_log2(rmax[i])) : G;
        if (g > G) g = G;
        e[i] = badA[i] ? OZ2O_EXP_NONFINITE : (E[i] == INT_MIN ? 0 : g - E[i]);
        if (P_rowmax) P_rowmax[i] = rmax[i];
    }
    for (int64_t j = 0; j < n; j++) {
        int h = cmax[j] ? floor_half(c.L + 12 - lambda_ceil_log2(cmax[j])) : G;
        if (h > G) h = G;
        f[j] = badB[j] ? OZ2O_EXP_NONFINITE : (F[j] == INT_MIN ? 0 : h - F[j]);
        if (P_colmax) P_colmax[j] = cmax[j];
    }
    free(E); free(F); free(badA); free(badB); free(Ah); free(Bh); free(rmax); free(cmax);
    return OZ2O_OK;
}

/* Alg. 1 lines 2-3: x' = trunc(2^e x), an FP64 integer.
 * Out is rows x len, row-major.  Non-finite rows give 0 (R13).                */
void oz2o_trunc_scale(int64_t rows, int64_t len, const double* X, int64_t s_row,
                      int64_t s_col, const int32_t* e, double* out) {
    #pragma omp parallel for schedule(static)
    for (int64_t r = 0; r < rows; r++)
        for (int64_t l = 0; l < len; l++)
            out[r * len + l] = e[r] == OZ2O_EXP_NONFINITE ? 0.0
                             : trunc(ldexp(X[r * s_row + l * s_col], e[r]));
}

/* Eq. (11), Alg. 1 lines 4-5: residue planes
 * out[t][r][l] = x'(r,l) mod m_t (Eq. 1), in [-m_t/2, m_t/2) -> int8.
 * For m_t = 256 the tie 128 gives -128.                    */
int oz2o_residues(int64_t rows, int64_t len, const double* Xp, int N, int8_t* out) {
    consts_t c; int rc = make_consts(N, &c); if (rc) return rc;
    #pragma omp parallel for schedule(static)
    for (int64_t r = 0; r < rows; r++)
        for (int64_t l = 0; l < len; l++) {
            wide_t x = w_from_double(Xp[r * len + l]);
            for (int t = 0; t < N; t++) {
                wide_t res = w_smod_small(x, c.m[t]);
                out[((int64_t)t * rows + r) * len + l] = (int8_t)(int64_t)res.l[0];
            }
        }
    return OZ2O_OK;
}

/* Alg. 1 line 6: C'_t = A'_t B'_t exactly.  Ar is [N][m][k],
 * Br is [N][n][k] (B'_t stored transposed), Cp is [N][m][n].  Sums are formed
 * in int32 over blocks of 2^16 terms (each block |sum| <= 2^16 * 2^14 < 2^31,
 * exact) and the blocks are added in int64; a result outside int32 is an
 * error (exact in INT32 for q < 2^17).                      */
int oz2o_modmul(int64_t m, int64_t n, int64_t k, const int8_t* Ar, const int8_t* Br,
                int N, int32_t* Cp) {
    int bad = 0;
    #pragma omp parallel for collapse(2) schedule(dynamic, 4) reduction(|:bad)
    for (int t = 0; t < N; t++)
        for (int64_t i = 0; i < m; i++) {
            const int8_t* a = Ar + ((int64_t)t * m + i) * k;
            for (int64_t j = 0; j < n; j++) {
                const int8_t* b = Br + ((int64_t)t * n + j) * k;
                int64_t acc = 0;
                for (int64_t l0 = 0; l0 < k; l0 += 65536) {
                    int64_t l1 = l0 + 65536 < k ? l0 + 65536 : k;
                    int32_t blk = 0;
                    for (int64_t l = l0; l < l1; l++) blk += (int32_t)a[l] * (int32_t)b[l];
                    acc += blk;
                }
                if (acc > INT32_MAX || acc < INT32_MIN) bad = 1;
                Cp[((int64_t)t * m + i) * n + j] = (int32_t)acc;
            }
        }
    return bad ? OZ2O_ERR_OVERFLOW : OZ2O_OK;
}

/* Alg. 1 lines 7-10 for one element, given the N products c'_t:
 *   line 7:  c''_t = c'_t - floor(c'_t / m_t) m_t       in [0, m_t)
 *   line 8:  S = sum_t c''_t w_t                         (exact)
 *   line 9:  X = S mod M                                 (Eq. 1, symmetric)
 *   line 10: c = 2^(-e-f) RN(X)                          (reading R10)        */
static double crt_one(const consts_t* c, const int64_t* cp, int64_t stride,
                      int32_t e, int32_t f, wide_t* Xo) {
    wide_t S = w_from_i64(0);
    for (int t = 0; t < c->N; t++) {
        int64_t v = cp[t * stride], mt = c->m[t];
        int64_t q = v >= 0 ? v / mt : -((-v + mt - 1) / mt);   /* floor(v / m_t) */
        int64_t cpp = v - q * mt;
        S = w_add(S, w_mul(w_from_i64(cpp), c->w[t]));
    }
    wide_t X = w_smod(S, c->M);
    if (Xo) *Xo = X;
    if (e == OZ2O_EXP_NONFINITE || f == OZ2O_EXP_NONFINITE) return NAN;
    return ldexp(w_to_double_rn(X), -(e + f));
}

/* Cp is [N][m][n]; C is m x n with leading dimension ldc; X_limbs (optional)
 * receives X as [m][n][4] little-endian 64-bit limbs.                          */
int oz2o_crt(int64_t m, int64_t n, int N, const int32_t* Cp, const int32_t* e,
             const int32_t* f, double* C, int64_t ldc, uint64_t* X_limbs) {
    consts_t c; int rc = make_consts(N, &c); if (rc) return rc;
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < m; i++)
        for (int64_t j = 0; j < n; j++) {
            wide_t X;
            int64_t cp[OZ2O_MAX_N];
            for (int t = 0; t < N; t++) cp[t] = Cp[(int64_t)t * m * n + i * n + j];
            C[i * ldc + j] = crt_one(&c, cp, 1, e[i], f[j], &X);
            if (X_limbs) for (int l = 0; l < WL; l++) X_limbs[(i * n + j) * WL + l] = X.l[l];
        }
    return OZ2O_OK;
}

/* Full Algorithm 1: C ~= A B, A m x k (lda), B k x n (ldb),
 * row-major.  The stages are the functions above applied in the paper's order;
 * the per-element work of lines 6-10 is done one output row at a time so that
 * the int32 products of a whole matrix need not be stored.  e_out / f_out
 * (optional) receive the exponent vectors.                                     */
int oz2o_dgemm(int64_t m, int64_t n, int64_t k, const double* A, int64_t lda,
               const double* B, int64_t ldb, double* C, int64_t ldc, int N, int mode,
               int32_t* e_out, int32_t* f_out) {
    consts_t c; int rc = make_consts(N, &c); if (rc) return rc;
    if (m < 0 || n < 0 || k < 0) return OZ2O_ERR_ARG;
    /* q >= 2^17: "apply block matrix multiplication".  The sum of the
     * block products is the same integer C'_t, so it is accumulated here in int64
     * (|C'_t| <= k 2^14 < 2^63) and reduced once (reading R12).                  */
    int32_t* e = (int32_t*)malloc(sizeof(int32_t) * (m ? m : 1));
    int32_t* f = (int32_t*)malloc(sizeof(int32_t) * (n ? n : 1));
    if (mode == OZ2O_MODE_FAST) {
        oz2o_scale_fast(m, k, A, lda, 1, N, e);
        oz2o_scale_fast(n, k, B, 1, ldb, N, f);
    } else if (mode == OZ2O_MODE_ACCU) {
        rc = oz2o_scale_accu(m, n, k, A, lda, B, ldb, N, e, f, NULL, NULL);
        if (rc) { free(e); free(f); return rc; }
    } else {
        rc = oz2o_scale_eq17(m, k, A, lda, 1, N, k, e);
        if (!rc) rc = oz2o_scale_eq17(n, k, B, 1, ldb, N, k, f);
        if (rc) { free(e); free(f); return rc; }
    }
    double* Ap = (double*)malloc(sizeof(double) * (m * k > 0 ? m * k : 1));
    double* Bp = (double*)malloc(sizeof(double) * (n * k > 0 ? n * k : 1));   /* B'^T: n x k */
    oz2o_trunc_scale(m, k, A, lda, 1, e, Ap);
    oz2o_trunc_scale(n, k, B, 1, ldb, f, Bp);
    int8_t* Ar = (int8_t*)malloc((size_t)N * (m * k > 0 ? m * k : 1));
    int8_t* Br = (int8_t*)malloc((size_t)N * (n * k > 0 ? n * k : 1));
    oz2o_residues(m, k, Ap, N, Ar);
    oz2o_residues(n, k, Bp, N, Br);
    free(Ap); free(Bp);
    #pragma omp parallel for schedule(dynamic, 1)
    for (int64_t i = 0; i < m; i++) {
        int64_t* cp = (int64_t*)malloc(sizeof(int64_t) * N);
        for (int64_t j = 0; j < n; j++) {
            for (int t = 0; t < N; t++) {
                const int8_t* a = Ar + ((int64_t)t * m + i) * k;
                const int8_t* b = Br + ((int64_t)t * n + j) * k;
                int64_t acc = 0;                       /* exact */
                for (int64_t l = 0; l < k; l++) acc += (int32_t)a[l] * (int32_t)b[l];
                cp[t] = acc;
            }
            C[i * ldc + j] = crt_one(&c, cp, 1, e[i], f[j], NULL);
        }
        free(cp);
    }
    if (e_out) memcpy(e_out, e, sizeof(int32_t) * m);
    if (f_out) memcpy(f_out, f, sizeof(int32_t) * n);
    free(e); free(f); free(Ar); free(Br);
    return OZ2O_OK;
}

/* ------------------------------------------------------------------------- */
/* Exact reference product (error metrics): Kulisch-style fixed-point sum      */
/* ------------------------------------------------------------------------- */
/* A binary64 product a*b = (ma 2^ea)(mb 2^eb) is a 106-bit integer times 2^(ea+eb),
 * the lsb is at 2^-2252 or above.  The accumulator holds sum(a_l b_l) * 2^BIAS exactly in
 * 32-bit digits stored in int64 cells (carry-save, normalised at the end).     */
#define KBIAS 2304       /* lsb of a product of two subnormals is 2^-2252 */
#define KDIG 146          /* 146 * 32 = 4672 bits: covers 2^-2304 .. 2^2368 */
typedef struct { int64_t d[KDIG]; } kacc_t;

static void kacc_add_product(kacc_t* a, double x, double y) {
    if (x == 0.0 || y == 0.0) return;
    int ex, ey;
    double fx = frexp(fabs(x), &ex), fy = frexp(fabs(y), &ey);
    uint64_t mx = (uint64_t)ldexp(fx, 53), my = (uint64_t)ldexp(fy, 53);
    int sign = (x < 0) != (y < 0) ? -1 : 1;
    u128 p = (u128)mx * my;                          /* < 2^106 */
    int64_t pos = (int64_t)(ex - 53) + (ey - 53) + KBIAS;   /* bit position of p's lsb */
    int64_t dig = pos / 32, sh = pos % 32;
    for (int j = 0; j < 4; j++) {                    /* p = sum_j p_j 2^(32 j) */
        uint64_t pj = (uint64_t)(p >> (32 * j)) & 0xffffffffull;
        uint64_t v = pj << sh;                       /* < 2^63 */
        a->d[dig + j] += sign * (int64_t)(v & 0xffffffffull);
        a->d[dig + j + 1] += sign * (int64_t)(v >> 32);
    }
}
static void kacc_normalise(kacc_t* a) {
    for (int i = 0; i < KDIG - 1; i++) {
        int64_t v = a->d[i];
        int64_t carry = v >> 32;                     /* floor division by 2^32 */
        a->d[i] = v - carry * 4294967296LL;
        a->d[i + 1] += carry;
    }
}
/* round-to-nearest-even of the accumulated value */
static double kacc_to_double(kacc_t a) {
    kacc_normalise(&a);
    int neg = a.d[KDIG - 1] < 0;
    if (neg) {                                       /* negate all digits, renormalise */
        for (int i = 0; i < KDIG; i++) a.d[i] = -a.d[i];
        kacc_normalise(&a);
    }
    int top = -1;
    for (int i = KDIG - 1; i >= 0; i--) if (a.d[i]) { top = i; break; }
    if (top < 0) return 0.0;
    int tb = 63 - __builtin_clzll((uint64_t)a.d[top]);      /* bit within top digit */
    int64_t msb = (int64_t)top * 32 + tb;                   /* absolute bit index */
    int64_t lsb_keep = msb - 52;                            /* keep 53 bits */
    uint64_t q = 0; int round = 0, sticky = 0;
    for (int64_t b = msb; b >= 0; b--) {
        int bit = (int)((a.d[b / 32] >> (b % 32)) & 1);
        if (b >= lsb_keep) q = (q << 1) | (uint64_t)bit;
        else if (b == lsb_keep - 1) round = bit;
        else if (bit) { sticky = 1; break; }
    }
    if (lsb_keep < 0) { q <<= -lsb_keep; lsb_keep = 0; }   /* fewer than 53 bits */
    if (round && (sticky || (q & 1))) q += 1;
    double v = ldexp((double)q, (int)(lsb_keep - KBIAS));
    return neg ? -v : v;
}

/* exact (AB)_ij and (|A||B|)_ij, each rounded once to nearest
 * for the listed (i, j) pairs.                                                  */
void oz2o_exact_entries(int64_t k, const double* A, int64_t lda, const double* B,
                        int64_t ldb, int64_t npairs, const int64_t* ii, const int64_t* jj,
                        double* ab, double* absab) {
    #pragma omp parallel for schedule(dynamic, 4)
    for (int64_t p = 0; p < npairs; p++) {
        kacc_t* s = (kacc_t*)calloc(1, sizeof(kacc_t));
        kacc_t* t = (kacc_t*)calloc(1, sizeof(kacc_t));
        for (int64_t l = 0; l < k; l++) {
            double a = A[ii[p] * lda + l], b = B[l * ldb + jj[p]];
            kacc_add_product(s, a, b);
            kacc_add_product(t, fabs(a), fabs(b));
            if ((l & ((1 << 24) - 1)) == (1 << 24) - 1) { kacc_normalise(s); kacc_normalise(t); }
        }
        if (ab) ab[p] = kacc_to_double(*s);
        if (absab) absab[p] = kacc_to_double(*t);
        free(s); free(t);
    }
}

/* The DGEMM surface around Algorithm 1 (reading R19, BLAS DGEMM semantics):
 * out = RN(alpha c + RN(beta c_old)) with one fused multiply-add; beta == 0
 * means c_old is not read (alpha c, one rounding).                             */
void oz2o_axpby(int64_t n, double alpha, const double* c, double beta, const double* c_old,
                double* out) {
    for (int64_t i = 0; i < n; i++)
        out[i] = beta == 0.0 ? alpha * c[i] : fma(alpha, c[i], beta * c_old[i]);
}

/* wide integer -> RN double, exposed so the conversion can be pinned against
 * an independent correctly-rounded conversion (Python's int -> float).         */
double oz2o_wide_to_double(const uint64_t* limbs4) {
    wide_t a; for (int i = 0; i < WL; i++) a.l[i] = limbs4[i];
    return w_to_double_rn(a);
}
/* integer value of an integral double, as limbs (pinned against Python int()) */
void oz2o_wide_from_double(double x, uint64_t* limbs4) {
    wide_t a = w_from_double(x);
    for (int i = 0; i < WL; i++) limbs4[i] = a.l[i];
}

void oz2o_set_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}
int oz2o_get_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
