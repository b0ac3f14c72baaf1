/*
 * oz2_fast_rule.h -- TEST INFRASTRUCTURE ONLY (part of the oracle): the OS
 * II-fast line-1 rule (reading R4) for one row / column, given the bound
 * exponent T.  Included by both oracle translation units (the INT8-modulus
 * regime takes T from Eq. (18)'s M, the FP64-prime regime from its own M).
 */
#pragma once
#include <stdint.h>
#include <stdlib.h>
#include <math.h>
#include <limits.h>

#ifndef OZ2O_KC
#define OZ2O_KC 256                     /* R4: chunk length */
#endif
#ifndef OZ2O_EXP_NONFINITE
#define OZ2O_EXP_NONFINITE INT32_MIN    /* R13 */
#endif

/* Mode FAST (OS II-fast: "employing the Cauchy-Schwarz inequality
 * for the line 1 to satisfy the condition (13)").  Reading R4:
 * integer, summation-order-independent bound on the 2-norm of each row:
 *   per chunk c of KC consecutive indices: E_c = max ilogb|x|,
 *     u = max(1, ceil(|x| 2^(15 - E_c))) for x != 0,  S_c = sum u^2 ;
 *   E = max_c E_c,  S = sum_c ceil(S_c / 4^(E - E_c)),  h = min{h : S <= 4^h},
 *   e = T + 15 - E - h   (so ||2^e x||_2 <= 2^T);  e = 0 for a zero row.
 * With ||2^e a_i||, ||2^f b_j|| <= 2^T, Cauchy-Schwarz gives
 * (|A'||B'|)_ij <= 2^(2T) <= 2^L < M/2, i.e. condition (13).                   */
static int32_t fast_exponent_one(int64_t len, const double* X, int64_t s_col, int T) {
    int E = INT_MIN;
    int64_t nch = (len + OZ2O_KC - 1) / OZ2O_KC;
    int* Ec = (int*)malloc(sizeof(int) * (nch ? nch : 1));
    uint64_t* Sc = (uint64_t*)malloc(sizeof(uint64_t) * (nch ? nch : 1));
    for (int64_t c = 0; c < nch; c++) {
        int64_t l0 = c * OZ2O_KC, l1 = l0 + OZ2O_KC < len ? l0 + OZ2O_KC : len;
        int Emax = INT_MIN;
        for (int64_t l = l0; l < l1; l++) {
            double x = X[l * s_col];
            if (!isfinite(x)) { free(Ec); free(Sc); return OZ2O_EXP_NONFINITE; }
            if (x != 0.0) { int ex = ilogb(x); if (ex > Emax) Emax = ex; }
        }
        uint64_t S = 0;
        if (Emax != INT_MIN) {
            for (int64_t l = l0; l < l1; l++) {
                double x = X[l * s_col];
                if (x == 0.0) continue;
                double v = ceil(ldexp(fabs(x), 15 - Emax));
                uint64_t u = v < 1.0 ? 1 : (uint64_t)v;   /* u in [1, 2^16] */
                S += u * u;
            }
        }
        Ec[c] = Emax; Sc[c] = S;
        if (Emax > E) E = Emax;
    }
    int32_t e;
    if (E == INT_MIN) {
        e = 0;                                            /* zero row (R4) */
    } else {
        uint64_t S = 0;
        for (int64_t c = 0; c < nch; c++) {
            if (Sc[c] == 0) continue;
            int64_t sh = 2 * (int64_t)(E - Ec[c]);
            uint64_t v = sh >= 64 ? 1 : (Sc[c] + ((1ull << sh) - 1)) >> sh;  /* ceil */
            S += v;
        }
        int h = 0;
        while (h < 32 && S > (1ull << (2 * h))) h++;
        e = T + 15 - E - h;
    }
    free(Ec); free(Sc);
    return e;
}

