// crt_device.cuh -- device functions of Parts 2-c, 3, 4 (Alg. 1 lines 7-10,
// PAPER.md:496-502), shared by the fused GEMM epilogue (gemm.cu) and the
// standalone CRT kernels (crt.cu, kslice.cu):
//   line 7:  c''_t = c'_t - floor(c'_t / m_t) m_t in [0, m_t)   (reduce_line7)
//   line 8:  S = sum_t c''_t w_t, w_t = M y_t / m_t, formed EXACTLY in integers:
//            per byte j of the weights, s_j = sum_g dp4a(c''_{4g..4g+3}, W_j[g])
//            (< 2^21), accumulated into 32-bit words with carries
//   line 9:  X = S - M floor(S/M + 1/2) (Eq. 1): Q = rint(S/M) from the top two
//            words in FP32 (within +-1), X = S - Q M mod 2^(32 W) by PTX carry
//            chains, one exact +-M correction into [-M/2, M/2)
//   line 10: C = 2^-(e+f) RN(X) (reading R10: X rounded to nearest even from its
//            integer bit fields, then the exact power-of-two scaling)
// The device recipe reproduces the exact big-integer result bit for bit; no FP64
// arithmetic (FP64 issue competes with the tcgen05 MMAs).
#pragma once
#include "oz2_device.cuh"
#include "oz2_kernels.h"

namespace oz2 {

// line 7: c'' = c' - floor(c'/m_t) m_t in [0, m_t), for any int32 c', in
// integer arithmetic: c' = hi 2^16 + lo (hi signed, lo in [0, 2^16)),
// y = hi k16s + lo + off7 == c' (mod m_t) with |k16s| <= m_t/2, so
// 0 <= y < 2^23 + 2^17, and the magic multiply gives floor(y / m_t) exactly
// (exact for y < 2^24).  Six integer instructions.
template <int NM>
__device__ __forceinline__ uint32_t reduce_line7(int32_t c, int t) {
    const Oz2Table& T = c_tab[NM];
    const uint32_t y = (uint32_t)((c >> 16) * T.k16s[t]) + ((uint32_t)c & 0xffffu) + T.off7[t];
    const uint32_t q = __umulhi(y, T.magic[t]);
    return q * T.negm[t] + y;                                   // y - q m_t (mod 2^32)
}

// line 7 for the GEMM drain, with the floor on the full-rate FP32 pipe instead
// of a quarter-rate IMAD.HI (tools/mb/op_rates.cu): c' = hi 2^18 + lo (hi
// signed, |hi| <= 2^13; lo in [0, 2^18)); L = lo | 0x4B200000 is the bits of the
// binary32 2^23 + 2^21 + lo; y' = hi k18s + L + K with k18s == 2^18 (mod m_t),
// |k18s| <= m_t / 2, and K = -8 k18s (so that the 2^21 offset cancels mod m_t)
// is the bits of 2^23 + y with y == c' (mod m_t), 2^20 <= y < 2^22.2.
// f = y - h_t exactly, one FMA f RN(1/m_t) + 1.5 2^23 rounds to 1.5 2^23 +
// floor(y / m_t) (|f| < 2^22.2: the product's error is < 0.27 / m_t, and
// (y - h_t) / m_t lies at least 1 / (2 m_t) from every half-integer), and the
// low byte of y' + qb (2^32 - m_t) is c'' (the bit offsets 0x4B000000 and
// 0x4B400000 m_t vanish mod 256).  Odd m_t only (m_1 = 256: the low byte of c').
// The upper bytes of the result are not the residue.
template <int NM>
__device__ __forceinline__ uint32_t reduce_line7_lowbyte(int32_t c, int t) {
    const Oz2Table& T = c_tab[NM];
    const uint32_t L = ((uint32_t)c & 0x3ffffu) | 0x4B200000u;
    const uint32_t y = (uint32_t)((c >> 18) * T.k18s[t]) + L + T.k18k[t];
    const float f = __fsub_rn(__uint_as_float(y), T.h23f[t]);                    // y - h_t, exact
    const uint32_t qb = __float_as_uint(__fmaf_rn(f, T.invm[t], 12582912.0f));
    return qb * T.negm[t] + y;
}

// ---------------------------------------------------------------------------
// multi-word (32-bit) two's-complement integers, PTX carry chains
// ---------------------------------------------------------------------------
// a -= b, a += b modulo 2^(32 W); one asm statement per chain (the carry flag
// does not survive between asm statements)
template <int W>
__device__ __forceinline__ void mw_sub(uint32_t (&a)[W], const uint32_t* b) {
    if constexpr (W == 1) {
        a[0] -= b[0];
    } else if constexpr (W == 2) {
        asm("sub.cc.u32 %0, %0, %2;\n\tsubc.u32 %1, %1, %3;"
            : "+r"(a[0]), "+r"(a[1])
            : "r"(b[0]), "r"(b[1]));
    } else if constexpr (W == 3) {
        asm("sub.cc.u32 %0, %0, %3;\n\tsubc.cc.u32 %1, %1, %4;\n\tsubc.u32 %2, %2, %5;"
            : "+r"(a[0]), "+r"(a[1]), "+r"(a[2])
            : "r"(b[0]), "r"(b[1]), "r"(b[2]));
    } else if constexpr (W == 4) {
        asm("sub.cc.u32 %0, %0, %4;\n\tsubc.cc.u32 %1, %1, %5;\n\tsubc.cc.u32 %2, %2, %6;\n\tsubc.u32 %3, %3, %7;"
            : "+r"(a[0]), "+r"(a[1]), "+r"(a[2]), "+r"(a[3])
            : "r"(b[0]), "r"(b[1]), "r"(b[2]), "r"(b[3]));
    } else if constexpr (W == 5) {
        asm("sub.cc.u32 %0, %0, %5;\n\tsubc.cc.u32 %1, %1, %6;\n\tsubc.cc.u32 %2, %2, %7;\n\tsubc.cc.u32 %3, %3, %8;\n\tsubc.u32 %4, %4, %9;"
            : "+r"(a[0]), "+r"(a[1]), "+r"(a[2]), "+r"(a[3]), "+r"(a[4])
            : "r"(b[0]), "r"(b[1]), "r"(b[2]), "r"(b[3]), "r"(b[4]));
    } else if constexpr (W == 6) {
        asm("sub.cc.u32 %0, %0, %6;\n\tsubc.cc.u32 %1, %1, %7;\n\tsubc.cc.u32 %2, %2, %8;\n\tsubc.cc.u32 %3, %3, %9;\n\tsubc.cc.u32 %4, %4, %10;\n\tsubc.u32 %5, %5, %11;"
            : "+r"(a[0]), "+r"(a[1]), "+r"(a[2]), "+r"(a[3]), "+r"(a[4]), "+r"(a[5])
            : "r"(b[0]), "r"(b[1]), "r"(b[2]), "r"(b[3]), "r"(b[4]), "r"(b[5]));
    } else {
        static_assert(W <= 6, "mw chain width");
    }
}
template <int W>
__device__ __forceinline__ void mw_add(uint32_t (&a)[W], const uint32_t* b) {
    if constexpr (W == 1) {
        a[0] += b[0];
    } else if constexpr (W == 2) {
        asm("add.cc.u32 %0, %0, %2;\n\taddc.u32 %1, %1, %3;"
            : "+r"(a[0]), "+r"(a[1])
            : "r"(b[0]), "r"(b[1]));
    } else if constexpr (W == 3) {
        asm("add.cc.u32 %0, %0, %3;\n\taddc.cc.u32 %1, %1, %4;\n\taddc.u32 %2, %2, %5;"
            : "+r"(a[0]), "+r"(a[1]), "+r"(a[2])
            : "r"(b[0]), "r"(b[1]), "r"(b[2]));
    } else if constexpr (W == 4) {
        asm("add.cc.u32 %0, %0, %4;\n\taddc.cc.u32 %1, %1, %5;\n\taddc.cc.u32 %2, %2, %6;\n\taddc.u32 %3, %3, %7;"
            : "+r"(a[0]), "+r"(a[1]), "+r"(a[2]), "+r"(a[3])
            : "r"(b[0]), "r"(b[1]), "r"(b[2]), "r"(b[3]));
    } else if constexpr (W == 5) {
        asm("add.cc.u32 %0, %0, %5;\n\taddc.cc.u32 %1, %1, %6;\n\taddc.cc.u32 %2, %2, %7;\n\taddc.cc.u32 %3, %3, %8;\n\taddc.u32 %4, %4, %9;"
            : "+r"(a[0]), "+r"(a[1]), "+r"(a[2]), "+r"(a[3]), "+r"(a[4])
            : "r"(b[0]), "r"(b[1]), "r"(b[2]), "r"(b[3]), "r"(b[4]));
    } else if constexpr (W == 6) {
        asm("add.cc.u32 %0, %0, %6;\n\taddc.cc.u32 %1, %1, %7;\n\taddc.cc.u32 %2, %2, %8;\n\taddc.cc.u32 %3, %3, %9;\n\taddc.cc.u32 %4, %4, %10;\n\taddc.u32 %5, %5, %11;"
            : "+r"(a[0]), "+r"(a[1]), "+r"(a[2]), "+r"(a[3]), "+r"(a[4]), "+r"(a[5])
            : "r"(b[0]), "r"(b[1]), "r"(b[2]), "r"(b[3]), "r"(b[4]), "r"(b[5]));
    } else {
        static_assert(W <= 6, "mw chain width");
    }
}

// 2^sc * RN(X) for a signed WX-word integer X (reading R10: round to nearest
// even, then scale), in integer arithmetic; only a subnormal or overflowing
// result takes the FP64 ldexp path.
template <int WX>
__device__ __forceinline__ double x_to_double_scaled(const uint32_t (&X)[WX], int sc) {
    constexpr int U = (WX + 1) / 2;                        // 64-bit words
    const uint32_t s = (uint32_t)((int32_t)X[WX - 1] >> 31);
    uint32_t mag[WX], sv[WX];
    #pragma unroll
    for (int i = 0; i < WX; i++) { mag[i] = X[i] ^ s; sv[i] = s; }
    mw_sub<WX>(mag, sv);                                   // |X| = (X ^ s) - s
    uint64_t u[U];
    #pragma unroll
    for (int i = 0; i < U; i++)
        u[i] = (uint64_t)mag[2 * i] | ((2 * i + 1 < WX ? (uint64_t)mag[2 * i + 1] : 0ull) << 32);
    uint64_t top, below = 0;
    int E0;                                                // |X| = (top + frac) 2^E0, bit 63 of top set
    if constexpr (U == 1) {
        if (u[0] == 0) return 0.0;
        const int lz = __clzll((long long)u[0]);
        top = u[0] << lz;
        E0 = -lz;
    } else {
        int lead = 0;
        #pragma unroll
        for (int i = 1; i < U; i++) if (u[i]) lead = i;
        uint64_t hi = u[0], lo = 0;
        #pragma unroll
        for (int i = 1; i < U; i++) if (lead == i) { hi = u[i]; lo = u[i - 1]; }
        if (hi == 0) return 0.0;
        const int lz = __clzll((long long)hi);
        top = lz ? (hi << lz) | (lo >> (64 - lz)) : hi;
        below = lz ? lo << lz : lo;
        if (lead == 0) below = 0;
        #pragma unroll
        for (int i = 0; i + 2 < U; i++) if (i + 1 < lead) below |= u[i];
        E0 = 64 * lead - lz;
    }
    uint64_t mant = top >> 11;                             // 53 bits, leading one at bit 52
    const uint64_t rbit = (top >> 10) & 1ull;
    const uint64_t sticky = ((top & 0x3ffull) | below) ? 1ull : 0ull;
    mant += rbit & (sticky | (mant & 1ull));               // round half to even (may reach 2^53)
    const int ebias = 63 + E0 + sc + 1023;                 // biased exponent of mant * 2^(11 + E0 + sc)
    const uint64_t sign = (uint64_t)(s & 0x80000000u) << 32;
    if (ebias >= 1 && ebias <= 2046)
        return __longlong_as_double((long long)(sign | (((uint64_t)(ebias - 1) << 52) + mant)));
    // rare: subnormal or overflowing result -- RN(X) is mant * 2^(11 + E0) exactly
    const double r = ldexp((double)mant, 11 + E0);
    return ldexp(s ? -r : r, sc);
}

// 4 x 4 byte transpose: out[e] byte i = byte e of in[i]
__device__ __forceinline__ void transpose4x4(uint32_t a, uint32_t b, uint32_t c, uint32_t d, uint32_t (&o)[4]) {
    const uint32_t ab_lo = prmt(a, b, 0x5140u), ab_hi = prmt(a, b, 0x7362u);
    const uint32_t cd_lo = prmt(c, d, 0x5140u), cd_hi = prmt(c, d, 0x7362u);
    o[0] = prmt(ab_lo, cd_lo, 0x5410u);
    o[1] = prmt(ab_lo, cd_lo, 0x7632u);
    o[2] = prmt(ab_hi, cd_hi, 0x5410u);
    o[3] = prmt(ab_hi, cd_hi, 0x7632u);
}

// lines 8-10 from the reduced residues c''_t in [0, m_t), packed 4 per word
// (byte i of P[g] = c''_(4g+i), 0 beyond N), entirely in integer arithmetic
// (FP64 in the GEMM epilogue would compete with the tensor pipe):
//   line 8:  S = sum_t c''_t w_t exactly: per byte j of the weights
//            s_j = sum_g dp4a(P[g], Wb[j][g]) < 2^21, S = sum_j s_j 2^(8j)
//            accumulated into 32-bit words (64-bit column sums, carries);
//   line 9:  Q = rint(S / M) from the top two words in FP32 (within +-1 of
//            floor(S/M + 1/2)), X = S - Q M mod 2^(32 WX), then one exact +-M
//            correction into [-M/2, M/2) -- the Eq. (1) result for every S;
//   line 10: C = 2^-(e+f) RN(X).
template <int NM>
__device__ __forceinline__ double crt_from_packed(const uint32_t (&P)[(NM + 3) / 4], int ei, int fj) {
    const Oz2Table& T = c_tab[NM];
    constexpr int G = (NM + 3) / 4, JB = crt_bytes(NM), WS = crt_swords(NM), WX = crt_words(NM);
    uint32_t S[WS];
    uint64_t carry = 0;
    #pragma unroll
    for (int w = 0; w < WS; w++) {
        uint64_t col = carry;
        #pragma unroll
        for (int i = 0; i < 4; i++) {
            const int j = 4 * w + i;
            if (j < JB) {
                uint32_t sj = 0;
                #pragma unroll
                for (int g = 0; g < G; g++) sj = dp4a_uu(P[g], T.Wb[j][g], sj);
                col += (uint64_t)sj << (8 * i);
            }
        }
        S[w] = (uint32_t)col;
        carry = col >> 32;
    }
    const float top = WS >= 2 ? fmaf(__uint2float_rn(S[WS - 1]), 4294967296.0f, __uint2float_rn(S[WS - 2]))
                              : __uint2float_rn(S[0]);
    const uint32_t Q = (uint32_t)(__float_as_int(fmaf(top, T.qscale, 12582912.0f)) - 0x4B400000);
    uint32_t X[WX], QM[WX];
    {
        uint64_t c = 0;
        #pragma unroll
        for (int w = 0; w < WX; w++) {
            X[w] = S[w];
            const uint64_t p = (uint64_t)Q * T.M32[w] + c;
            QM[w] = (uint32_t)p;
            c = p >> 32;
        }
    }
    mw_sub<WX>(X, QM);                                     // X = S - Q M  (mod 2^(32 WX))
    uint32_t D[WX];
    #pragma unroll
    for (int w = 0; w < WX; w++) D[w] = X[w];
    mw_sub<WX>(D, T.Mh32);                                 // X - M/2
    if ((int32_t)D[WX - 1] >= 0) {
        mw_sub<WX>(X, T.M32);
    } else {
        #pragma unroll
        for (int w = 0; w < WX; w++) D[w] = X[w];
        mw_add<WX>(D, T.Mh32);                             // X + M/2
        if ((int32_t)D[WX - 1] < 0) mw_add<WX>(X, T.M32);
    }
    if (ei == OZ2_EXP_NONFINITE_DEV || fj == OZ2_EXP_NONFINITE_DEV) return __longlong_as_double(0x7ff8000000000000ll);
    return x_to_double_scaled<WX>(X, -(ei + fj));
}

template <int NM>
__device__ __forceinline__ double crt_element(const int32_t (&cp)[NM], int ei, int fj) {
    constexpr int G = (NM + 3) / 4;
    uint32_t P[G];
    #pragma unroll
    for (int g = 0; g < G; g++) P[g] = 0;
    #pragma unroll
    for (int t = 0; t < NM; t++) P[t / 4] |= reduce_line7<NM>(cp[t], t) << (8 * (t % 4));
    return crt_from_packed<NM>(P, ei, fj);
}

}  // namespace oz2
