// crt.cu -- Parts 2-c, 3, 4 of Ozaki scheme II (Alg. 1 lines 7-10,
// PAPER.md:496-502) on sm_100a, exactly:
//   line 7:  c''_t = c'_t - floor(c'_t / m_t) m_t                 in [0, m_t)
//   line 8:  S = sum_t c''_t w_t, w_t = M y_t / m_t, held as P FP64 piece sums
//            S_p = sum_t c''_t W[p][t] (W < 2^38, c'' < 2^8, N <= 20 => every
//            product < 2^46 and every partial sum < 2^51: exact)
//   line 9:  X = S - M floor(S/M + 1/2) (Eq. 1): Q from the top two pieces in
//            FP64, X_p = S_p - Q M_p exact, X assembled as a 192-bit integer and
//            corrected by +-M if Q was off by one (so X is exact for every S)
//   line 10: C = 2^-(e+f) RN(X)  (reading R10: round X to nearest even, then scale)
// The device recipe reproduces the exact big-integer result bit for bit.
#include "oz2_device.cuh"
#include "oz2_kernels.h"

namespace oz2 {

// line 7: c'' = c' - floor(c'/m_t) m_t in [0, m_t), for any int32 c', in
// integer arithmetic: u = c' mod 2^32 = hi 2^16 + lo, y = hi (2^16 mod m_t) + lo
// (+ (-2^32) mod m_t when c' < 0) == c' (mod m_t), y < 2^24, then the magic
// multiply gives floor(y / m_t) exactly.
template <int NM>
__device__ __forceinline__ uint32_t reduce_line7(int32_t c, int t) {
    const Oz2Table& T = c_tab[NM];
    const uint32_t u = (uint32_t)c;
    const uint32_t y = (u >> 16) * T.k16[t] + (u & 0xffffu) + ((uint32_t)(c >> 31) & T.g32[t]);
    const uint32_t q = __umulhi(y, T.magic[t]);
    return y - q * (uint32_t)T.m[t];
}

// exact uint32 (< 2^52) -> double without the conversion pipe
__device__ __forceinline__ double u32_to_double(uint32_t r) {
    return __hiloint2double(0x43300000, (int)r) - 4503599627370496.0;   // (2^52 + r) - 2^52
}

// ---------------------------------------------------------------------------
// multi-limb integers (L = 4: 128 bit, L = 6: 192 bit) with PTX carry chains
// ---------------------------------------------------------------------------
template <int L> struct Limbs { uint32_t w[L]; };

__device__ __forceinline__ void add4(Limbs<4>& a, const Limbs<4>& b) {
    asm("add.cc.u32 %0, %0, %4;\n\taddc.cc.u32 %1, %1, %5;\n\taddc.cc.u32 %2, %2, %6;\n\taddc.u32 %3, %3, %7;"
        : "+r"(a.w[0]), "+r"(a.w[1]), "+r"(a.w[2]), "+r"(a.w[3]) : "r"(b.w[0]), "r"(b.w[1]), "r"(b.w[2]), "r"(b.w[3]));
}
__device__ __forceinline__ void sub4(Limbs<4>& a, const Limbs<4>& b) {
    asm("sub.cc.u32 %0, %0, %4;\n\tsubc.cc.u32 %1, %1, %5;\n\tsubc.cc.u32 %2, %2, %6;\n\tsubc.u32 %3, %3, %7;"
        : "+r"(a.w[0]), "+r"(a.w[1]), "+r"(a.w[2]), "+r"(a.w[3]) : "r"(b.w[0]), "r"(b.w[1]), "r"(b.w[2]), "r"(b.w[3]));
}
__device__ __forceinline__ void add6(Limbs<6>& a, const Limbs<6>& b) {
    asm("add.cc.u32 %0, %0, %6;\n\taddc.cc.u32 %1, %1, %7;\n\taddc.cc.u32 %2, %2, %8;\n\t"
        "addc.cc.u32 %3, %3, %9;\n\taddc.cc.u32 %4, %4, %10;\n\taddc.u32 %5, %5, %11;"
        : "+r"(a.w[0]), "+r"(a.w[1]), "+r"(a.w[2]), "+r"(a.w[3]), "+r"(a.w[4]), "+r"(a.w[5])
        : "r"(b.w[0]), "r"(b.w[1]), "r"(b.w[2]), "r"(b.w[3]), "r"(b.w[4]), "r"(b.w[5]));
}
__device__ __forceinline__ void sub6(Limbs<6>& a, const Limbs<6>& b) {
    asm("sub.cc.u32 %0, %0, %6;\n\tsubc.cc.u32 %1, %1, %7;\n\tsubc.cc.u32 %2, %2, %8;\n\t"
        "subc.cc.u32 %3, %3, %9;\n\tsubc.cc.u32 %4, %4, %10;\n\tsubc.u32 %5, %5, %11;"
        : "+r"(a.w[0]), "+r"(a.w[1]), "+r"(a.w[2]), "+r"(a.w[3]), "+r"(a.w[4]), "+r"(a.w[5])
        : "r"(b.w[0]), "r"(b.w[1]), "r"(b.w[2]), "r"(b.w[3]), "r"(b.w[4]), "r"(b.w[5]));
}
template <int L> __device__ __forceinline__ void ladd(Limbs<L>& a, const Limbs<L>& b) {
    if constexpr (L == 4) add4(a, b); else add6(a, b);
}
template <int L> __device__ __forceinline__ void lsub(Limbs<L>& a, const Limbs<L>& b) {
    if constexpr (L == 4) sub4(a, b); else sub6(a, b);
}
template <int L> __device__ __forceinline__ Limbs<L> lzero() {
    Limbs<L> z;
    #pragma unroll
    for (int i = 0; i < L; i++) z.w[i] = 0;
    return z;
}
template <int L> __device__ __forceinline__ Limbs<L> lconst(const uint64_t (&v)[3]) {
    Limbs<L> z;
    #pragma unroll
    for (int i = 0; i < L; i++) z.w[i] = (uint32_t)(v[i / 2] >> (32 * (i & 1)));
    return z;
}
// (vh:vl) * 2^(38 p) placed into L limbs (bits beyond 32 L dropped: arithmetic mod 2^(32 L))
template <int L, int P>
__device__ __forceinline__ Limbs<L> place(uint32_t vl, uint32_t vh) {
    constexpr int S = 38 * P, q = S / 32, r = S % 32;
    Limbs<L> x = lzero<L>();
    if constexpr (r == 0) {
        if (q < L) x.w[q] = vl;
        if (q + 1 < L) x.w[q + 1] = vh;
    } else {
        if (q < L) x.w[q] = vl << r;
        if (q + 1 < L) x.w[q + 1] = __funnelshift_l(vl, vh, r);
        if (q + 2 < L) x.w[q + 2] = vh >> (32 - r);
    }
    return x;
}

// 2^sc * RN(X) for a signed L-limb integer X (reading R10: round, then scale)
template <int L>
__device__ __forceinline__ double limbs_to_double_scaled(Limbs<L> X, int sc) {
    const bool neg = (int32_t)X.w[L - 1] < 0;
    Limbs<L> mag = lzero<L>();
    lsub<L>(mag, X);                                       // -X
    #pragma unroll
    for (int i = 0; i < L; i++) mag.w[i] = neg ? mag.w[i] : X.w[i];
    // 64-bit words, least significant first
    uint64_t w[L / 2];
    #pragma unroll
    for (int i = 0; i < L / 2; i++) w[i] = ((uint64_t)mag.w[2 * i + 1] << 32) | mag.w[2 * i];
    double r;
    int sh = 0;
    // the highest non-zero 64-bit word
    int lead = 0;
    #pragma unroll
    for (int i = 1; i < L / 2; i++) if (w[i]) lead = i;
    if (lead == 0) {
        r = __ull2double_rn(w[0]);                          // exact rounding of a 64-bit integer
    } else {
        const uint64_t hi = w[lead], lo = w[lead - 1];
        const int lz = __clzll((long long)hi);
        const uint64_t top = lz ? (hi << lz) | (lo >> (64 - lz)) : hi;   // the 64 leading bits
        uint64_t below = lo << lz;                         // bits below the window in this word
        #pragma unroll
        for (int i = 0; i < L / 2 - 2; i++) if (i < lead - 1) below |= w[i];
        sh = 64 * lead - lz;
        r = __ull2double_rn(top | (below ? 1ull : 0ull));   // sticky below the round bit
    }
    if (neg) r = -r;
    const int s2 = sc + sh;
    if (s2 >= -1022 && s2 <= 1023) {
        const double p = r * __longlong_as_double((long long)(s2 + 1023) << 52);
        if (fabs(p) >= 0x1p-1022 || r == 0.0) return p;     // exact
    }
    return ldexp(ldexp(r, sh), sc);                         // rare: extreme exponents (one rounding)
}

template <int P, int L>
__device__ __forceinline__ Limbs<L> assemble_biased(const uint64_t (&b)[5]) {
    Limbs<L> X = place<L, 0>((uint32_t)b[0], (uint32_t)(b[0] >> 32));
    if constexpr (P > 1) ladd<L>(X, place<L, 1>((uint32_t)b[1], (uint32_t)(b[1] >> 32)));
    if constexpr (P > 2) ladd<L>(X, place<L, 2>((uint32_t)b[2], (uint32_t)(b[2] >> 32)));
    if constexpr (P > 3) ladd<L>(X, place<L, 3>((uint32_t)b[3], (uint32_t)(b[3] >> 32)));
    if constexpr (P > 4) ladd<L>(X, place<L, 4>((uint32_t)b[4], (uint32_t)(b[4] >> 32)));
    return X;
}

// lines 8-10 from the reduced residues r_t = c''_t in [0, m_t):
//   S_p = sum_t r_t W[p][t] exactly (W < 2^38, r < 2^8, N <= 20: every partial
//   sum < 2^51); Q ~ S/M rounded (from the top two pieces, within +-1 of
//   floor(S/M + 1/2)); X_p = S_p - Q M_p with |X_p| < 2^51, so X_p + 1.5*2^52 is
//   exact and its bit pattern is X_p + 0x4338000000000000: the pieces are
//   summed as integers (mod 2^128, or 2^192 for N >= 16), the bias removed,
//   and X corrected by +-M into [-M/2, M/2) -- the exact Eq. (1) result.
template <int NM>
__device__ __forceinline__ double crt_from_residues(const uint32_t (&r)[NM], int ei, int fj) {
    const Oz2Table& T = c_tab[NM];
    constexpr int P = crt_pieces(NM);
    constexpr int L = NM <= 15 ? 4 : 6;                          // |X| < M/2 < 2^118 (N <= 15)
    constexpr double MAGIC = 6755399441055744.0;                 // 1.5 * 2^52
    double S[P];
    #pragma unroll
    for (int p = 0; p < P; p++) S[p] = 0.0;
    #pragma unroll
    for (int t = 0; t < NM; t++) {
        const double rt = u32_to_double(r[t]);
        #pragma unroll
        for (int p = 0; p < P; p++) S[p] = fma(rt, T.W[p][t], S[p]);       // exact
    }
    const double top = P >= 2 ? fma(S[P - 1], 0x1p38, S[P - 2]) : S[0];
    const double Q = fma(top, T.invM, MAGIC) - MAGIC;                       // rint(S / M), approximately
    uint64_t b[5] = {0, 0, 0, 0, 0};
    #pragma unroll
    for (int p = 0; p < P; p++) b[p] = (uint64_t)__double_as_longlong(fma(-Q, T.Mp[p], S[p] + MAGIC));
    Limbs<L> X = assemble_biased<P, L>(b);
    lsub<L>(X, lconst<L>(T.bias));
    // Eq. (1) range [-M/2, M/2): Q is within one of the exact quotient
    Limbs<L> D = X;
    lsub<L>(D, lconst<L>(T.Mhalf));                              // X - M/2
    Limbs<L> E = X;
    ladd<L>(E, lconst<L>(T.Mhalf));                              // X + M/2
    if ((int32_t)D.w[L - 1] >= 0) lsub<L>(X, lconst<L>(T.Mw));
    else if ((int32_t)E.w[L - 1] < 0) ladd<L>(X, lconst<L>(T.Mw));
    if (ei == OZ2_EXP_NONFINITE_DEV || fj == OZ2_EXP_NONFINITE_DEV) return __longlong_as_double(0x7ff8000000000000ll);
    return limbs_to_double_scaled<L>(X, -(ei + fj));
}

template <int NM>
__device__ __forceinline__ double crt_element(const int32_t (&cp)[NM], int ei, int fj) {
    uint32_t r[NM];
    #pragma unroll
    for (int t = 0; t < NM; t++) r[t] = reduce_line7<NM>(cp[t], t);
    return crt_from_residues<NM>(r, ei, fj);
}

template <int NM>
__global__ void __launch_bounds__(256)
crt_kernel(const int32_t* __restrict__ cprod, int64_t m, int64_t n, const int32_t* __restrict__ e,
           const int32_t* __restrict__ f, double* __restrict__ C, int64_t ldc) {
    int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (idx >= m * n) return;
    int64_t i = idx / n, j = idx % n;
    int32_t cp[NM];
    #pragma unroll
    for (int t = 0; t < NM; t++) cp[t] = __ldg(cprod + t * m * n + idx);
    C[i * ldc + j] = crt_element<NM>(cp, e[i], f[j]);
}

template <int NM>
static void launch_crt_nm(const int32_t* cprod, int64_t m, int64_t n, const int32_t* e, const int32_t* f,
                          double* C, int64_t ldc, cudaStream_t st) {
    int64_t tot = m * n;
    crt_kernel<NM><<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(cprod, m, n, e, f, C, ldc);
}

void launch_crt(const int32_t* cprod, int64_t m, int64_t n, const int32_t* e, const int32_t* f,
                int N, double* C, int64_t ldc, cudaStream_t st) {
    if (m * n == 0) return;
    switch (N) {
        case 2: launch_crt_nm<2>(cprod, m, n, e, f, C, ldc, st); break;
        case 3: launch_crt_nm<3>(cprod, m, n, e, f, C, ldc, st); break;
        case 4: launch_crt_nm<4>(cprod, m, n, e, f, C, ldc, st); break;
        case 5: launch_crt_nm<5>(cprod, m, n, e, f, C, ldc, st); break;
        case 6: launch_crt_nm<6>(cprod, m, n, e, f, C, ldc, st); break;
        case 7: launch_crt_nm<7>(cprod, m, n, e, f, C, ldc, st); break;
        case 8: launch_crt_nm<8>(cprod, m, n, e, f, C, ldc, st); break;
        case 9: launch_crt_nm<9>(cprod, m, n, e, f, C, ldc, st); break;
        case 10: launch_crt_nm<10>(cprod, m, n, e, f, C, ldc, st); break;
        case 11: launch_crt_nm<11>(cprod, m, n, e, f, C, ldc, st); break;
        case 12: launch_crt_nm<12>(cprod, m, n, e, f, C, ldc, st); break;
        case 13: launch_crt_nm<13>(cprod, m, n, e, f, C, ldc, st); break;
        case 14: launch_crt_nm<14>(cprod, m, n, e, f, C, ldc, st); break;
        case 15: launch_crt_nm<15>(cprod, m, n, e, f, C, ldc, st); break;
        case 16: launch_crt_nm<16>(cprod, m, n, e, f, C, ldc, st); break;
        case 17: launch_crt_nm<17>(cprod, m, n, e, f, C, ldc, st); break;
        case 18: launch_crt_nm<18>(cprod, m, n, e, f, C, ldc, st); break;
        case 19: launch_crt_nm<19>(cprod, m, n, e, f, C, ldc, st); break;
        case 20: launch_crt_nm<20>(cprod, m, n, e, f, C, ldc, st); break;
        default: break;
    }
}

}  // namespace oz2
