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

struct U192 { uint64_t w0, w1, w2; };

__device__ __forceinline__ U192 u192_from_i64(long long v) {
    U192 r; r.w0 = (uint64_t)v; r.w1 = r.w2 = v < 0 ? ~0ull : 0ull; return r;
}
__device__ __forceinline__ U192 u192_add(U192 a, U192 b) {
    U192 r;
    r.w0 = a.w0 + b.w0;
    uint64_t c0 = r.w0 < a.w0;
    uint64_t t = a.w1 + b.w1;
    uint64_t c1 = t < a.w1;
    r.w1 = t + c0;
    c1 += r.w1 < t;
    r.w2 = a.w2 + b.w2 + c1;
    return r;
}
__device__ __forceinline__ U192 u192_neg(U192 a) {
    U192 r; r.w0 = ~a.w0; r.w1 = ~a.w1; r.w2 = ~a.w2;
    return u192_add(r, u192_from_i64(1));
}
// v * 2^s for a signed 64-bit v, 0 <= s < 128, as a 192-bit two's complement
__device__ __forceinline__ U192 u192_shl_i64(long long v, int s) {
    U192 x = u192_from_i64(v);
    if (s >= 64) { x.w2 = x.w1; x.w1 = x.w0; x.w0 = 0; s -= 64; }
    if (s > 0) {
        x.w2 = (x.w2 << s) | (x.w1 >> (64 - s));
        x.w1 = (x.w1 << s) | (x.w0 >> (64 - s));
        x.w0 <<= s;
    }
    return x;
}
__device__ __forceinline__ bool u192_neg_p(U192 a) { return (long long)a.w2 < 0; }
// signed compare a >= b
__device__ __forceinline__ bool u192_ge(U192 a, U192 b) {
    if ((long long)a.w2 != (long long)b.w2) return (long long)a.w2 > (long long)b.w2;
    if (a.w1 != b.w1) return a.w1 > b.w1;
    return a.w0 >= b.w0;
}

// logical right shift, 0 <= s < 192
__device__ __forceinline__ U192 u192_shr(U192 a, int s) {
    if (s >= 128) { a.w0 = a.w2 >> (s - 128); a.w1 = 0; a.w2 = 0; return a; }
    if (s >= 64) { a.w0 = a.w1; a.w1 = a.w2; a.w2 = 0; s -= 64; }
    if (s) {
        a.w0 = (a.w0 >> s) | (a.w1 << (64 - s));
        a.w1 = (a.w1 >> s) | (a.w2 << (64 - s));
        a.w2 >>= s;
    }
    return a;
}

// 2^-(e+f) RN(X)   (Alg. 1 line 10, reading R10)
__device__ __forceinline__ double u192_to_double_scaled(U192 X, int sc) {
    const bool neg = u192_neg_p(X);
    if (neg) X = u192_neg(X);
    double r;
    if (X.w2 == 0 && X.w1 == 0) {
        r = __ull2double_rn(X.w0);                       // correctly rounded
    } else {
        const int bl = X.w2 ? 192 - __clzll((long long)X.w2) : 128 - __clzll((long long)X.w1);
        const int sh = bl - 64;                          // 1 .. 127
        const uint64_t top = u192_shr(X, sh).w0;         // the 64 leading bits
        uint64_t low;                                    // the sh dropped bits, != 0 ?
        if (sh < 64) low = X.w0 & ((1ull << sh) - 1);
        else low = X.w0 | (X.w1 & ((1ull << (sh - 64)) - 1));
        // 64 -> 53 bits drops 11: a sticky bit OR-ed into bit 0 rounds correctly
        r = __ull2double_rn(top | (low ? 1ull : 0ull));
        r = r * __longlong_as_double((long long)(sh + 1023) << 52);   // exact
    }
    if (neg) r = -r;
    if (sc >= -1022 && sc <= 1023) {
        const double p = r * __longlong_as_double((long long)(sc + 1023) << 52);
        if (fabs(p) >= 0x1p-1022 || r == 0.0) return p;  // exact
    }
    return ldexp(r, sc);                                 // subnormal / extreme: one rounding
}

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

// v * 2^s (v < 2^64, s a compile-time multiple of 38 below 192) added to Y, mod 2^192
template <int S>
__device__ __forceinline__ U192 u192_add_shl(U192 Y, uint64_t v) {
    U192 x;
    if (S == 0) { x.w0 = v; x.w1 = 0; x.w2 = 0; }
    else if (S < 64) { x.w0 = v << S; x.w1 = v >> (64 - S); x.w2 = 0; }
    else if (S == 64) { x.w0 = 0; x.w1 = v; x.w2 = 0; }
    else if (S < 128) { x.w0 = 0; x.w1 = v << (S - 64); x.w2 = v >> (128 - S); }
    else if (S == 128) { x.w0 = 0; x.w1 = 0; x.w2 = v; }
    else { x.w0 = 0; x.w1 = 0; x.w2 = v << (S - 128); }
    return u192_add(Y, x);
}

template <int P>
__device__ __forceinline__ U192 assemble_biased(const uint64_t (&b)[5]) {
    U192 Y = {0, 0, 0};
    Y = u192_add_shl<0>(Y, b[0]);
    if (P > 1) Y = u192_add_shl<38>(Y, b[1]);
    if (P > 2) Y = u192_add_shl<76>(Y, b[2]);
    if (P > 3) Y = u192_add_shl<114>(Y, b[3]);
    if (P > 4) Y = u192_add_shl<152>(Y, b[4]);
    return Y;
}

// lines 8-10 from the reduced residues r_t = c''_t in [0, m_t):
//   S_p = sum_t r_t W[p][t] exactly (W < 2^38, r < 2^8, N <= 20: every partial
//   sum < 2^51); Q ~ S/M rounded (from the top two pieces, within +-1 of
//   floor(S/M + 1/2)); X_p = S_p - Q M_p with |X_p| < 2^51, so X_p + 1.5*2^52 is
//   exact and its bit pattern is X_p + 0x4338000000000000: the pieces are
//   summed as integers, the bias removed, and X corrected by +-M into
//   [-M/2, M/2) -- the exact Eq. (1) result for every S.
template <int NM>
__device__ __forceinline__ double crt_from_residues(const uint32_t (&r)[NM], int ei, int fj) {
    const Oz2Table& T = c_tab[NM];
    constexpr int P = crt_pieces(NM);
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
    U192 X = assemble_biased<P>(b);
    X = u192_add(X, u192_neg(U192{T.bias[0], T.bias[1], T.bias[2]}));
    const U192 Mw = {T.Mw[0], T.Mw[1], T.Mw[2]};
    const U192 Mh = {T.Mhalf[0], T.Mhalf[1], T.Mhalf[2]};
    if (u192_ge(X, Mh)) X = u192_add(X, u192_neg(Mw));                   // X >= M/2
    else if (!u192_ge(X, u192_neg(Mh))) X = u192_add(X, Mw);              // X < -M/2
    if (ei == OZ2_EXP_NONFINITE_DEV || fj == OZ2_EXP_NONFINITE_DEV) return __longlong_as_double(0x7ff8000000000000ll);
    return u192_to_double_scaled(X, -(ei + fj));
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
