// scale.cu -- Part 1 and Part 2-a of Ozaki scheme II on sm_100a:
// Alg. 1 lines 1-5: exponent vectors e (rows of A) and f
// (columns of B), A' = trunc(D A), B' = trunc(B E), and the N symmetric int8
// residue planes (Eq. 11).
//
// Exponent rule FAST (reading R4): for each chunk of KC = 256
// consecutive inner indices, E_c = max ilogb|x| and S_c = sum u^2 with
// u = ceil(|x| 2^(15-E_c)) (>= 1 for x != 0); then E = max E_c,
// S = sum ceil(S_c / 4^(E-E_c)), h = min{h : S <= 4^h}, e = T + 15 - E - h.
// All integer, so the result does not depend on the reduction order.
//
// Residues: x = trunc(2^e a) as a 64-bit (N <= 16) or 96-bit (N > 16) two's
// complement integer; for odd m_t, y = sum_b byte_b(x) (2^(8b) mod m_t) with
// dp4a (+ (-2^64) mod m_t when x < 0), q = floor((y + h_t)/m_t) by a magic
// multiply, r = y - q m_t in [-h_t, h_t] (Eq. 1 for odd m); for m_1 = 256 the
// residue is the low byte of x (Eq. 1 tie 128 -> -128 = int8 wrap).
#include "oz2_device.cuh"
#include "oz2_kernels.h"

namespace oz2 {

constexpr int KC = 256;            // FAST chunk length (reading R4)
constexpr int ROW_THREADS = 256;
constexpr int MAX_CHUNKS = 512;    // k < 2^17

// ---------------------------------------------------------------------------
// FAST-rule per-element contribution: u^2 with u = ceil(mant 2^(ex + 15 - Ec))
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint64_t u_squared(const Dec& d, int Ec) {
    if (d.cls != 1) return 0;
    // |x| 2^(15-Ec) = mant 2^(-rs) < 2^16; rs >= 37 for normal x, but a
    // subnormal x has a short mantissa and rs may be <= 0 (exact left shift)
    int rs = -(d.ex + 15 - Ec);
    uint64_t u = rs <= 0 ? (d.mant << (-rs))
               : rs >= 64 ? 1ull : ((d.mant + ((1ull << rs) - 1)) >> rs);
    return u * u;
}

__device__ __forceinline__ uint64_t ceil_shift(uint64_t S, int sh) {
    if (S == 0) return 0;
    if (sh >= 64) return 1;
    return (S + ((1ull << sh) - 1)) >> sh;
}

// h = min{h >= 0 : S <= 4^h}
__device__ __forceinline__ int log4_ceil(uint64_t S) {
    if (S <= 1) return 0;
    int bl = 64 - __clzll((long long)(S - 1));
    return (bl + 1) / 2;
}

__device__ __forceinline__ int warp_max(int v) {
    #pragma unroll
    for (int o = 16; o; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ uint64_t warp_sum64(uint64_t v) {
    #pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// ---------------------------------------------------------------------------
// Residues of one integer (two's complement words) for modulus index t
// ---------------------------------------------------------------------------
template <int NM, int WORDS>
__device__ __forceinline__ uint32_t residue_odd(int t, const uint32_t (&w)[3], bool neg) {
    const Oz2Table& T = c_tab[NM];
    uint32_t acc = (uint32_t)T.h[t] + (neg ? (uint32_t)(WORDS == 2 ? T.g64[t] : T.g96[t]) : 0u);
    acc = dp4a_uu(w[0], T.cw[0][t], acc);
    acc = dp4a_uu(w[1], T.cw[1][t], acc);
    if (WORDS == 3) acc = dp4a_uu(w[2], T.cw[2][t], acc);
    uint32_t q = __umulhi(acc, T.magic[t]);
    return acc - q * (uint32_t)T.m[t] - (uint32_t)T.h[t];      // low byte = int8 residue
}

// x = trunc(2^e a) split into words; returns false-y (zeros) for e = sentinel
template <int WORDS>
__device__ __forceinline__ void to_words(double a, int e, uint32_t (&w)[3], bool& neg) {
    if (e == OZ2_EXP_NONFINITE_DEV) { w[0] = w[1] = w[2] = 0; neg = false; return; }
    double v = trunc(scale_pow2(a, e));
    if (WORDS == 2) {
        long long x = __double2ll_rz(v);
        w[0] = (uint32_t)x; w[1] = (uint32_t)((unsigned long long)x >> 32); w[2] = 0;
        neg = x < 0;
    } else {
        double hi = floor(v * 0x1p-32);              // exact
        double lo = fma(-hi, 0x1p32, v);             // exact, in [0, 2^32)
        long long h = __double2ll_rz(hi);
        w[0] = __double2uint_rz(lo);
        w[1] = (uint32_t)h; w[2] = (uint32_t)((unsigned long long)h >> 32);
        neg = v < 0.0;
    }
}

// ---------------------------------------------------------------------------
// exponent of one row (CTA-wide); x(l) = X[l * s]; result broadcast via smem
// ---------------------------------------------------------------------------
struct RowSmem {
    int Ec[MAX_CHUNKS];
    unsigned long long Sc[MAX_CHUNKS];
    int bad;
    int e;
};

template <int MODE>
__device__ int row_exponent(const double* __restrict__ X, int64_t k, int64_t s, int Tb, int kstar,
                            RowSmem& sm) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nwarps = blockDim.x >> 5;
    const int nch = (int)((k + KC - 1) / KC);
    if (threadIdx.x == 0) sm.bad = 0;
    __syncthreads();
    for (int c = warp; c < nch; c += nwarps) {
        double v[KC / 32];
        int64_t base = (int64_t)c * KC;
        #pragma unroll
        for (int j = 0; j < KC / 32; j++) {
            int64_t l = base + lane + 32 * j;
            v[j] = l < k ? __ldg(X + l * s) : 0.0;
        }
        int E = INT32_MIN;
        bool bad = false;
        #pragma unroll
        for (int j = 0; j < KC / 32; j++) {
            Dec d = decompose(v[j]);
            if (d.cls == 2) bad = true;
            if (d.cls == 1) E = max(E, d.ilogb);
        }
        E = warp_max(E);
        if (__any_sync(0xffffffffu, bad) && lane == 0) sm.bad = 1;
        uint64_t S = 0;
        if (MODE == 0 && E != INT32_MIN) {
            #pragma unroll
            for (int j = 0; j < KC / 32; j++) S += u_squared(decompose(v[j]), E);
            S = warp_sum64(S);
        }
        if (lane == 0) { sm.Ec[c] = E; sm.Sc[c] = S; }
    }
    __syncthreads();
    if (warp == 0) {
        int E = INT32_MIN;
        for (int c = lane; c < nch; c += 32) E = max(E, sm.Ec[c]);
        E = warp_max(E);
        int e;
        if (E == INT32_MIN) {
            e = 0;                                            // zero row
        } else if (MODE == 0) {
            uint64_t S = 0;
            for (int c = lane; c < nch; c += 32)
                if (sm.Ec[c] != INT32_MIN) S += ceil_shift(sm.Sc[c], 2 * (E - sm.Ec[c]));
            S = warp_sum64(S);
            e = Tb + 15 - E - log4_ceil(S);
        } else {
            e = kstar - 1 - E;                                // EQ17 (reading R5)
        }
        if (sm.bad) e = OZ2_EXP_NONFINITE_DEV;
        if (lane == 0) sm.e = e;
    }
    __syncthreads();
    return sm.e;
}

// residues of row i of A for all N moduli: planes out[t][i][l], 4 elements per thread
template <int NM, int WORDS>
__device__ void row_residues(const double* __restrict__ X, int64_t k, int e, int8_t* __restrict__ out,
                             int64_t plane_stride) {
    const bool vec = ((reinterpret_cast<uintptr_t>(X) & 15) == 0);
    for (int64_t l0 = 4 * (int64_t)threadIdx.x; l0 < k; l0 += 4 * (int64_t)blockDim.x) {
        double a[4];
        if (vec && l0 + 4 <= k) {
            double2 p = __ldg(reinterpret_cast<const double2*>(X + l0));
            double2 q = __ldg(reinterpret_cast<const double2*>(X + l0 + 2));
            a[0] = p.x; a[1] = p.y; a[2] = q.x; a[3] = q.y;
        } else {
            #pragma unroll
            for (int j = 0; j < 4; j++) a[j] = (l0 + j < k) ? __ldg(X + l0 + j) : 0.0;
        }
        uint32_t w[4][3];
        bool neg[4];
        #pragma unroll
        for (int j = 0; j < 4; j++) to_words<WORDS>(a[j], e, w[j], neg[j]);
        uint32_t* dst = reinterpret_cast<uint32_t*>(out + l0);
        // t = 0: m = 256, the low byte of x
        dst[0] = pack_lo_bytes(w[0][0], w[1][0], w[2][0], w[3][0]);
        #pragma unroll
        for (int t = 1; t < NM; t++) {
            uint32_t r0 = residue_odd<NM, WORDS>(t, w[0], neg[0]);
            uint32_t r1 = residue_odd<NM, WORDS>(t, w[1], neg[1]);
            uint32_t r2 = residue_odd<NM, WORDS>(t, w[2], neg[2]);
            uint32_t r3 = residue_odd<NM, WORDS>(t, w[3], neg[3]);
            *reinterpret_cast<uint32_t*>(out + t * plane_stride + l0) = pack_lo_bytes(r0, r1, r2, r3);
        }
    }
}

// ---------------------------------------------------------------------------
// Row kernels (A: m x k, row-major, lda)
// ---------------------------------------------------------------------------
// what: 1 = exponents, 2 = residues (given e), 3 = both
template <int NM, int WORDS, int MODE>
__global__ void __launch_bounds__(ROW_THREADS)
rows_kernel(const double* __restrict__ A, int64_t m, int64_t k, int64_t lda, int what, int kstar,
            int32_t* __restrict__ e_io, int8_t* __restrict__ res, int64_t ldr) {
    __shared__ RowSmem sm;
    const int64_t i = blockIdx.x;
    if (i >= m) return;
    const double* X = A + i * lda;
    int e;
    if (what & 1) {
        e = row_exponent<MODE>(X, k, 1, c_tab[NM].T, kstar, sm);
        if (threadIdx.x == 0) e_io[i] = e;
    } else {
        e = e_io[i];
    }
    if (what & 2) row_residues<NM, WORDS>(X, k, e, res + i * ldr, m * ldr);
}

// A' = trunc(D A) as FP64 (split API)
__global__ void trunc_rows_kernel(const double* __restrict__ A, int64_t m, int64_t k, int64_t lda,
                                  const int32_t* __restrict__ e, double* __restrict__ out) {
    int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (idx >= m * k) return;
    int64_t i = idx / k, l = idx % k;
    int ei = e[i];
    out[idx] = ei == OZ2_EXP_NONFINITE_DEV ? 0.0 : trunc(scale_pow2(A[i * lda + l], ei));
}

// ---------------------------------------------------------------------------
// Column kernels (B: k x n, row-major, ldb)
// ---------------------------------------------------------------------------
// chunk statistics: block (32 columns) x (one KC chunk), 8 warps x 32 rows
template <int MODE>
__global__ void __launch_bounds__(256)
cols_stats_kernel(const double* __restrict__ B, int64_t k, int64_t n, int64_t ldb,
                  int32_t* __restrict__ Ec_out, unsigned long long* __restrict__ Sc_out,
                  int32_t* __restrict__ bad_out) {
    __shared__ int sE[8][32];
    __shared__ unsigned long long sS[8][32];
    __shared__ int sBad[8][32];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t j = (int64_t)blockIdx.x * 32 + lane;
    const int64_t c = blockIdx.y;
    const int64_t r0 = c * KC + warp * 32;
    double v[32];
    #pragma unroll
    for (int q = 0; q < 32; q++) {
        int64_t l = r0 + q;
        v[q] = (j < n && l < k) ? __ldg(B + l * ldb + j) : 0.0;
    }
    int E = INT32_MIN;
    int bad = 0;
    #pragma unroll
    for (int q = 0; q < 32; q++) {
        Dec d = decompose(v[q]);
        if (d.cls == 2) bad = 1;
        if (d.cls == 1) E = max(E, d.ilogb);
    }
    sE[warp][lane] = E;
    sBad[warp][lane] = bad;
    __syncthreads();
    int Ec = INT32_MIN;
    #pragma unroll
    for (int w = 0; w < 8; w++) Ec = max(Ec, sE[w][lane]);
    uint64_t S = 0;
    if (MODE == 0 && Ec != INT32_MIN) {
        #pragma unroll
        for (int q = 0; q < 32; q++) S += u_squared(decompose(v[q]), Ec);
    }
    sS[warp][lane] = S;
    __syncthreads();
    if (warp == 0 && j < n) {
        uint64_t St = 0;
        int b = 0;
        #pragma unroll
        for (int w = 0; w < 8; w++) { St += sS[w][lane]; b |= sBad[w][lane]; }
        Ec_out[c * n + j] = Ec;
        Sc_out[c * n + j] = St;
        if (b) atomicOr(bad_out + j, 1);
    }
}

template <int MODE>
__global__ void cols_finalize_kernel(const int32_t* __restrict__ Ec, const unsigned long long* __restrict__ Sc,
                                     const int32_t* __restrict__ bad, int64_t n, int nch, int Tb, int kstar,
                                     int32_t* __restrict__ f) {
    int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (j >= n) return;
    int E = INT32_MIN;
    for (int c = 0; c < nch; c++) E = max(E, Ec[(int64_t)c * n + j]);
    int e;
    if (E == INT32_MIN) {
        e = 0;
    } else if (MODE == 0) {
        uint64_t S = 0;
        for (int c = 0; c < nch; c++) {
            int Ecc = Ec[(int64_t)c * n + j];
            if (Ecc != INT32_MIN) S += ceil_shift(Sc[(int64_t)c * n + j], 2 * (E - Ecc));
        }
        e = Tb + 15 - E - log4_ceil(S);
    } else {
        e = kstar - 1 - E;
    }
    f[j] = bad[j] ? OZ2_EXP_NONFINITE_DEV : e;
}

// residues of B columns into K-major planes out[t][j][l]: thread = column j,
// 16 consecutive l (one 16-byte store per modulus); block = 32 cols x 128 l
template <int NM, int WORDS>
__global__ void __launch_bounds__(256, 2)
cols_residues_kernel(const double* __restrict__ B, int64_t k, int64_t n, int64_t ldb,
                     const int32_t* __restrict__ f, int8_t* __restrict__ out, int64_t ldr) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t j = (int64_t)blockIdx.x * 32 + lane;
    const int64_t l0 = (int64_t)blockIdx.y * 128 + warp * 16;
    if (j >= n || l0 >= k) return;
    const int e = f[j];
    uint32_t w[16][3];
    bool neg[16];
    #pragma unroll
    for (int q = 0; q < 16; q++) {
        int64_t l = l0 + q;
        double a = l < k ? __ldg(B + l * ldb + j) : 0.0;
        to_words<WORDS>(a, e, w[q], neg[q]);
    }
    const int64_t plane = n * ldr;
    int8_t* dst = out + j * ldr + l0;
    // l0 < k <= ldr, all multiples of 16: the 16-byte store stays inside the row
    {
        uint4 o;
        o.x = pack_lo_bytes(w[0][0], w[1][0], w[2][0], w[3][0]);
        o.y = pack_lo_bytes(w[4][0], w[5][0], w[6][0], w[7][0]);
        o.z = pack_lo_bytes(w[8][0], w[9][0], w[10][0], w[11][0]);
        o.w = pack_lo_bytes(w[12][0], w[13][0], w[14][0], w[15][0]);
        *reinterpret_cast<uint4*>(dst) = o;
    }
    #pragma unroll
    for (int t = 1; t < NM; t++) {
        uint32_t r[16];
        #pragma unroll
        for (int q = 0; q < 16; q++) r[q] = residue_odd<NM, WORDS>(t, w[q], neg[q]);
        uint4 o;
        o.x = pack_lo_bytes(r[0], r[1], r[2], r[3]);
        o.y = pack_lo_bytes(r[4], r[5], r[6], r[7]);
        o.z = pack_lo_bytes(r[8], r[9], r[10], r[11]);
        o.w = pack_lo_bytes(r[12], r[13], r[14], r[15]);
        *reinterpret_cast<uint4*>(dst + t * plane) = o;
    }
}

__global__ void trunc_cols_kernel(const double* __restrict__ B, int64_t k, int64_t n, int64_t ldb,
                                  const int32_t* __restrict__ f, double* __restrict__ out) {
    int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;   // over k x n, B order
    if (idx >= k * n) return;
    int64_t l = idx / n, j = idx % n;
    int fj = f[j];
    out[j * k + l] = fj == OZ2_EXP_NONFINITE_DEV ? 0.0 : trunc(scale_pow2(B[l * ldb + j], fj));
}

// ---------------------------------------------------------------------------
// host launchers
// ---------------------------------------------------------------------------
template <int NM>
static void launch_rows_nm(const double* A, int64_t m, int64_t k, int64_t lda, int what, int mode,
                           int kstar, int32_t* e, int8_t* res, int64_t ldr, cudaStream_t st) {
    dim3 grid((unsigned)m), block(ROW_THREADS);
    constexpr int W = NM <= 16 ? 2 : 3;
    if (mode == 0) rows_kernel<NM, W, 0><<<grid, block, 0, st>>>(A, m, k, lda, what, kstar, e, res, ldr);
    else rows_kernel<NM, W, 1><<<grid, block, 0, st>>>(A, m, k, lda, what, kstar, e, res, ldr);
}

template <int NM>
static void launch_cols_res_nm(const double* B, int64_t k, int64_t n, int64_t ldb, const int32_t* f,
                               int8_t* res, int64_t ldr, cudaStream_t st) {
    dim3 grid((unsigned)((n + 31) / 32), (unsigned)((k + 127) / 128)), block(256);
    constexpr int W = NM <= 16 ? 2 : 3;
    cols_residues_kernel<NM, W><<<grid, block, 0, st>>>(B, k, n, ldb, f, res, ldr);
}

#define OZ2_DISPATCH_N(N, FN, ...)                                                   \
    switch (N) {                                                                     \
        case 2: FN<2>(__VA_ARGS__); break;   case 3: FN<3>(__VA_ARGS__); break;      \
        case 4: FN<4>(__VA_ARGS__); break;   case 5: FN<5>(__VA_ARGS__); break;      \
        case 6: FN<6>(__VA_ARGS__); break;   case 7: FN<7>(__VA_ARGS__); break;      \
        case 8: FN<8>(__VA_ARGS__); break;   case 9: FN<9>(__VA_ARGS__); break;      \
        case 10: FN<10>(__VA_ARGS__); break; case 11: FN<11>(__VA_ARGS__); break;    \
        case 12: FN<12>(__VA_ARGS__); break; case 13: FN<13>(__VA_ARGS__); break;    \
        case 14: FN<14>(__VA_ARGS__); break; case 15: FN<15>(__VA_ARGS__); break;    \
        case 16: FN<16>(__VA_ARGS__); break; case 17: FN<17>(__VA_ARGS__); break;    \
        case 18: FN<18>(__VA_ARGS__); break; case 19: FN<19>(__VA_ARGS__); break;    \
        case 20: FN<20>(__VA_ARGS__); break; default: break;                         \
    }

void launch_rows(const double* A, int64_t m, int64_t k, int64_t lda, int N, int what, int mode,
                 int kstar, int32_t* e, int8_t* res, int64_t ldr, cudaStream_t st) {
    if (m == 0) return;
    OZ2_DISPATCH_N(N, launch_rows_nm, A, m, k, lda, what, mode, kstar, e, res, ldr, st);
}

void launch_trunc_rows(const double* A, int64_t m, int64_t k, int64_t lda, const int32_t* e,
                       double* out, cudaStream_t st) {
    int64_t tot = m * k;
    if (!tot) return;
    trunc_rows_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(A, m, k, lda, e, out);
}

size_t cols_stats_bytes(int64_t k, int64_t n) {
    int64_t nch = (k + KC - 1) / KC;
    return (size_t)(nch * n) * (sizeof(int32_t) + sizeof(unsigned long long)) + (size_t)n * sizeof(int32_t) + 256;
}

void launch_cols_exponents(const double* B, int64_t k, int64_t n, int64_t ldb, int N, int mode,
                           int kstar, int32_t* f, void* scratch, cudaStream_t st) {
    if (n == 0) return;
    int64_t nch = (k + KC - 1) / KC;
    if (nch == 0) {                       // k == 0: zero columns
        cudaMemsetAsync(f, 0, sizeof(int32_t) * n, st);
        return;
    }
    unsigned long long* Sc = reinterpret_cast<unsigned long long*>(scratch);
    int32_t* Ec = reinterpret_cast<int32_t*>(Sc + nch * n);
    int32_t* bad = Ec + nch * n;
    cudaMemsetAsync(bad, 0, sizeof(int32_t) * n, st);
    dim3 grid((unsigned)((n + 31) / 32), (unsigned)nch);
    if (mode == 0) cols_stats_kernel<0><<<grid, 256, 0, st>>>(B, k, n, ldb, Ec, Sc, bad);
    else cols_stats_kernel<1><<<grid, 256, 0, st>>>(B, k, n, ldb, Ec, Sc, bad);
    unsigned g2 = (unsigned)((n + 255) / 256);
    if (mode == 0) cols_finalize_kernel<0><<<g2, 256, 0, st>>>(Ec, Sc, bad, n, (int)nch, host_T(N), kstar, f);
    else cols_finalize_kernel<1><<<g2, 256, 0, st>>>(Ec, Sc, bad, n, (int)nch, host_T(N), kstar, f);
}

void launch_cols_residues(const double* B, int64_t k, int64_t n, int64_t ldb, const int32_t* f, int N,
                          int8_t* res, int64_t ldr, cudaStream_t st) {
    if (n == 0 || k == 0) return;
    OZ2_DISPATCH_N(N, launch_cols_res_nm, B, k, n, ldb, f, res, ldr, st);
}

void launch_trunc_cols(const double* B, int64_t k, int64_t n, int64_t ldb, const int32_t* f,
                       double* out, cudaStream_t st) {
    int64_t tot = k * n;
    if (!tot) return;
    trunc_cols_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(B, k, n, ldb, f, out);
}

}  // namespace oz2
