// fp64mod.cu -- the FP64 prime-modulus regime of Ozaki scheme II (PAPER.md:
// 508-557, Sec. 3.2, Eqs. 19-21): C ~= A B with s primes
// m_t < 2^b, b = floor((55 - ceil(log2 k))/2) (reading F1: q m^2 <= 2^55 = 4
// u^-1, Eq. 19; for q = 1024 this is Eq. 21 verbatim), so that every residue
// product A'_t B'_t is EXACT in binary64 (Eq. 20: q (m/2)^2 <= u^-1) and runs
// on the FP64 tensor cores; the CRT reconstructs X exactly in integers and the
// result is written as v binary64 words per entry (reading F3) -- precision
// beyond binary64 (k_A ~ 170 at s = 16).
//
//   line 1   : the OS II-fast rule (reading R4) with this M's T (reading F2),
//              from the K-split statistics kernels (kslice.cu)
//   lines 2-5: fp64mod_residues_kernel -- x = trunc(2^e a) = mant 2^sh exactly,
//              r_t = (mant mod m_t)(2^sh mod m_t) mod m_t, symmetric (Eq. 1),
//              stored as binary64 planes [s][rows][ld] (exact integers)
//   line 6   : cuBLAS DGEMM, strided-batched over the s moduli (a plain library
//              GEMM of exact integer-valued operands)
//   lines 7-10: fp64mod_crt_kernel -- c''_t = C'_t mod m_t, S = sum c''_t w_t
//              in 32-bit limbs, X = S - M round(S/M) exactly, v words of
//              2^-(e+f) X, each the nearest binary64 to the remaining integer
#include "oz2_device.cuh"
#include "oz2_kernels.h"

#include <dlfcn.h>

#include <mutex>
#include <vector>

namespace oz2 {

// per (s, q) constants, passed to the kernels by value
struct F64Tab {
    int s, nw;                       // moduli; 32-bit words of M (and of every w_t)
    int L, T;
    int64_t m[F64_MAX_S];
    double md[F64_MAX_S], minv[F64_MAX_S];
    uint32_t w[F64_MAX_S][F64_MAX_W];   // w_t = M y_t / m_t, little-endian words
    uint32_t M[F64_MAX_W];
    uint32_t Mh[F64_MAX_W];             // floor(M / 2)
    double Mtop;                        // the top two words of M as a double (quotient estimate)
};

// ---------------------------------------------------------------------------
// host: primes, M, y_t, w_t (little big-integer helpers on 32-bit words)
// ---------------------------------------------------------------------------
static bool is_prime_u64(uint64_t v) {
    if (v < 2) return false;
    for (uint64_t d = 2; d * d <= v; d++)
        if (v % d == 0) return false;
    return true;
}

int f64_prime_bits(int64_t q) {
    int lq = 0;
    while (((int64_t)1 << lq) < q) lq++;
    return (55 - lq) / 2;
}

static void big_mul_small(std::vector<uint32_t>& a, uint64_t s) {
    uint64_t carry = 0;
    for (auto& x : a) {
        const unsigned __int128 p = (unsigned __int128)x * s + carry;
        x = (uint32_t)p;
        carry = (uint64_t)(p >> 32);
    }
    while (carry) { a.push_back((uint32_t)carry); carry >>= 32; }
}
static uint64_t big_divmod_small(std::vector<uint32_t>& a, uint64_t d) {   // a /= d, returns a mod d
    unsigned __int128 r = 0;
    for (int i = (int)a.size() - 1; i >= 0; i--) {
        r = (r << 32) | a[i];
        a[i] = (uint32_t)(r / d);
        r %= d;
    }
    while (a.size() > 1 && a.back() == 0) a.pop_back();
    return (uint64_t)r;
}
static int big_bitlen(const std::vector<uint32_t>& a) {
    for (int i = (int)a.size() - 1; i >= 0; i--)
        if (a[i]) return 32 * i + 32 - __builtin_clz(a[i]);
    return 0;
}

static int build_f64tab(int s, int64_t q, F64Tab* T) {
    if (s < 2 || s > F64_MAX_S || q < 1) return -1;
    *T = F64Tab{};
    T->s = s;
    const int b = f64_prime_bits(q);
    uint64_t v = ((uint64_t)1 << b) - 1;
    for (int t = 0; t < s; v--) {
        if (v < 3) return -1;
        if (is_prime_u64(v)) T->m[t++] = (int64_t)v;
    }
    std::vector<uint32_t> M{1};
    for (int t = 0; t < s; t++) big_mul_small(M, (uint64_t)T->m[t]);
    const int nw = (int)M.size() + 1;                    // one spare word: w_t < M
    if (nw > F64_MAX_W) return -1;
    T->nw = nw;
    for (int i = 0; i < (int)M.size(); i++) T->M[i] = M[i];
    std::vector<uint32_t> Mh = M;
    {   // floor(M / 2)
        uint32_t carry = 0;
        for (int i = (int)Mh.size() - 1; i >= 0; i--) {
            const uint32_t x = Mh[i];
            Mh[i] = (x >> 1) | (carry << 31);
            carry = x & 1;
        }
    }
    for (int i = 0; i < (int)Mh.size(); i++) T->Mh[i] = Mh[i];
    // L = floor(log2(M/2 - 1)) = bitlen(floor(M/2) - 1) - 1 (M odd), T = floor(L/2)
    {
        std::vector<uint32_t> x = Mh;
        for (auto& w : x) { if (w--) break; }           // floor(M/2) - 1 (no underflow: M >> 2)
        T->L = big_bitlen(x) - 1;
        T->T = T->L / 2;
    }
    for (int t = 0; t < s; t++) {
        const uint64_t mt = (uint64_t)T->m[t];
        std::vector<uint32_t> Mt = M;
        big_divmod_small(Mt, mt);                        // M_t = M / m_t (exact)
        std::vector<uint32_t> tmp = Mt;
        const uint64_t a = big_divmod_small(tmp, mt);    // M_t mod m_t
        // y_t = a^-1 mod m_t (extended Euclid), least positive (reading R2)
        int64_t old_r = (int64_t)a, r = (int64_t)mt, old_s = 1, ss = 0;
        while (r) {
            const int64_t quo = old_r / r;
            int64_t x = old_r - quo * r; old_r = r; r = x;
            x = old_s - quo * ss; old_s = ss; ss = x;
        }
        if (old_r != 1) return -1;
        const uint64_t y = (uint64_t)(((old_s % (int64_t)mt) + (int64_t)mt) % (int64_t)mt);
        big_mul_small(Mt, y);
        for (int i = 0; i < (int)Mt.size() && i < F64_MAX_W; i++) T->w[t][i] = Mt[i];
        T->md[t] = (double)T->m[t];
        T->minv[t] = 1.0 / (double)T->m[t];
    }
    const int top = (int)M.size() - 1;
    T->Mtop = (double)M[top] * 4294967296.0 + (top >= 1 ? (double)M[top - 1] : 0.0);
    return 0;
}

// ---------------------------------------------------------------------------
// lines 2-5: residue planes (binary64), rows of A (is_cols = 0: element (i, l),
// exponent e[i]) or columns of B (is_cols = 1: element (l, j), exponent e[j]),
// the plane keeps the operand's own row-major layout [s][R][C] with ld = C
// ---------------------------------------------------------------------------
// a mod m for 0 <= a < 2^53 (doubles holding integers, m < 2^23): the quotient
// estimate is within one, the fma remainder exact
__device__ __forceinline__ double mod_small(double a, double m, double minv) {
    const double q = floor(a * minv);
    double r = fma(-q, m, a);
    if (r < 0) r += m;
    if (r >= m) r -= m;
    return r;
}

// reading F6 (double-word inputs, Eqs. 22-23): for x1 = 2^e a1, x2 = 2^e a2
// with |x2| <= u |x1|, trunc(x1 + x2) = trunc(x1) + adj, where f1 = x1 -
// trunc(x1) is exact, (s, t) = TwoSum(f1, x2) is the exact sum f1 + x2, and adj
// = floor(s + t) (x1 > 0) or ceil(s + t) (x1 < 0), in {-2, ..., 1} / {-1, ..., 2};
// a scaled second word below 2^-64 acts only through its sign (+-2^-64)
__device__ __forceinline__ double trunc_adj_mw(double x1, double x2) {
    if (x2 != 0.0 && fabs(x2) < 0x1p-64) x2 = copysign(0x1p-64, x2);
    const double f1 = x1 - trunc(x1);
    const double s = f1 + x2, bb = s - f1, t = (f1 - (s - bb)) + (x2 - bb);
    if (x1 > 0.0) return floor(s) - ((s == floor(s) && t < 0.0) ? 1.0 : 0.0);
    if (x1 < 0.0) return ceil(s) + ((s == ceil(s) && t > 0.0) ? 1.0 : 0.0);
    return 0.0;
}

// |a1| + |a2| rounded upward (line 1 of double-word inputs, reading F6), into a
// packed R x C matrix
__global__ void __launch_bounds__(256)
fp64mod_abs_sum_up_kernel(const double* __restrict__ X, const double* __restrict__ X2, int64_t R, int64_t Cc,
                          int64_t ld, double* __restrict__ out) {
    const int64_t total = R * Cc;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = idx / Cc, c = idx % Cc;
        out[idx] = __dadd_ru(fabs(X[r * ld + c]), fabs(X2[r * ld + c]));
    }
}

__global__ void __launch_bounds__(256)
fp64mod_residues_kernel(const double* __restrict__ X, const double* __restrict__ X2, int64_t R, int64_t Cc,
                        int64_t ld, int is_cols, const int32_t* __restrict__ ex,
                        const uint32_t* __restrict__ pow2tab, double* __restrict__ out,
                        const __grid_constant__ F64Tab T) {
    // 2^j mod m_t for j < F64_POW2 (host table): |x| < 2^(T + 1), x = mant 2^sh, sh <= T - 52
    __shared__ float p2[F64_MAX_S][F64_POW2];            // values < 2^22: exact in binary32
    for (int x = threadIdx.x; x < T.s * F64_POW2; x += blockDim.x)
        p2[x / F64_POW2][x % F64_POW2] = (float)pow2tab[x];
    __syncthreads();
    const int64_t total = R * Cc, plane = R * Cc;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = idx / Cc, c = idx % Cc;
        const int e = ex[is_cols ? c : r];
        double x = 0.0, adj = 0.0;
        if (e != OZ2_EXP_NONFINITE_DEV) {
            const double x1 = scale_pow2(X[r * ld + c], e);
            x = trunc(x1);                                              // Alg. 1 lines 2-3
            if (X2) adj = trunc_adj_mw(x1, scale_pow2(X2[r * ld + c], e));
        }
        // residues of the integral doubles x (and adj, reading F6: adj may be as large
        // as u |x1|) from |v| = mant 2^sh, mant < 2^53 an integer (sh = 0 when |v| < 2^53)
        #pragma unroll 1
        for (int t = 0; t < T.s; t++) {
            const double mt = T.md[t], mi = T.minv[t];
            double rr = 0.0;
            #pragma unroll
            for (int part = 0; part < 2; part++) {
                const double vv = part == 0 ? x : adj;
                if (vv == 0.0) continue;
                const uint64_t bits = (uint64_t)__double_as_longlong(vv);
                const int bexp = (int)((bits >> 52) & 0x7ff);
                double mant;
                int sh;
                if (bexp >= 1023 + 53) {
                    mant = (double)((bits & 0xfffffffffffffull) | (1ull << 52));
                    sh = bexp - 1075;
                } else {
                    mant = fabs(vv);
                    sh = 0;
                }
                double r = mod_small(mod_small(mant, mt, mi) * (double)p2[t][sh], mt, mi);   // |v| mod m_t
                if (vv < 0.0 && r != 0.0) r = mt - r;                                       // v mod m_t
                rr = mod_small(rr + r, mt, mi);
            }
            out[(int64_t)t * plane + idx] = rr > 0.5 * (mt - 1.0) ? rr - mt : rr;        // Eq. (1), m_t odd
        }
    }
}

// ---------------------------------------------------------------------------
// lines 7-10
// ---------------------------------------------------------------------------
// nearest binary64 to the signed integer X (NW 32-bit words, two's complement),
// and X -= that value (exact); the power-of-two scaling is applied by the caller
template <int NW>
__device__ __forceinline__ double take_word(uint32_t (&X)[NW]) {
    const bool neg = (int32_t)X[NW - 1] < 0;
    uint32_t a[NW];
    if (neg) {
        uint64_t c = 1;
        #pragma unroll
        for (int i = 0; i < NW; i++) { c += (uint64_t)(~X[i]); a[i] = (uint32_t)c; c >>= 32; }
    } else {
        #pragma unroll
        for (int i = 0; i < NW; i++) a[i] = X[i];
    }
    int top = -1;
    #pragma unroll
    for (int i = 0; i < NW; i++) if (a[i]) top = i;
    if (top < 0) return 0.0;
    const int bl = 32 * top + 32 - __clz(a[top]);
    double v;
    uint32_t q[NW];                                      // |value taken| in words
    #pragma unroll
    for (int i = 0; i < NW; i++) q[i] = 0;
    if (bl <= 53) {
        uint64_t x = a[0];
        if (NW > 1) x |= (uint64_t)a[1] << 32;
        v = (double)x;                                   // exact
        q[0] = a[0];
        if (NW > 1) q[1] = a[1];
    } else {
        const int drop = bl - 53;                        // keep bits [drop, bl)
        // the 53 kept bits, the round bit and the sticky bits below it
        uint64_t keep = 0;
        #pragma unroll
        for (int i = 0; i < NW; i++) {
            const int lo = 32 * i;                       // bit position of a[i]'s bit 0
            if (lo + 32 <= drop || lo >= bl) continue;
            const int s = lo - drop;
            keep |= s >= 0 ? (uint64_t)a[i] << s : (uint64_t)a[i] >> (-s);
        }
        keep &= (1ull << 53) - 1;
        keep |= 1ull << 52;
        const int rb = drop - 1;
        const bool round = (a[rb >> 5] >> (rb & 31)) & 1;
        bool sticky = false;
        #pragma unroll
        for (int i = 0; i < NW; i++) {
            const int lo = 32 * i;
            if (lo >= rb) continue;
            const uint32_t mask = lo + 32 <= rb ? 0xffffffffu : ((1u << (rb - lo)) - 1);
            sticky |= (a[i] & mask) != 0;
        }
        uint64_t qm = keep + ((round && (sticky || (keep & 1))) ? 1 : 0);
        int qe = drop;
        if (qm >> 53) { qm >>= 1; qe++; }                // carried into 2^53
        v = ldexp((double)qm, qe);
        // q = qm << qe as words
        #pragma unroll
        for (int i = 0; i < NW; i++) {
            const int lo = 32 * i;
            const int s = lo - qe;                       // word i holds bits s.. of qm
            uint32_t w = 0;
            if (s >= 0 && s < 64) w = (uint32_t)(qm >> s);
            else if (s < 0 && s > -32) w = (uint32_t)(qm << (-s));
            q[i] = w;
        }
    }
    // X -= +-q
    if (neg) {
        uint64_t c = 0;
        #pragma unroll
        for (int i = 0; i < NW; i++) { c += (uint64_t)X[i] + q[i]; X[i] = (uint32_t)c; c >>= 32; }
    } else {
        int64_t c = 0;
        #pragma unroll
        for (int i = 0; i < NW; i++) { c += (int64_t)X[i] - (int64_t)q[i]; X[i] = (uint32_t)c; c >>= 32; }
    }
    return neg ? -v : v;
}

template <int NW>
__global__ void __launch_bounds__(128)
fp64mod_crt_kernel(const double* __restrict__ Cp, int64_t m, int64_t n, const int32_t* __restrict__ e,
                   const int32_t* __restrict__ f, int v, double* __restrict__ C, int64_t ldc, int64_t strideC,
                   const __grid_constant__ F64Tab T) {
    const int64_t total = m * n;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = idx / n, j = idx % n;
        // line 8: S = sum_t c''_t w_t, 64-bit column sums of 22-bit x 32-bit products
        uint64_t acc[NW];
        #pragma unroll
        for (int w = 0; w < NW; w++) acc[w] = 0;
        for (int t = 0; t < T.s; t++) {
            const double c = Cp[(int64_t)t * total + idx];          // exact integer, |c| <= 2^53
            double q = floor(c * T.minv[t]);
            double r = fma(-q, T.md[t], c);                          // exact
            if (r < 0) r += T.md[t];
            if (r >= T.md[t]) r -= T.md[t];                          // line 7: c'' in [0, m_t)
            const uint64_t cc = (uint64_t)r;
            #pragma unroll
            for (int w = 0; w < NW; w++) acc[w] += cc * T.w[t][w];
        }
        uint32_t S[NW];
        {
            uint64_t carry = 0;
            #pragma unroll
            for (int w = 0; w < NW; w++) { const uint64_t x = acc[w] + carry; S[w] = (uint32_t)x; carry = x >> 32; }
        }
        // line 9: X = S - M round(S / M); Q from the top words (within +-1), then exact corrections
        const int tw = T.nw - 2;                                     // the top word of M
        double stop = 0.0;
        #pragma unroll
        for (int w = 0; w < NW; w++) {
            if (w == tw + 1) stop += (double)S[w] * 18446744073709551616.0;
            if (w == tw) stop += (double)S[w] * 4294967296.0;
            if (w == tw - 1) stop += (double)S[w];
        }
        const uint32_t Q = (uint32_t)floor(stop / T.Mtop + 0.5);
        uint32_t X[NW];
        {
            uint64_t borrow = 0, carry = 0;
            #pragma unroll
            for (int w = 0; w < NW; w++) {
                const uint64_t p = (uint64_t)Q * T.M[w] + carry;     // Q M, word w
                carry = p >> 32;
                const int64_t d = (int64_t)S[w] - (int64_t)(uint32_t)p - (int64_t)borrow;
                X[w] = (uint32_t)d;
                borrow = d < 0 ? 1 : 0;
            }
        }
        // into [-M/2, M/2): X >= M/2 (> floor(M/2) for odd M) -> X -= M; X < -M/2 -> X += M
        for (int it = 0; it < 2; it++) {
            const bool neg = (int32_t)X[NW - 1] < 0;
            int cmp = 0;                                             // |X| vs floor(M/2)
            uint32_t a[NW];
            if (neg) {
                uint64_t c = 1;
                #pragma unroll
                for (int w = 0; w < NW; w++) { c += (uint64_t)(~X[w]); a[w] = (uint32_t)c; c >>= 32; }
            } else {
                #pragma unroll
                for (int w = 0; w < NW; w++) a[w] = X[w];
            }
            #pragma unroll
            for (int w = NW - 1; w >= 0; w--)
                if (cmp == 0 && a[w] != T.Mh[w]) cmp = a[w] > T.Mh[w] ? 1 : -1;
            if (cmp <= 0) break;                                     // |X| <= floor(M/2) = (M-1)/2
            if (neg) {
                uint64_t c = 0;
                #pragma unroll
                for (int w = 0; w < NW; w++) { c += (uint64_t)X[w] + T.M[w]; X[w] = (uint32_t)c; c >>= 32; }
            } else {
                int64_t c = 0;
                #pragma unroll
                for (int w = 0; w < NW; w++) { c += (int64_t)X[w] - (int64_t)T.M[w]; X[w] = (uint32_t)c; c >>= 32; }
            }
        }
        // line 10 + reading F3: v words of 2^-(e_i + f_j) X
        const int ei = e[i], fj = f[j];
        double* out = C + i * ldc + j;
        for (int w = 0; w < v; w++) {
            double word = take_word<NW>(X);
            if (ei == OZ2_EXP_NONFINITE_DEV || fj == OZ2_EXP_NONFINITE_DEV) word = __longlong_as_double(0x7ff8000000000000ll);
            else word = scale_pow2(word, -(ei + fj));
            out[(int64_t)w * strideC] = word;
        }
    }
}

// ---------------------------------------------------------------------------
// cuBLAS DGEMM (dlopen'd: the library loads without cuBLAS; only this regime needs it)
// ---------------------------------------------------------------------------
typedef int (*cublasCreate_t)(void**);
typedef int (*cublasSetStream_t)(void*, cudaStream_t);
typedef int (*cublasDgemmSB_t)(void*, int, int, int, int, int, const double*, const double*, int, long long,
                               const double*, int, long long, const double*, double*, int, long long, int);
static std::mutex g_cublas_mu;
static void* g_cublas_lib = nullptr;
static cublasCreate_t p_create = nullptr;
static cublasSetStream_t p_setstream = nullptr;
static cublasDgemmSB_t p_dgemm_sb = nullptr;
static void* g_cublas_h[64] = {nullptr};

static int cublas_ready(int dev) {
    std::lock_guard<std::mutex> lk(g_cublas_mu);
    if (!g_cublas_lib) {
        const char* names[] = {"libcublas.so.12", "libcublas.so", "/usr/local/cuda/lib64/libcublas.so.12"};
        for (const char* nm : names)
            if ((g_cublas_lib = dlopen(nm, RTLD_NOW | RTLD_GLOBAL))) break;
        if (!g_cublas_lib) return -1;
        p_create = (cublasCreate_t)dlsym(g_cublas_lib, "cublasCreate_v2");
        p_setstream = (cublasSetStream_t)dlsym(g_cublas_lib, "cublasSetStream_v2");
        p_dgemm_sb = (cublasDgemmSB_t)dlsym(g_cublas_lib, "cublasDgemmStridedBatched");
        if (!p_create || !p_setstream || !p_dgemm_sb) return -1;
    }
    if (dev < 0 || dev >= 64) return -1;
    if (!g_cublas_h[dev] && p_create(&g_cublas_h[dev]) != 0) return -1;
    return 0;
}

// ---------------------------------------------------------------------------
// launcher
// ---------------------------------------------------------------------------
static std::mutex g_tab_mu;

int f64_tables(int s, int64_t q, int64_t* moduli, uint32_t* M_words, int32_t* L, int32_t* Tt) {
    F64Tab T;
    if (build_f64tab(s, q, &T)) return -1;
    for (int t = 0; t < s; t++) if (moduli) moduli[t] = T.m[t];
    if (M_words) for (int w = 0; w < F64_MAX_W; w++) M_words[w] = T.M[w];
    if (L) *L = T.L;
    if (Tt) *Tt = T.T;
    return 0;
}

size_t f64_workspace_bytes(int64_t m, int64_t n, int64_t k, int s) {
    auto r = [](size_t b) { return (b + 255) / 256 * 256; };
    return r((size_t)s * 8 * (size_t)(m * k)) + r((size_t)s * 8 * (size_t)(k * n)) + r((size_t)s * 8 * (size_t)(m * n)) +
           r(8 * (size_t)(m * k)) + r(8 * (size_t)(k * n)) +                     // double-word bounds (F6)
           2 * r(4 * (size_t)(m > 0 ? m : 1)) + 2 * r(4 * (size_t)(n > 0 ? n : 1)) + r(8 * (size_t)(m > 0 ? m : 1)) +
           r(8 * (size_t)(n > 0 ? n : 1)) + r(cols_stats_bytes(k, n)) + r(4 * (size_t)s * F64_POW2) + 256;
}

template <int NW>
static void launch_crt_nw(const double* Cp, int64_t m, int64_t n, const int32_t* e, const int32_t* f, int v,
                          double* C, int64_t ldc, int64_t strideC, const F64Tab& T, cudaStream_t st) {
    const int64_t total = m * n;
    const unsigned g = (unsigned)std::min<int64_t>((total + 127) / 128, 148 * 16);
    (fp64mod_crt_kernel<NW><<<g, 128, 0, st>>>(Cp, m, n, e, f, v, C, ldc, strideC, T), count_launch());
}

int launch_fp64mod(int device, const double* A, const double* A2, int64_t m, int64_t k, int64_t lda,
                   const double* B, const double* B2, int64_t n, int64_t ldb, int s, int v, double* C, int64_t ldc,
                   int64_t strideC, uint8_t* ws, cudaStream_t st) {
    F64Tab T;
    if (build_f64tab(s, k, &T)) return -1;
    if (cublas_ready(device)) return -2;
    // 2^j mod m_t, j < F64_POW2 (host, exact integer arithmetic)
    std::vector<uint32_t> pow2tab((size_t)s * F64_POW2);
    for (int t = 0; t < s; t++) {
        uint64_t r = 1;
        for (int j = 0; j < F64_POW2; j++) { pow2tab[(size_t)t * F64_POW2 + j] = (uint32_t)r; r = (r * 2) % (uint64_t)T.m[t]; }
    }
    uint8_t* p = ws;
    auto take = [&](size_t bytes) { uint8_t* q = p; p += (bytes + 255) / 256 * 256; return q; };
    double* Ares = (double*)take(sizeof(double) * (size_t)s * m * k);
    double* Bres = (double*)take(sizeof(double) * (size_t)s * k * n);
    double* Cp = (double*)take(sizeof(double) * (size_t)s * m * n);
    int32_t* e = (int32_t*)take(sizeof(int32_t) * (size_t)(m > 0 ? m : 1));
    int32_t* f = (int32_t*)take(sizeof(int32_t) * (size_t)(n > 0 ? n : 1));
    int32_t* EA = (int32_t*)take(sizeof(int32_t) * (size_t)(m > 0 ? m : 1));
    int32_t* EB = (int32_t*)take(sizeof(int32_t) * (size_t)(n > 0 ? n : 1));
    unsigned long long* SA = (unsigned long long*)take(8 * (size_t)(m > 0 ? m : 1));
    unsigned long long* SB = (unsigned long long*)take(8 * (size_t)(n > 0 ? n : 1));
    void* stats = take(cols_stats_bytes(k, n));
    uint32_t* p2d = (uint32_t*)take(sizeof(uint32_t) * pow2tab.size());
    double* Abar = A2 ? (double*)take(sizeof(double) * (size_t)m * k) : nullptr;
    double* Bbar = B2 ? (double*)take(sizeof(double) * (size_t)k * n) : nullptr;
    if (cudaMemcpyAsync(p2d, pow2tab.data(), sizeof(uint32_t) * pow2tab.size(), cudaMemcpyHostToDevice, st) !=
        cudaSuccess)
        return -4;
    // line 1 (reading F2): FAST statistics (phase 1: max chunk exponents; phase 2: sums), then e, f with T;
    // double-word inputs (F6): the statistics of |x1| + |x2| rounded up
    const double* As = A;
    int64_t ldas = lda;
    const double* Bs = B;
    int64_t ldbs = ldb;
    if (A2) {
        const unsigned g = (unsigned)std::max<int64_t>(1, std::min<int64_t>((m * k + 255) / 256, 148 * 8));
        (fp64mod_abs_sum_up_kernel<<<g, 256, 0, st>>>(A, A2, m, k, lda, Abar), count_launch());
        As = Abar; ldas = k;
    }
    if (B2) {
        const unsigned g = (unsigned)std::max<int64_t>(1, std::min<int64_t>((k * n + 255) / 256, 148 * 8));
        (fp64mod_abs_sum_up_kernel<<<g, 256, 0, st>>>(B, B2, k, n, ldb, Bbar), count_launch());
        Bs = Bbar; ldbs = n;
    }
    launch_kslice_rows(As, m, k, ldas, 0, nullptr, EA, nullptr, st);
    launch_kslice_rows(As, m, k, ldas, 0, EA, nullptr, SA, st);
    launch_kslice_cols(Bs, k, n, ldbs, 0, nullptr, EB, nullptr, stats, st);
    launch_kslice_cols(Bs, k, n, ldbs, 0, EB, nullptr, SB, stats, st);
    launch_exponents_T(EA, SA, m, T.T, e, st);
    launch_exponents_T(EB, SB, n, T.T, f, st);
    // lines 2-5
    {
        const unsigned g = (unsigned)std::max<int64_t>(1, std::min<int64_t>((m * k + 255) / 256, 148 * 8));
        (fp64mod_residues_kernel<<<g, 256, 0, st>>>(A, A2, m, k, lda, 0, e, p2d, Ares, T), count_launch());
        const unsigned g2 = (unsigned)std::max<int64_t>(1, std::min<int64_t>((k * n + 255) / 256, 148 * 8));
        (fp64mod_residues_kernel<<<g2, 256, 0, st>>>(B, B2, k, n, ldb, 1, f, p2d, Bres, T), count_launch());
    }
    // line 6: C'_t = A'_t B'_t on the FP64 tensor cores, exact (Eq. 20); row-major
    // C (m x n) = A B  <=>  column-major C^T = B^T A^T
    {
        std::lock_guard<std::mutex> lk(g_cublas_mu);
        void* hb = g_cublas_h[device];
        p_setstream(hb, st);
        const double one = 1.0, zero = 0.0;
        if (p_dgemm_sb(hb, 0, 0, (int)n, (int)m, (int)k, &one, Bres, (int)n, (long long)(k * n), Ares, (int)k,
                       (long long)(m * k), &zero, Cp, (int)n, (long long)(m * n), s) != 0)
            return -3;
    }
    // lines 7-10
    if (T.nw <= 6) launch_crt_nw<6>(Cp, m, n, e, f, v, C, ldc, strideC, T, st);   // word count >= T.nw
    else if (T.nw <= 9) launch_crt_nw<9>(Cp, m, n, e, f, v, C, ldc, strideC, T, st);
    else if (T.nw <= 12) launch_crt_nw<12>(Cp, m, n, e, f, v, C, ldc, strideC, T, st);
    else if (T.nw <= 15) launch_crt_nw<15>(Cp, m, n, e, f, v, C, ldc, strideC, T, st);
    else launch_crt_nw<F64_MAX_W>(Cp, m, n, e, f, v, C, ldc, strideC, T, st);
    return 0;
}

}  // namespace oz2
