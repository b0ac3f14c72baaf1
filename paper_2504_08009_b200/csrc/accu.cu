// accu.cu -- Alg. 1 line 1 by the OS II-accu rule (
// reading R18 in DESIGN.md) on sm_100a:
//   1. E_i = ilogb max_l |a_il| per row of op(A), F_j per column of op(B);
//   2. 7-bit upper approximations ahat = ceil(|a| 2^(6 - E)) in [1, 128] (0 for
//      a = 0), as unsigned int8 K-major planes (rows_hat7 / cols_hat7);
//   3. P = Ahat Bhat^T on the tensor cores (tcgen05 kind::i8, unsigned), whose
//      epilogue keeps only max_j P_ij and max_i P_ij (gemm.cu, NM < 0);
//   4. g = min(G, floor((L + 12 - ceil(log2 max P)) / 2)), e = g - E (accu_finalize).
// Every step is an integer, order-independent operation: the exponents are
// bit-identical to the oracle's for any tiling or reduction order.
#include "oz2_device.cuh"
#include "oz2_kernels.h"

namespace oz2 {

// ceil(|x| 2^(6 - E)) for x != 0 with ilogb|x| <= E, in integer arithmetic:
// |x| = mant 2^ex, so the value is mant >> s rounded up (s = E - 6 - ex),
// clamped below at 1; result in [1, 128]
__device__ __forceinline__ uint32_t hat7(double x, int E) {
    const uint64_t b = (uint64_t)__double_as_longlong(x) & 0x7fffffffffffffffull;
    if (b == 0) return 0;
    const int ef = (int)(b >> 52);
    const uint64_t mant = ef ? ((b & 0xfffffffffffffull) | (1ull << 52)) : b;
    const int ex = ef ? ef - 1075 : -1074;
    const int s = E - 6 - ex;
    uint64_t u;
    if (s >= 64) u = 1;
    else if (s > 0) u = (mant + ((1ull << s) - 1)) >> s;
    else u = mant << (-s);                                     // tiny subnormal row maxima only
    return u ? (uint32_t)u : 1u;
}

__device__ __forceinline__ uint64_t block_max_u64(uint64_t v, uint64_t* red) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    #pragma unroll
    for (int o = 16; o; o >>= 1) {
        const uint64_t w = __shfl_xor_sync(0xffffffffu, v, o);
        v = w > v ? w : v;
    }
    if (lane == 0) red[warp] = v;
    __syncthreads();
    uint64_t r = 0;
    for (int i = 0; i < (int)(blockDim.x >> 5); i++) r = red[i] > r ? red[i] : r;
    return r;
}

// one CTA per row of X (rows x k, ld): E (or the zero / non-finite marker) and
// the row's ahat bytes into hat[row][0..ldr) (zero padded); the second pass
// re-reads the row from L2
__global__ void __launch_bounds__(256)
rows_hat7_kernel(const double* __restrict__ X, int64_t rows, int64_t k, int64_t ld, int32_t* __restrict__ Eout,
                 uint8_t* __restrict__ hat, int64_t ldr) {
    __shared__ uint64_t red[32];
    const int64_t i = blockIdx.x;
    if (i >= rows) return;
    const double* x = X + i * ld;
    // pass 1: the largest |x| bit pattern (orders like |x|; Inf/NaN above every finite)
    uint64_t mb = 0;
    for (int64_t l = threadIdx.x; l < k; l += blockDim.x) {
        const uint64_t b = (uint64_t)__double_as_longlong(x[l]) & 0x7fffffffffffffffull;
        mb = b > mb ? b : mb;
    }
    mb = block_max_u64(mb, red);
    int E;
    if (mb >= 0x7ff0000000000000ull) E = OZ2_EXP_NONFINITE_DEV;
    else if (mb == 0) E = OZ2_EXP_ZERO_DEV;
    else {
        const int ef = (int)(mb >> 52);
        E = ef ? ef - 1023 : (63 - __clzll((long long)mb)) - 1074;
    }
    if (threadIdx.x == 0) Eout[i] = E;
    // pass 2: ahat bytes, 8 per thread per step
    uint8_t* out = hat + i * ldr;
    for (int64_t l0 = 8 * (int64_t)threadIdx.x; l0 < ldr; l0 += 8 * (int64_t)blockDim.x) {
        uint32_t w[2] = {0u, 0u};
        #pragma unroll
        for (int j = 0; j < 8; j++) {
            const int64_t l = l0 + j;
            const uint32_t u = (l < k && E > OZ2_EXP_ZERO_DEV) ? hat7(x[l], E) : 0u;
            w[j >> 2] |= u << (8 * (j & 3));
        }
        *reinterpret_cast<uint2*>(out + l0) = make_uint2(w[0], w[1]);     // ldr % 16 == 0
    }
}

// columns of X (k x cols, ld) -> ahat^T planes hat[col][0..ldr): block = 32
// columns x 64 rows; each thread packs 8 consecutive k of one column (coalesced
// loads across the warp) and the bytes are transposed through shared memory
// into 8-byte pieces of each column's 64-byte segment
__global__ void __launch_bounds__(256)
cols_hat7_kernel(const double* __restrict__ X, int64_t k, int64_t cols, int64_t ld, const int32_t* __restrict__ F,
                 uint8_t* __restrict__ hat, int64_t ldr) {
    __shared__ __align__(16) uint2 s[32][8];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t j0 = (int64_t)blockIdx.x * 32, l0 = (int64_t)blockIdx.y * 64;
    {
        const int64_t j = j0 + lane;
        const int E = j < cols ? F[j] : OZ2_EXP_ZERO_DEV;
        uint32_t w[2] = {0u, 0u};
        #pragma unroll
        for (int q = 0; q < 8; q++) {
            const int64_t l = l0 + warp * 8 + q;
            const uint32_t u = (j < cols && l < k && E > OZ2_EXP_ZERO_DEV) ? hat7(X[l * ld + j], E) : 0u;
            w[q >> 2] |= u << (8 * (q & 3));
        }
        s[lane][warp] = make_uint2(w[0], w[1]);
    }
    __syncthreads();
    const int c = threadIdx.x >> 3, seg = threadIdx.x & 7;        // column, 8-byte segment
    const int64_t l = l0 + seg * 8;
    if (j0 + c < cols && l < ldr) *reinterpret_cast<uint2*>(hat + (j0 + c) * ldr + l) = s[c][seg];
}

// step 4: e = min(G, floor((L + 12 - ceil(log2 Pmax)) / 2)) - E
__global__ void accu_finalize_kernel(const int32_t* __restrict__ E, const uint32_t* __restrict__ Pmax, int64_t cnt,
                                     int L, int G, int32_t* __restrict__ e) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= cnt) return;
    const int Ei = E[i];
    if (Ei == OZ2_EXP_NONFINITE_DEV) { e[i] = OZ2_EXP_NONFINITE_DEV; return; }
    if (Ei == OZ2_EXP_ZERO_DEV) { e[i] = 0; return; }
    const uint32_t p = Pmax[i];
    int g = G;
    if (p) {
        const int lam = p <= 1 ? 0 : 32 - __clz((int)(p - 1));   // ceil(log2 p)
        const int v = L + 12 - lam;
        g = min(G, v >= 0 ? v / 2 : -((-v + 1) / 2));
    }
    e[i] = g - Ei;
}

void launch_rows_hat7(const double* X, int64_t rows, int64_t k, int64_t ld, int32_t* E, uint8_t* hat, int64_t ldr,
                      cudaStream_t st) {
    if (rows <= 0) return;
    (rows_hat7_kernel<<<(unsigned)rows, 256, 0, st>>>(X, rows, k, ld, E, hat, ldr), count_launch());
}

void launch_cols_hat7(const double* X, int64_t k, int64_t cols, int64_t ld, const int32_t* F, uint8_t* hat,
                      int64_t ldr, cudaStream_t st) {
    if (cols <= 0) return;
    dim3 grid((unsigned)((cols + 31) / 32), (unsigned)((ldr + 63) / 64));
    (cols_hat7_kernel<<<grid, 256, 0, st>>>(X, k, cols, ld, F, hat, ldr), count_launch());
}

void launch_accu_finalize(const int32_t* E, const uint32_t* Pmax, int64_t cnt, int N, int32_t* e, cudaStream_t st) {
    if (cnt <= 0) return;
    const int G = N <= 16 ? 61 : 93;
    (accu_finalize_kernel<<<(unsigned)((cnt + 255) / 256), 256, 0, st>>>(E, Pmax, cnt, host_L(N), G, e), count_launch());
}

}  // namespace oz2
