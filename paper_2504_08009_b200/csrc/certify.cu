// certify.cu -- a certificate of the uniqueness condition (13) for
// caller-supplied line-1 exponents ("If 2 c_max < M is
// satisfied, we can find the matrix X ... If M is smaller than or equal to
// 2 c_max, we may find multiple candidates of the result").
//
// The OS II-fast exponents e^F (reading R4) guarantee ||2^{e^F_i} a_i||_2 <= 2^T
// for every row of A (and the same for the columns of B), and truncation only
// shrinks magnitudes, so for any exponents e, f:
//   (|A'||B'|)_ij <= ||a'_i||_2 ||b'_j||_2 <= 2^{(e_i - e^F_i) + T} 2^{(f_j - f^F_j) + T}
// by Cauchy-Schwarz.  beta = max_i (e_i - e^F_i) + max_j (f_j - f^F_j) + 2T is
// therefore a bound c_max <= 2^beta, and beta <= L (2^L <= M/2 - 1) certifies
// (13).  For k < 2^17 the OS II-accu bound (certify_p_kernel) is formed too and
// the smaller of the two is reported.  A sufficient condition only.  Exponents
// under which some |trunc(2^e a)| would not fit the residue kernels' integers
// (63 bits for N <= 16, 95 bits otherwise) give beta = INT32_MAX (refused).  Rows / columns that are zero or
// hold Inf/NaN, and rows / columns whose caller exponent is the non-finite
// sentinel, do not take part (their entries of C are 0 or NaN by construction).
#include "oz2_device.cuh"
#include "oz2_kernels.h"

namespace oz2 {

__device__ __forceinline__ int clamp_i32(long long v) {
    return v > INT32_MAX ? INT32_MAX : (v < INT32_MIN + 2 ? INT32_MIN + 2 : (int)v);
}

// one CTA per row of A: the FAST statistics (one pass), then
// atomicMax(dmax, e_i - e^F_i) for a row that takes part
__global__ void __launch_bounds__(256)
certify_rows_kernel(const double* __restrict__ A, int64_t m, int64_t k, int64_t lda, const int32_t* __restrict__ e,
                    int Tb, int width, int* __restrict__ dmax, int* __restrict__ wflag) {
    extern __shared__ __align__(16) unsigned char row_smem[];
    const int64_t i = blockIdx.x;
    if (i >= m) return;
    const int64_t nch = (k + KC - 1) / KC;
    RowSmem sm;
    sm.Sc = reinterpret_cast<unsigned long long*>(row_smem);
    sm.Ec = reinterpret_cast<int*>(row_smem + sizeof(unsigned long long) * (nch > 0 ? nch : 1));
    sm.misc = sm.Ec + (nch > 0 ? nch : 1);
    row_chunk_stats<0>(A + i * lda, k, sm);
    if (threadIdx.x >= 32) return;
    const int lane = threadIdx.x;
    int E = INT32_MIN;
    for (int c = lane; c < (int)nch; c += 32) E = max(E, sm.Ec[c]);
    E = warp_max(E);
    if (E == INT32_MIN || sm.misc[0]) return;             // zero row / Inf or NaN in the row
    uint64_t S = 0;
    for (int c = lane; c < (int)nch; c += 32)
        if (sm.Ec[c] != INT32_MIN) S += ceil_shift(sm.Sc[c], 2 * (E - sm.Ec[c]));
    S = warp_sum64(S);
    const int ei = e[i];
    if (lane == 0 && ei != OZ2_EXP_NONFINITE_DEV) {
        const long long eF = (long long)Tb + 15 - E - log4_ceil(S);
        atomicMax(dmax, clamp_i32((long long)ei - eF));
        if ((long long)ei + E + 1 > width) atomicOr(wflag, 1);     // |a'| < 2^(e + E + 1) must fit
    }
}

// columns: per-chunk statistics from cols_stats_kernel ([nch][n])
__global__ void certify_cols_kernel(const int32_t* __restrict__ Ec, const unsigned long long* __restrict__ Sc,
                                    const int32_t* __restrict__ bad, int64_t n, int nch,
                                    const int32_t* __restrict__ f, int Tb, int width, int* __restrict__ dmax,
                                    int* __restrict__ wflag) {
    const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (j >= n) return;
    int E = INT32_MIN;
    for (int c = 0; c < nch; c++) E = max(E, Ec[(int64_t)c * n + j]);
    if (E == INT32_MIN || bad[j] || f[j] == OZ2_EXP_NONFINITE_DEV) return;
    uint64_t S = 0;
    for (int c = 0; c < nch; c++) {
        const int x = Ec[(int64_t)c * n + j];
        if (x != INT32_MIN) S += ceil_shift(Sc[(int64_t)c * n + j], 2 * (E - x));
    }
    const long long fF = (long long)Tb + 15 - E - log4_ceil(S);
    atomicMax(dmax, clamp_i32((long long)f[j] - fF));
    if ((long long)f[j] + E + 1 > width) atomicOr(wflag, 1);
}

// the OS II-accu bound (reading R18): with E_i = max ilogb |a_il|, the 7-bit
// approximations give (|A||B|)_ij <= P_ij 2^(E_i + F_j - 12), P = Ahat Bhat^T, and
// P_ij <= sqrt(R_i C_j) with the row / column maxima R, C of P; so for g_i =
// e_i + E_i, h_j = f_j + F_j:
//   (|A'||B'|)_ij <= 2^((2 g_i - 12 + lambda_i) / 2 + (2 h_j - 12 + mu_j) / 2),
// lambda = ceil(log2 R), mu = ceil(log2 C).  dmax2[0] = max over the rows of
// 2 g_i - 12 + lambda_i (dmax2[1]: columns).  The accu rule's own exponents
// satisfy each term <= L by construction, which the
// Cauchy-Schwarz bound above does not always certify.
__global__ void certify_p_kernel(const int32_t* __restrict__ E, const uint32_t* __restrict__ Pmax,
                                 const int32_t* __restrict__ e, int64_t cnt, int* __restrict__ dmax) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= cnt) return;
    const int Ei = E[i];
    const uint32_t p = Pmax[i];
    if (Ei == OZ2_EXP_NONFINITE_DEV || Ei == OZ2_EXP_ZERO_DEV || p == 0 || e[i] == OZ2_EXP_NONFINITE_DEV) return;
    const int lam = p <= 1 ? 0 : 32 - __clz((int)(p - 1));              // ceil(log2 p)
    atomicMax(dmax, clamp_i32(2LL * ((long long)e[i] + Ei) - 12 + lam));
}

// beta = min(beta_CS, beta_P): beta_CS = dmax[0] + dmax[1] + 2T, beta_P =
// ceil((dmax[2] + dmax[3]) / 2) (when computed); INT32_MIN if no row or no
// column takes part.  Either is an upper bound of log2 c_max.
__global__ void certify_finalize_kernel(const int* __restrict__ dmax, int Tb, int with_p, int32_t* __restrict__ beta) {
    if (dmax[4]) { *beta = INT32_MAX; return; }            // a scaled entry exceeds the kernels' integers
    const int a = dmax[0], b = dmax[1];
    if (a == INT32_MIN || b == INT32_MIN) { *beta = INT32_MIN; return; }
    long long bt = (long long)a + b + 2LL * Tb;
    if (with_p) {
        const int c = dmax[2], d = dmax[3];
        if (c != INT32_MIN && d != INT32_MIN) {
            const long long s = (long long)c + d;
            const long long bp = s >= 0 ? (s + 1) / 2 : -((-s) / 2);     // ceil(s / 2)
            bt = bp < bt ? bp : bt;
        }
    }
    *beta = clamp_i32(bt);
}

// refusal (the error behaviour of the certified calls): when beta > L every
// entry of C becomes NaN -- no silently wrong candidate leaves the library --
// and the handle's sticky status word records OZ2_ERR_NOT_UNIQUE
__global__ void refuse_kernel(const int32_t* __restrict__ beta, int L, double* __restrict__ C, int64_t m, int64_t n,
                              int64_t ldc, int* __restrict__ status) {
    const int b = *beta;
    if (b == INT32_MIN || b <= L) return;
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicOr(status, 1);
    const double nan = __longlong_as_double(0x7ff8000000000000ll);
    const int64_t tot = m * n;
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < tot; x += (int64_t)gridDim.x * blockDim.x)
        C[(x / n) * ldc + x % n] = nan;
}

__global__ void certify_init_kernel(int* __restrict__ dmax) {
    if (threadIdx.x < 4) dmax[threadIdx.x] = INT32_MIN;
    if (threadIdx.x == 4) dmax[4] = 0;
}

void launch_certify(const double* A, int64_t m, int64_t k, int64_t lda, const double* B, int64_t n, int64_t ldb,
                    const int32_t* e, const int32_t* f, int N, int* dmax4, void* stats_scratch, int32_t* beta,
                    const AccuBound* ab, cudaStream_t st) {
    const int Tb = host_T(N);
    // the residue kernels hold trunc(2^e a) in 63 (N <= 16) or 95 bits (scale.cu BW_8 / BW_12)
    const int width = N <= 16 ? 63 : 95;
    int* dmax2 = dmax4;
    (certify_init_kernel<<<1, 32, 0, st>>>(dmax4), count_launch());
    if (m > 0 && k > 0) {
        const size_t smem = row_smem_bytes(k);
        if (smem > 48 * 1024) cudaFuncSetAttribute(certify_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        (certify_rows_kernel<<<(unsigned)m, 256, smem, st>>>(A, m, k, lda, e, Tb, width, dmax2, dmax4 + 4),
         count_launch());
    }
    const int64_t nch = (k + KC - 1) / KC;
    if (n > 0 && nch > 0) {
        unsigned long long* Sc = reinterpret_cast<unsigned long long*>(stats_scratch);
        int32_t* Ec = reinterpret_cast<int32_t*>(Sc + nch * n);
        int32_t* bad = Ec + nch * n;
        cudaMemsetAsync(bad, 0, sizeof(int32_t) * n, st);
        dim3 grid((unsigned)((n + 31) / 32), (unsigned)nch);
        (cols_stats_kernel<0><<<grid, 32 * CS_WARPS, 0, st>>>(B, k, n, ldb, Ec, Sc, bad), count_launch());
        (certify_cols_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(Ec, Sc, bad, n, (int)nch, f, Tb, width,
                                                                            dmax2 + 1, dmax4 + 4),
         count_launch());
    }
    if (ab) {
        if (m > 0) (certify_p_kernel<<<(unsigned)((m + 255) / 256), 256, 0, st>>>(ab->E, ab->rowmax, e, m, dmax4 + 2), count_launch());
        if (n > 0) (certify_p_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(ab->F, ab->colmax, f, n, dmax4 + 3), count_launch());
    }
    (certify_finalize_kernel<<<1, 1, 0, st>>>(dmax4, Tb, ab ? 1 : 0, beta), count_launch());
}

void launch_refuse(const int32_t* beta, int N, double* C, int64_t m, int64_t n, int64_t ldc, int* status,
                   cudaStream_t st) {
    if (m * n == 0) return;
    (refuse_kernel<<<148, 256, 0, st>>>(beta, host_L(N), C, m, n, ldc, status), count_launch());
}

}  // namespace oz2
