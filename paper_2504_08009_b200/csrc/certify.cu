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
// (13).  It is a sufficient condition only.  Rows / columns that are zero or
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
                    int Tb, int* __restrict__ dmax) {
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
    }
}

// columns: per-chunk statistics from cols_stats_kernel ([nch][n])
__global__ void certify_cols_kernel(const int32_t* __restrict__ Ec, const unsigned long long* __restrict__ Sc,
                                    const int32_t* __restrict__ bad, int64_t n, int nch,
                                    const int32_t* __restrict__ f, int Tb, int* __restrict__ dmax) {
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
}

// beta = dmax[0] + dmax[1] + 2T, or INT32_MIN if no row or no column takes part
__global__ void certify_finalize_kernel(const int* __restrict__ dmax, int Tb, int32_t* __restrict__ beta) {
    const int a = dmax[0], b = dmax[1];
    *beta = (a == INT32_MIN || b == INT32_MIN) ? INT32_MIN : clamp_i32((long long)a + b + 2LL * Tb);
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

void launch_certify(const double* A, int64_t m, int64_t k, int64_t lda, const double* B, int64_t n, int64_t ldb,
                    const int32_t* e, const int32_t* f, int N, int* dmax2, void* stats_scratch, int32_t* beta,
                    cudaStream_t st) {
    const int Tb = host_T(N);
    static const int init[2] = {INT32_MIN, INT32_MIN};
    cudaMemcpyAsync(dmax2, init, sizeof(init), cudaMemcpyHostToDevice, st);
    if (m > 0 && k > 0) {
        const size_t smem = row_smem_bytes(k);
        if (smem > 48 * 1024) cudaFuncSetAttribute(certify_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        certify_rows_kernel<<<(unsigned)m, 256, smem, st>>>(A, m, k, lda, e, Tb, dmax2);
    }
    const int64_t nch = (k + KC - 1) / KC;
    if (n > 0 && nch > 0) {
        unsigned long long* Sc = reinterpret_cast<unsigned long long*>(stats_scratch);
        int32_t* Ec = reinterpret_cast<int32_t*>(Sc + nch * n);
        int32_t* bad = Ec + nch * n;
        cudaMemsetAsync(bad, 0, sizeof(int32_t) * n, st);
        dim3 grid((unsigned)((n + 31) / 32), (unsigned)nch);
        cols_stats_kernel<0><<<grid, 32 * CS_WARPS, 0, st>>>(B, k, n, ldb, Ec, Sc, bad);
        certify_cols_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(Ec, Sc, bad, n, (int)nch, f, Tb, dmax2 + 1);
    }
    certify_finalize_kernel<<<1, 1, 0, st>>>(dmax2, Tb, beta);
}

void launch_refuse(const int32_t* beta, int N, double* C, int64_t m, int64_t n, int64_t ldc, int* status,
                   cudaStream_t st) {
    if (m * n == 0) return;
    refuse_kernel<<<148, 256, 0, st>>>(beta, host_L(N), C, m, n, ldc, status);
}

}  // namespace oz2
