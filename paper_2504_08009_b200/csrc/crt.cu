// crt.cu -- standalone kernels of Parts 2-c, 3, 4 (Alg. 1 lines 7-10,
// PAPER.md:496-502): the split-API CRT over int32 products (oz2_crt), the
// BLAS beta / alpha = 0 helpers and the TRMM triangle copy.  The arithmetic
// itself (exact integer CRT, reading R9/R10) is in crt_device.cuh.
#include "crt_device.cuh"

namespace oz2 {
// C = beta C, or C = 0 when beta == 0 (C not read: BLAS semantics)
// C := beta C (0 if beta == 0); tri = 1 / 2: only the lower / upper triangle (SYRK)
__global__ void scale_c_kernel(double* __restrict__ C, int64_t m, int64_t n, int64_t ldc, double beta, int tri) {
    const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (idx >= m * n) return;
    const int64_t i = idx / n, j = idx % n;
    if ((tri == 1 && j > i) || (tri == 2 && j < i)) return;
    double* c = C + i * ldc + j;
    *c = beta == 0.0 ? 0.0 : beta * *c;
}

void launch_scale_c(double* C, int64_t m, int64_t n, int64_t ldc, double beta, cudaStream_t st, int tri) {
    const int64_t tot = m * n;
    if (tot <= 0) return;
    (scale_c_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(C, m, n, ldc, beta, tri), count_launch());
}

// TRMM operand: T = the uplo triangle of the n x n matrix A (1 = lower, 2 =
// upper), zeros elsewhere, ones on the diagonal when unit != 0 (BLAS diag = 'U')
__global__ void tri_copy_kernel(const double* __restrict__ A, int64_t n, int64_t lda, int uplo, int unit,
                                double* __restrict__ T) {
    const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (idx >= n * n) return;
    const int64_t i = idx / n, j = idx % n;
    double v = 0.0;
    if (i == j) v = unit ? 1.0 : A[i * lda + j];
    else if (uplo == 1 ? j < i : j > i) v = A[i * lda + j];
    T[idx] = v;
}

void launch_tri_copy(const double* A, int64_t n, int64_t lda, int uplo, int unit, double* T, cudaStream_t st) {
    const int64_t tot = n * n;
    if (tot <= 0) return;
    (tri_copy_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(A, n, lda, uplo, unit, T), count_launch());
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
    (crt_kernel<NM><<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(cprod, m, n, e, f, C, ldc), count_launch());
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
