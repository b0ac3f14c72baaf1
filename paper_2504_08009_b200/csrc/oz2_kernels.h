// oz2_kernels.h -- host-side launchers of the sm_100a kernels (api.cu calls these).
#pragma once

#include <vector>
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace oz2 {

// bit length of M = prod of the first N moduli (N = 2..20; tables.cpp computes M
// itself and api.cu checks that its limb and word counts agree with these)
__host__ __device__ constexpr int m_bits(int N) {
    constexpr int b[21] = {0, 8, 16, 24, 32, 40, 48, 56, 64, 72, 80, 87, 95, 103, 110, 118, 126, 133, 141, 148, 156};
    return b[N];
}
// bytes of M; 32-bit words of S < 2^13 M; 32-bit words of X in [-3M/2, 3M/2)
__host__ __device__ constexpr int crt_bytes(int N) { return (m_bits(N) + 7) / 8; }
__host__ __device__ constexpr int crt_swords(int N) { return (m_bits(N) + 13 + 31) / 32; }
__host__ __device__ constexpr int crt_words(int N) { return (m_bits(N) + 2 + 31) / 32; }

int host_T(int N);   // floor(L/2) for N moduli (host copy of the table)
int host_L(int N);   // floor(log2(M/2 - 1))

// scale.cu -- Alg. 1 lines 1-5
void launch_init_bfrag(cudaStream_t st);   // once per device after the tables: the residue MMAs' B fragments
// what: 1 = exponents e, 2 = residues (given e), 3 = both (one pass per row)
// pstride: bytes between residue planes (default m * ldr)
// xbits: a bound |trunc(2^e a)| < 2^xbits of the line-1 rule in use (selects the
// residue kernels' integer width; 64 = the widest for N, always valid)
void launch_rows(const double* A, int64_t m, int64_t k, int64_t lda, int N, int what, int mode,
                 int kstar, int32_t* e, int8_t* res, int64_t ldr, cudaStream_t st, int64_t pstride = 0,
                 int xbits = 64);
void launch_trunc_rows(const double* A, int64_t m, int64_t k, int64_t lda, const int32_t* e,
                       double* out, cudaStream_t st);
size_t cols_stats_bytes(int64_t k, int64_t n);
void launch_cols_exponents(const double* B, int64_t k, int64_t n, int64_t ldb, int N, int mode,
                           int kstar, int32_t* f, void* scratch, cudaStream_t st);
// pstride: bytes between residue planes (default n * ldr)
void launch_cols_residues(const double* B, int64_t k, int64_t n, int64_t ldb, const int32_t* f, int N,
                          int8_t* res, int64_t ldr, cudaStream_t st, int64_t pstride = 0, int xbits = 64);
void launch_trunc_cols(const double* B, int64_t k, int64_t n, int64_t ldb, const int32_t* f,
                       double* out, cudaStream_t st);

// gemm.cu -- Alg. 1 line 6 on tcgen05 (kind::i8)
cudaError_t upload_tables_gemm(const void* tabs, size_t bytes);   // gemm.cu's copy of c_tab
int gemm_cta_group();   // 1 or 2 (CTA pairs, cta_group::2)
int gemm_bk();          // bytes of K per shared-memory stage (128, or 64 when built with -DOZ2_BK=64)
int launch_modmul(const CUtensorMap* tmA, const CUtensorMap* tmB, int64_t m, int64_t n, int64_t k,
                  int N, int32_t* cprod, uint32_t* sync_ctr, int num_sms, cudaStream_t st);
// + Alg. 1 lines 7-10 fused into the epilogue (uint8 residue scratch, exact CRT)
size_t fused_scratch_bytes(int64_t m, int64_t n, int N, int num_sms);
// fewer output tiles than CTA pairs: spread (tile, modulus) units (launch_modmul_residues + CRT kernel)
bool gemm_unit_parallel(int64_t m, int64_t n, int num_sms);
// (alpha, beta) != (1, 0): C = alpha AB + beta C in the epilogue (BLAS semantics)
int launch_modmul_fused(const CUtensorMap* tmA, const CUtensorMap* tmB, int64_t m, int64_t n, int64_t k,
                        int N, uint8_t* scratch, const int32_t* e, const int32_t* f, double* C, int64_t ldc,
                        uint32_t* sync_ctr, int num_sms, cudaStream_t st, double alpha = 1.0,
                        double beta = 0.0, int tri = 0, const uint32_t* tiles = nullptr, int ntiles = 0,
                        int kskip = 0);
// SYRK (tri = 1 lower, 2 upper; m = n): the output tiles of the fused GEMM that
// meet the triangle, in the GEMM's raster order, packed (tm << 16) | tn
std::vector<uint32_t> tri_tile_list(int64_t m, int64_t n, int tri, int num_sms);
// C = beta C (beta != 0) or 0: the alpha = 0 / k = 0 cases of the DGEMM surface
void launch_scale_c(double* C, int64_t m, int64_t n, int64_t ldc, double beta, cudaStream_t st, int tri = 0);
void launch_tri_copy(const double* A, int64_t n, int64_t lda, int uplo, int unit, double* T, cudaStream_t st);

// accu.cu -- Alg. 1 line 1 by the OS II-accu rule (reading R18)
void launch_rows_hat7(const double* X, int64_t rows, int64_t k, int64_t ld, int32_t* E, uint8_t* hat, int64_t ldr,
                      cudaStream_t st);
void launch_cols_hat7(const double* X, int64_t k, int64_t cols, int64_t ld, const int32_t* F, uint8_t* hat,
                      int64_t ldr, cudaStream_t st);
void launch_accu_finalize(const int32_t* E, const uint32_t* Pmax, int64_t cnt, int N, int32_t* e, cudaStream_t st);
// the line-1 bound GEMM P = Ahat Bhat^T (unsigned int8): only row / column maxima
// of P leave the chip (atomicMax into rowmax[m], colmax[n], zeroed here first)
int launch_bound_gemm(const CUtensorMap* tmA, const CUtensorMap* tmB, int64_t m, int64_t n, int64_t k,
                      uint32_t* rowmax, uint32_t* colmax, uint32_t* sync_ctr, int num_sms, cudaStream_t st);

// kslice.cu -- K-split pieces (statistics phases, residue sum + CRT)
void launch_kslice_rows(const double* A, int64_t m, int64_t k, int64_t lda, int mode, const int32_t* Eg,
                        int32_t* E_out, unsigned long long* S_out, cudaStream_t st);
void launch_kslice_cols(const double* B, int64_t k, int64_t n, int64_t ldb, int mode, const int32_t* Eg,
                        int32_t* E_out, unsigned long long* S_out, void* scratch, cudaStream_t st);
void launch_exponents_from_stats(const int32_t* E, const unsigned long long* S, int64_t cnt, int N, int mode,
                                 int kstar, int32_t* e, cudaStream_t st);
void launch_crt_sum(const uint8_t* R, int G, int64_t part_stride, int64_t m, int64_t n, const int32_t* e,
                    const int32_t* f, int N, double* C, int64_t ldc, cudaStream_t st);
// line 6 + 7 only: c''_t = C'_t mod m_t in [0, m_t) as uint8 planes, K-blocked;
// layout [m / rows_per_block][N][rows_per_block][n] (rows_per_block = m: [N][m][n])
int launch_modmul_residues(const CUtensorMap* tmA, const CUtensorMap* tmB, int64_t m, int64_t n, int64_t k, int N,
                           uint8_t* scratch, uint8_t* R, int64_t rows_per_block, uint32_t* sync_ctr, int num_sms,
                           cudaStream_t st);

// certify.cu -- condition (13) certificate for caller-supplied exponents
// dmax4: five device ints (scratch); stats_scratch: cols_stats_bytes(k, n);
// ab (or NULL): the OS II-accu line-1 bound of the same product (E, F, row /
// column maxima of P), giving the second, often tighter, bound
struct AccuBound {
    const int32_t* E;
    const int32_t* F;
    const uint32_t* rowmax;
    const uint32_t* colmax;
};
void launch_certify(const double* A, int64_t m, int64_t k, int64_t lda, const double* B, int64_t n, int64_t ldb,
                    const int32_t* e, const int32_t* f, int N, int* dmax4, void* stats_scratch, int32_t* beta,
                    const AccuBound* ab, cudaStream_t st);
// beta > L: C := NaN and atomicOr(status, 1)
void launch_refuse(const int32_t* beta, int N, double* C, int64_t m, int64_t n, int64_t ldc, int* status,
                   cudaStream_t st);

// fp64mod.cu -- the FP64 prime-modulus regime (Eqs. 19-21)
constexpr int F64_MAX_S = 22;      // primes (reading F4)
constexpr int F64_MAX_W = 17;      // 32-bit words of S = sum c''_t w_t < s 2^22 M < 2^511
constexpr int F64_POW2 = 256;      // 2^j mod m_t table: trunc(2^e a) < 2^(T+1) <= 2^242 = mant 2^sh, sh < 192
int f64_prime_bits(int64_t q);
int f64_tables(int s, int64_t q, int64_t* moduli, uint32_t* M_words, int32_t* L, int32_t* T);
size_t f64_workspace_bytes(int64_t m, int64_t n, int64_t k, int s);
// 0 ok, -1 bad (s, k), -2 cuBLAS unavailable, -3 cuBLAS error, -4 CUDA error
// A2, B2: NULL or the second words of double-word inputs (reading F6)
int launch_fp64mod(int device, const double* A, const double* A2, int64_t m, int64_t k, int64_t lda,
                   const double* B, const double* B2, int64_t n, int64_t ldb, int s, int v, double* C, int64_t ldc,
                   int64_t strideC, uint8_t* ws, cudaStream_t st);
void launch_exponents_T(const int32_t* E, const unsigned long long* S, int64_t cnt, int T, int32_t* e,
                        cudaStream_t st);

// crt.cu -- Alg. 1 lines 7-10
void launch_crt(const int32_t* cprod, int64_t m, int64_t n, const int32_t* e, const int32_t* f,
                int N, double* C, int64_t ldc, cudaStream_t st);

}  // namespace oz2
