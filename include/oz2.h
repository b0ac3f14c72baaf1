/*
 * oz2.h -- C ABI of liboz2.so: FP64 matrix multiplication C = AB emulated by
 * Ozaki scheme II on the INT8 tensor cores of NVIDIA B200 (sm_100a).
 *
 * Method: Algorithm 1 of Ozaki, Uchino, Imamura, "Ozaki Scheme II: A
 * GEMM-oriented emulation of floating-point matrix multiplication using an
 * integer modular technique" (arXiv 2504.08009), with the
 * OS II-fast scaling rule.  Citations "PAPER.md:L" are lines
 * of the paper's LaTeX source; readings R1..R17 are listed in DESIGN.md.
 *
 * Conventions (all entry points):
 *  - Matrices are ROW-MAJOR with a leading dimension in elements: A is m x k
 *    (lda >= k), B is k x n (ldb >= n), C is m x n (ldc >= n).
 *    writes A in F^{p x q}, B in F^{q x r}; here m = p, k = q, n = r.  For
 *    column-major (BLAS) semantics call with (n, m, k, B, ldb, A, lda, C, ldc).
 *  - Every matrix / vector pointer is a DEVICE pointer owned by the caller,
 *    except in oz2_dgemm_host (host pointers).  The library never frees
 *    caller memory.
 *  - Calls are ASYNCHRONOUS on the handle's stream (oz2_set_stream; default
 *    the legacy default stream) except oz2_dgemm_host, which synchronises.
 *    No call synchronises the device.  A handle may not be used by two host
 *    threads at once; distinct handles are independent.
 *  - num_moduli N must be in [2, 20]; the moduli are the first N entries of
 *    (256, 255, 253, 251, 247, 239, 233, 229, 227, 223, 217, 211, 199, 197,
 *    193, 191, 241, 181, 179, 173): Eq. (18) for N <= 16,
 *    then reading R1.
 *  - k must be < OZ2_MAX_K = 2^20.  The int32 products are exact for k < 2^17
 *    (PAPER.md:457-458); for larger k the GEMM splits K into blocks of at most
 *    1023 * 128 = 130944 ("block matrix multiplication") and adds
 *    their residues mod m_t.  oz2_modmul (raw int32 products) keeps k < 2^17.
 *  - Rows of A / columns of B holding Inf or NaN give exponent
 *    OZ2_EXP_NONFINITE and NaN in the corresponding row / column of C
 *    (reading R13; the paper assumes finite data).
 *  - Return value: OZ2_OK or an OZ2_ERR_* code; oz2_strerror() describes it.
 *    On error nothing has been launched (argument errors) or the CUDA error
 *    is reported (OZ2_ERR_CUDA) and the outputs are undefined.
 */
#ifndef OZ2_H
#define OZ2_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define OZ2_OK 0
#define OZ2_ERR_INVALID_ARG 1   /* negative size, ld too small, NULL, bad mode */
#define OZ2_ERR_NUM_MODULI 2    /* N outside [2, 20] */
#define OZ2_ERR_K_TOO_LARGE 3   /* k >= OZ2_MAX_K (oz2_modmul: k >= 2^17) */
#define OZ2_MAX_K (1 << 20)
#define OZ2_ERR_BUDGET 4        /* EQ17 mode: Eq. (17) gives k_A < 1 */
#define OZ2_ERR_CUDA 5          /* a CUDA runtime / driver call failed */
#define OZ2_ERR_NO_DEVICE 6     /* no sm_100 device */
#define OZ2_ERR_WORKSPACE 7     /* caller workspace too small */
#define OZ2_ERR_NOT_UNIQUE 8    /* condition (13), 2 c_max < M, not certified for
                                   caller-supplied exponents: C was set to NaN (see oz2_certify) */

#define OZ2_MODE_FAST 0   /* OS II-fast: Cauchy-Schwarz bound, reading R4 */
#define OZ2_MODE_EQ17 1   /* Eqs. (15)-(17): k_A = k_B = floor(log2((M/2-1)/q)/2) */
#define OZ2_MODE_ACCU 2   /* OS II-accu: an INT8 GEMM of 7-bit upper approximations of |A|, |B|
                             bounds |A'||B'|, reading R18; k < 2^17 */

#define OZ2_EXP_NONFINITE INT32_MIN

typedef struct oz2_context* oz2_handle_t;

/* ---- handle -------------------------------------------------------------- */
/* Create a handle bound to CUDA device `device` (mode FAST, legacy stream,
 * library-managed workspace).  *h receives the handle. */
int oz2_create(oz2_handle_t* h, int device);
/* Destroy a handle; frees its library-managed workspace.  Does not synchronise
 * the stream: the caller must not destroy a handle with work in flight. */
int oz2_destroy(oz2_handle_t h);
/* Subsequent calls launch on `stream` (a cudaStream_t; NULL = legacy). */
int oz2_set_stream(oz2_handle_t h, void* stream);
/* OZ2_MODE_FAST (default), OZ2_MODE_EQ17 or OZ2_MODE_ACCU: the rule for Alg. 1
 * line 1.  ACCU couples the operands (e depends on B, f on A): the split-API
 * oz2_scale_rows / oz2_scale_cols reject it (use oz2_scale_accu). */
int oz2_set_mode(oz2_handle_t h, int mode);
/* Use caller-owned device memory [ptr, ptr+bytes) as workspace (NULL, 0 =
 * library-managed, grown on demand with cudaMalloc).  Must stay valid and
 * unused by others while calls on this handle are in flight. */
int oz2_set_workspace(oz2_handle_t h, void* ptr, size_t bytes);
/* Workspace bytes oz2_dgemm_ex / oz2_dgemm_op / one batch item need for (m, n, k, N). */
size_t oz2_workspace_bytes(int64_t m, int64_t n, int64_t k, int num_moduli);

/* ---- main entry points ---------------------------------------------------- */
/* C := fl(A B) by Algorithm 1: all stages on the GPU.
 * Uses a per-device default handle (mode FAST, legacy stream).
 * m, n, k >= 0; k == 0 gives C = 0. */
int oz2_dgemm(int64_t m, int64_t n, int64_t k, const double* A, int64_t lda,
              const double* B, int64_t ldb, double* C, int64_t ldc, int num_moduli);
/* Same, on handle h (its stream, mode and workspace). */
int oz2_dgemm_ex(oz2_handle_t h, int64_t m, int64_t n, int64_t k, const double* A,
                 int64_t lda, const double* B, int64_t ldb, double* C, int64_t ldc,
                 int num_moduli);
/* The DGEMM surface ("GEMM ... depending on the
 * structure"; semantics of BLAS DGEMM, reading R19), row-major:
 *   C := alpha op(A) op(B) + beta C,  op(A) m x k, op(B) k x n, C m x n,
 *   transA = OZ2_OP_N: A stored m x k (lda >= k); OZ2_OP_T: A stored k x m (lda >= m);
 *   transB = OZ2_OP_N: B stored k x n (ldb >= n); OZ2_OP_T: B stored n x k (ldb >= k).
 * The product is Algorithm 1's C (exponents of the rows of op(A) and columns of
 * op(B)); then each entry is RN(alpha c + RN(beta c_old)) (one fma; exactly c
 * for alpha = 1, beta = 0).  beta == 0: C is not read.  alpha == 0 or k == 0:
 * no product, C := beta C.  (Column-major BLAS calls map by swapping A and B.) */
#define OZ2_OP_N 0
#define OZ2_OP_T 1
int oz2_dgemm_op(oz2_handle_t h, int transA, int transB, int64_t m, int64_t n, int64_t k,
                 double alpha, const double* A, int64_t lda, const double* B, int64_t ldb,
                 double beta, double* C, int64_t ldc, int num_moduli);
/* SYRK-structured product ("GEMM, TRMM, or SYRK"; BLAS
 * DSYRK semantics, reading R19), row-major:
 *   trans = OZ2_OP_N: C := alpha A A^T + beta C, A stored n x k (lda >= k);
 *   trans = OZ2_OP_T: C := alpha A^T A + beta C, A stored k x n (lda >= n);
 *   uplo = OZ2_LOWER / OZ2_UPPER: only that triangle of C (n x n, ldc >= n,
 *   diagonal included) is read or written; the other is left untouched.
 * Every written entry is bit-identical to the same entry of oz2_dgemm_op(A,
 * A^T): op(A)^T's column exponents are op(A)'s row exponents, so A is converted
 * once (one set of residue planes serves both operands) and only the output
 * tiles that meet the triangle are multiplied (about half the GEMM work).
 * Errors as oz2_dgemm_op; uplo / trans out of range: OZ2_ERR_INVALID_ARG. */
#define OZ2_LOWER 1
#define OZ2_UPPER 2
int oz2_dsyrk(oz2_handle_t h, int uplo, int trans, int64_t n, int64_t k, double alpha,
              const double* A, int64_t lda, double beta, double* C, int64_t ldc, int num_moduli);
/* TRMM-structured product (BLAS DTRMM semantics, reading
 * R19), row-major, in place:
 *   side = OZ2_LEFT:  B := alpha op(A) B, A m x m (lda >= m);
 *   side = OZ2_RIGHT: B := alpha B op(A), A n x n (lda >= n);  B m x n (ldb >= n);
 *   uplo: which triangle of A is referenced; diag = OZ2_UNIT: its diagonal is
 *   taken as 1 (not read), OZ2_NON_UNIT: read.
 * The product is Algorithm 1 on T = tri(A) (zeros outside the triangle), so
 * every entry is bit-identical to oz2_dgemm_op(T, B) scaled by alpha; the GEMM
 * skips, per output tile, the k-blocks where op(T) is zero (about half the
 * work).  The masked copy T lives in handle-owned memory (grown on demand).
 * Errors as oz2_dgemm_op; side / uplo / transA / diag out of range:
 * OZ2_ERR_INVALID_ARG. */
#define OZ2_LEFT 0
#define OZ2_RIGHT 1
#define OZ2_NON_UNIT 0
#define OZ2_UNIT 1
int oz2_dtrmm(oz2_handle_t h, int side, int uplo, int transA, int diag, int64_t m, int64_t n,
              double alpha, const double* A, int64_t lda, double* B, int64_t ldb, int num_moduli);
/* Alg. 1 lines 2-10 with caller-supplied line-1 exponents e[m], f[n] (device
 * int32, OZ2_EXP_NONFINITE allowed): C = D^-1 X E^-1.  For sharded line-1 rules
 * (e.g. OS II-accu across row blocks, where f is a MIN all-reduce of the
 * ranks' partial f).  Condition (13) is certified on the
 * device (oz2_certify; one statistics pass over A and B) unless disabled with
 * oz2_set_certify(h, 0): if the certificate fails, every entry of C is set to
 * NaN and the handle's status records OZ2_ERR_NOT_UNIQUE (read it with
 * oz2_status -- the call itself does not synchronise). */
int oz2_dgemm_scaled(oz2_handle_t h, int64_t m, int64_t n, int64_t k, const double* A,
                     int64_t lda, const double* B, int64_t ldb, const int32_t* e,
                     const int32_t* f, double* C, int64_t ldc, int num_moduli);
/* ---- condition (13) certificates (Eq. 13: 2 c_max < M) ----
 * oz2_certify writes to the device int32 *beta a bound c_max <= 2^beta for the
 * product A B under caller-supplied exponents e[m], f[n]:
 *   beta = max_i (e_i - e^F_i) + max_j (f_j - f^F_j) + 2T,
 * where e^F, f^F are the OS II-fast exponents (reading R4), which guarantee
 * ||2^(e^F_i) a_i||_2 <= 2^T; by Cauchy-Schwarz (|A'||B'|)_ij <= 2^beta.  Rows /
 * columns that are zero, hold Inf/NaN, or carry the OZ2_EXP_NONFINITE exponent do
 * not take part; INT32_MIN if nothing does.  For k < 2^17 the OS II-accu bound
 * (row / column maxima of the 7-bit bound GEMM, reading R18) is formed as well
 * and the smaller bound is reported.  Exponents under which some trunc(2^e a)
 * would not fit the residue kernels' integers (63 bits for N <= 16, 95 bits
 * otherwise) give beta = INT32_MAX.  beta <= L (oz2_tables) certifies
 * uniqueness; it is a sufficient condition (the bounds may overestimate).
 * The certified stage calls (oz2_crt, oz2_crt_sum with a non-NULL beta, and
 * oz2_dgemm_scaled) refuse when beta > L: C := NaN and the handle's sticky
 * status becomes OZ2_ERR_NOT_UNIQUE -- no host synchronisation.
 * oz2_status synchronises the handle's stream and returns (and clears) it. */
int oz2_certify(oz2_handle_t h, int64_t m, int64_t n, int64_t k, const double* A, int64_t lda,
                const double* B, int64_t ldb, const int32_t* e, const int32_t* f, int num_moduli,
                int32_t* beta);
int oz2_set_certify(oz2_handle_t h, int enable);
int oz2_status(oz2_handle_t h);
/* Prepared operands: oz2_prepare_a converts A (m x k) and oz2_prepare_b converts
 * B (k x n) once (Alg. 1 lines 1-5 for that operand: its exponents and its N
 * residue planes) into device memory owned by the returned object (freed by
 * oz2_release, which waits for the device).  Since e_i depends on row i of A
 * only and f_j on column j of B only (FAST / EQ17; ACCU couples the operands
 * and is rejected), the products are bit-identical to oz2_dgemm_ex(A, B):
 *   oz2_dgemm_prepared(h, pb, m, A, C): lines 1, 2, 4 for A, then 6-10 against pb;
 *   oz2_dgemm_prep2(h, pa, pb, C):      lines 6-10 only (pa->k == pb->k, same N).
 * Used by the row-block and column-panel pipelines (one B, many row blocks of
 * A; one A, many column panels of B).  The handle's mode must equal the mode
 * the objects were prepared with; the objects are read-only afterwards and may
 * be used by several handles of the same device (stream ordering is the
 * caller's). */
typedef struct oz2_prepared* oz2_prep_t;
int oz2_prepare_a(oz2_handle_t h, int64_t m, int64_t k, const double* A, int64_t lda,
                  int num_moduli, oz2_prep_t* out);
int oz2_prepare_b(oz2_handle_t h, int64_t k, int64_t n, const double* B, int64_t ldb,
                  int num_moduli, oz2_prep_t* out);
int oz2_dgemm_prepared(oz2_handle_t h, oz2_prep_t pb, int64_t m, const double* A, int64_t lda,
                       double* C, int64_t ldc);
int oz2_dgemm_prep2(oz2_handle_t h, oz2_prep_t pa, oz2_prep_t pb, double* C, int64_t ldc);
/* Convert another matrix of the same shape (and side, N, mode) into p's memory,
 * replacing its contents (stream-ordered on h: work already queued that reads
 * p sees the old contents).  The pipelines reuse two objects per operand. */
int oz2_reprepare(oz2_handle_t h, oz2_prep_t p, const double* X, int64_t ld);
int oz2_release(oz2_prep_t p);
/* Limit the persistent GEMM to `sms` SMs (0 = all; rounded down to even), e.g.
 * to leave SMs to NCCL kernels that overlap it.  Results do not depend on it. */
int oz2_set_sm_limit(oz2_handle_t h, int sms);
/* ---- K-split (2-D multi-GPU) pieces, FAST / EQ17 --------------------------
 * Each rank holds A[:, K_r] (m x k_r) and B[K_r, :] (k_r x n), K_r starting on
 * a multiple of 256 (the FAST rule's chunk grid, reading R4).  The exponents of
 * the whole product then follow from two small all-reduces:
 *   phase 1: oz2_kslice_stats_rows / _cols(E_global = NULL) -> E_out: the max
 *            chunk exponent (INT32_MIN: no non-zero entry; INT32_MAX: Inf/NaN)
 *            -> all-reduce MAX;
 *   phase 2: the same with E_global -> S_out: sum of ceil(S_c / 4^(E - E_c))
 *            over the rank's chunks (uint64) -> all-reduce SUM;
 *   oz2_exponents_from_stats(E, S, k_total) -> e (or f), bit-identical to the
 *   one-GPU rule (EQ17: phase 1 and k_total suffice).
 * oz2_modmul_residues: Alg. 1 lines 6-7 on the rank's residue planes,
 * R = C'_t mod m_t in [0, m_t) as uint8, layout [m/rpb][N][rpb][n]
 * (rows_per_block rpb; 0 = m), ready for an all-to-all to row-block owners.
 * oz2_crt_sum: c''_t = (sum over the parts g of R + g * part_stride) mod m_t
 * (linearity of mod), then lines 8-10: C = D^-1 X E^-1 for the local rows
 * (beta: as oz2_crt).
 * All device pointers; asynchronous on the handle's stream. */
int oz2_kslice_stats_rows(oz2_handle_t h, int64_t m, int64_t k, const double* A, int64_t lda,
                          const int32_t* E_global, int32_t* E_out, uint64_t* S_out);
int oz2_kslice_stats_cols(oz2_handle_t h, int64_t k, int64_t n, const double* B, int64_t ldb,
                          const int32_t* E_global, int32_t* E_out, uint64_t* S_out);
int oz2_exponents_from_stats(oz2_handle_t h, int64_t count, const int32_t* E, const uint64_t* S,
                             int64_t k_total, int num_moduli, int32_t* e);
int oz2_modmul_residues(oz2_handle_t h, int64_t m, int64_t n, int64_t k, const int8_t* Ares,
                        const int8_t* Bres, int64_t ld_res, int num_moduli, uint8_t* R,
                        int64_t rows_per_block);
int oz2_crt_sum(oz2_handle_t h, int parts, int64_t m, int64_t n, const uint8_t* R,
                int64_t part_stride, const int32_t* e, const int32_t* f, int num_moduli,
                double* C, int64_t ldc, const int32_t* beta);
/* batch independent products: A + b*strideA, B + b*strideB, C + b*strideC
 * (elements), b = 0..batch-1, in stream order on one workspace. */
int oz2_dgemm_strided_batched(oz2_handle_t h, int transA, int transB, int64_t m, int64_t n,
                              int64_t k, double alpha, const double* A, int64_t lda,
                              int64_t strideA, const double* B, int64_t ldb, int64_t strideB,
                              double beta, double* C, int64_t ldc, int64_t strideC,
                              int64_t batch, int num_moduli);

/* End-to-end variant with HOST buffers: copies A and B to the device, runs
 * Algorithm 1 and copies C back, then synchronises.  Copies and computation
 * are pipelined (bit-identical to oz2_dgemm_ex):
 *  - m, n >= 8192 (FAST / EQ17): 4 column panels of B x row blocks of A; the
 *    H2D stream interleaves B0, A0, B1, A1, ..., each panel / block is
 *    converted once when it lands, each (block, panel) product runs as soon as
 *    both are on the device, and its C tile is copied back at once on a second
 *    copy stream (OZ2_HOST_2D=0 selects the row-block pipeline below);
 *  - otherwise row blocks of A / C (multiples of 256 rows; for m >= 12288 a
 *    1024-row head, 4096-row middle blocks and a shrinking tail) after B;
 *  - OZ2_MODE_ACCU (f depends on all of A): copy, compute, copy back.
 * Copies overlap only if the host buffers are page-locked.  Workspace
 * (ctx-owned or oz2_set_workspace): oz2_workspace_bytes(m, n, k, N) +
 * 8 (mk + kn + mn) + 1 KiB. */
int oz2_dgemm_host(oz2_handle_t h, int64_t m, int64_t n, int64_t k, const double* A,
                   int64_t lda, const double* B, int64_t ldb, double* C, int64_t ldc,
                   int num_moduli);

/* ---- the FP64 prime-modulus regime (Sec. 3.2) -----------
 * C ~= A B with s pairwise-coprime primes m_t: the s largest primes below 2^b,
 * b = floor((55 - ceil(log2 k)) / 2) (reading F1), so that k m_t^2 <= 2^55 =
 * 4 u^-1 (Eq. 19) and every residue product is exact in binary64 (Eq. 20);
 * for k = 1024 the moduli are Eq. (21) verbatim.  Line 1 is the OS II-fast rule
 * with this M's T (reading F2); lines 2-5 form binary64 residue planes; line 6
 * runs as s FP64 tensor-core GEMMs (cuBLAS DGEMM, strided batched, loaded at
 * run time); lines 7-10 reconstruct X exactly and write v binary64 words per
 * entry (reading F3: word w at C + w * strideC, most significant first, each
 * the nearest binary64 to what the earlier words leave) -- results beyond
 * binary64 precision (k_A ~ 170 at s = 16).
 * s in [2, 22]; v in [1, 4]; m k, k n, m n < 2^31 (cuBLAS).  Workspace:
 * oz2_fp64mod_workspace_bytes (8 s (mk + kn + mn) + small).  Errors as
 * oz2_dgemm_ex; cuBLAS missing or failing: OZ2_ERR_CUDA. */
int oz2_dgemm_fp64mod(oz2_handle_t h, int64_t m, int64_t n, int64_t k, const double* A,
                      int64_t lda, const double* B, int64_t ldb, int s, int v, double* C,
                      int64_t ldc, int64_t strideC);
/* The same for double-word inputs (Eqs. 22-23, reading F6): A = A + A2, B = B + B2
 * (A2, B2 with the leading dimensions of A, B; either may be NULL = zero),
 * with |A2| <= u |A| and |B2| <= u |B| elementwise (Eq. 23; u = 2^-53).  Line 1
 * uses |A| + |A2| rounded upward; trunc(2^e (a + a2)) is formed exactly. */
int oz2_dgemm_fp64mod_dw(oz2_handle_t h, int64_t m, int64_t n, int64_t k, const double* A,
                         const double* A2, int64_t lda, const double* B, const double* B2,
                         int64_t ldb, int s, int v, double* C, int64_t ldc, int64_t strideC);
size_t oz2_fp64mod_workspace_bytes(int64_t m, int64_t n, int64_t k, int s);
/* The regime's constants (host only): moduli[s], M as 17 little-endian 32-bit
 * words, L = floor(log2(M/2 - 1)), T = floor(L/2); q = the inner dimension. */
int oz2_fp64mod_tables(int s, int64_t q, int64_t* moduli, uint32_t* M_words, int32_t* L, int32_t* T);

/* ---- split API: each stage of Algorithm 1 on its own (stage parity) ------- */
/* Alg. 1 line 1 for the rows of A (m x k): e[i] such that D = diag(2^e[i])
 * (reading R4 / R5 by the handle's mode).  e: int32[m]. */
int oz2_scale_rows(oz2_handle_t h, int64_t m, int64_t k, const double* A, int64_t lda,
                   int num_moduli, int32_t* e);
/* Alg. 1 line 1 for the columns of B (k x n): f[j], E = diag(2^f[j]).  f: int32[n]. */
int oz2_scale_cols(oz2_handle_t h, int64_t k, int64_t n, const double* B, int64_t ldb,
                   int num_moduli, int32_t* f);
/* Alg. 1 line 1 by the OS II-accu rule (reading R18) for the product A B
 * (A m x k, B k x n, row-major; k < 2^17): e[m], f[n].  Any handle mode. */
int oz2_scale_accu(oz2_handle_t h, int64_t m, int64_t n, int64_t k, const double* A, int64_t lda,
                   const double* B, int64_t ldb, int num_moduli, int32_t* e, int32_t* f);
/* Alg. 1 line 2: Ap = trunc(D A), m x k row-major FP64 integers (ld = k). */
int oz2_trunc_rows(oz2_handle_t h, int64_t m, int64_t k, const double* A, int64_t lda,
                   const int32_t* e, double* Ap);
/* Alg. 1 line 3, transposed: BpT = trunc(B E)^T, n x k row-major (ld = k). */
int oz2_trunc_cols(oz2_handle_t h, int64_t k, int64_t n, const double* B, int64_t ldb,
                   const int32_t* f, double* BpT);
/* Alg. 1 lines 2+4 (Eq. 11): int8 planes
 * Ares[t][i][l] = trunc(2^e[i] a_il) mod m_t (Eq. 1), t < N, i < m, l < k,
 * plane row stride ld_res (a multiple of 16, >= k), plane stride m*ld_res.
 * Bytes [k, ld_res) of each row are unspecified. */
int oz2_residues_rows(oz2_handle_t h, int64_t m, int64_t k, const double* A, int64_t lda,
                      const int32_t* e, int num_moduli, int8_t* Ares, int64_t ld_res);
/* Alg. 1 lines 3+5 for B, stored K-major (transposed):
 * Bres[t][j][l] = trunc(2^f[j] b_lj) mod m_t, plane stride n*ld_res. */
int oz2_residues_cols(oz2_handle_t h, int64_t k, int64_t n, const double* B, int64_t ldb,
                      const int32_t* f, int num_moduli, int8_t* Bres, int64_t ld_res);
/* Alg. 1 line 6 on the INT8 tensor cores: Cprod[t][i][j] = sum_l
 * Ares[t][i][l] Bres[t][j][l] exactly (int32).
 * Cprod: int32[N][m][n]. */
int oz2_modmul(oz2_handle_t h, int64_t m, int64_t n, int64_t k, const int8_t* Ares,
               const int8_t* Bres, int64_t ld_res, int num_moduli, int32_t* Cprod);
/* Alg. 1 lines 7-10: c''_t = Cprod_t mod m_t in [0, m_t), X = (sum_t c''_t
 * M y_t / m_t) mod M (Eq. 1), C[i][j] = 2^-(e[i]+f[j]) RN(X)  (reading R10).
 * beta (device int32 from oz2_certify, or NULL = not certified): beta > L
 * refuses (C := NaN, status OZ2_ERR_NOT_UNIQUE; see oz2_certify). */
int oz2_crt(oz2_handle_t h, int64_t m, int64_t n, const int32_t* Cprod, const int32_t* e,
            const int32_t* f, int num_moduli, double* C, int64_t ldc, const int32_t* beta);

/* ---- constants (host memory, no device needed) ----------------------------
 * moduli[N], y[N] (M_t y_t == 1 mod m_t, least positive), w_words[5*N] with
 * w_t = M y_t / m_t = sum_x w_words[5*t + x] 2^(32 x) (the CRT weights of Alg. 1
 * line 8), M_words[5] the same split of M = prod m_t,
 * *nbytes = bytes of M (the kernels' dp4a limbs of w_t),
 * *L = floor(log2(M/2 - 1)), *T = floor(L/2).  Any output pointer may be NULL. */
int oz2_tables(int num_moduli, int32_t* moduli, int32_t* y, uint32_t* w_words, uint32_t* M_words,
               int32_t* nbytes, int32_t* L, int32_t* T);
/* Eq. (17) in exact integer form: max{kappa : q 4^kappa <= M/2 - 1}, -1 if none. */
int oz2_eq17_k(int num_moduli, int64_t q);

/* ---- tracing ----------------------------------------------------------------
 * With profiling enabled, every oz2_dgemm_ex call records CUDA events on the
 * handle's stream at its stage boundaries (no host synchronisation).
 * oz2_stage_times waits for the recorded events, writes the summed device
 * milliseconds of each stage since the last read into ms[0..OZ2_NUM_STAGES-1]
 * (order: OZ2_STAGE_*), the number of calls into *calls, and resets. */
#define OZ2_NUM_STAGES 5
#define OZ2_STAGE_ROWS 0    /* rows of A (lines 1, 2, 4) [+ B if OZ2_CONV_OVERLAP=1]   */
#define OZ2_STAGE_COLSTATS 1/* columns of B: exponents (line 1)                      */
#define OZ2_STAGE_COLRES 2  /* columns of B: residues (lines 3, 5)                   */
#define OZ2_STAGE_GEMM 3    /* N modular products on tcgen05 (line 6) [+ fused 7-10] */
#define OZ2_STAGE_CRT 4     /* CRT + inverse scaling (lines 7-10) if not fused       */
int oz2_set_profiling(oz2_handle_t h, int enable);
int oz2_stage_times(oz2_handle_t h, double* ms, int64_t* calls);

const char* oz2_strerror(int code);
/* 100 * major + minor */
int oz2_version(void);
/* Kernels the library has launched since it was loaded (all handles, all
 * devices): every launch site counts itself, so the difference across a timed
 * region is the number of liboz2 kernels that ran in it. */
unsigned long long oz2_kernel_launches(void);

#ifdef __cplusplus
}
#endif
#endif /* OZ2_H */
