// kslice.cu -- K-split (2-D) multi-GPU pieces: every rank holds
// a slice of the inner dimension, A[:, K_r] and B[K_r, :], with K_r boundaries
// on the KC = 256 chunk grid of the FAST rule (reading R4).  Because that rule
// is built from per-chunk integer statistics combined by max and by ceil-sums,
// the exponents of the full product follow from two tiny all-reduces:
//   phase 1: E_i = max over the rank's chunks of E_c   (all-reduce MAX)
//   phase 2: S_i = sum over the rank's chunks of ceil(S_c / 4^(E_i - E_c)) with
//            the global E_i                              (all-reduce SUM)
// then e_i = T + 15 - E_i - h(S_i) exactly as on one GPU (EQ17: e = k* - 1 - E
// with k* from the full k).  Markers: E = INT32_MIN no non-zero entry,
// INT32_MAX an Inf / NaN (MAX propagates it).  The per-modulus products of the
// slices are reduced mod m_t (Alg. 1 line 7) and summed mod m_t across ranks
// (linearity of mod) before the CRT: oz2_crt_sum.
#include "crt_device.cuh"

namespace oz2 {

constexpr int KS_EMAX_MARK = INT32_MAX;       // a non-finite entry in the row / column

// one CTA per row: phase 1 (Eg == nullptr) E_out[i]; phase 2 S_out[i] given Eg[i]
template <int MODE>
__global__ void __launch_bounds__(256)
kslice_rows_kernel(const double* __restrict__ A, int64_t m, int64_t k, int64_t lda, const int32_t* __restrict__ Eg,
                   int32_t* __restrict__ E_out, unsigned long long* __restrict__ S_out) {
    extern __shared__ __align__(16) unsigned char row_smem[];
    const int64_t i = blockIdx.x;
    if (i >= m) return;
    const int64_t nch = (k + KC - 1) / KC;
    RowSmem sm;
    sm.Sc = reinterpret_cast<unsigned long long*>(row_smem);
    sm.Ec = reinterpret_cast<int*>(row_smem + sizeof(unsigned long long) * (nch > 0 ? nch : 1));
    sm.misc = sm.Ec + (nch > 0 ? nch : 1);
    row_chunk_stats<MODE>(A + i * lda, k, sm);
    if (threadIdx.x >= 32) return;
    const int lane = threadIdx.x;
    if (!Eg) {
        int E = INT32_MIN;
        for (int c = lane; c < (int)nch; c += 32) E = max(E, sm.Ec[c]);
        E = warp_max(E);
        if (lane == 0) E_out[i] = sm.misc[0] ? KS_EMAX_MARK : E;
    } else {
        const int E = Eg[i];
        uint64_t S = 0;
        if (E != INT32_MIN && E != KS_EMAX_MARK)
            for (int c = lane; c < (int)nch; c += 32)
                if (sm.Ec[c] != INT32_MIN) S += ceil_shift(sm.Sc[c], 2 * (E - sm.Ec[c]));
        S = warp_sum64(S);
        if (lane == 0) S_out[i] = S;
    }
}

// columns: per-chunk statistics from cols_stats_kernel ([nch][n]), then the phase
__global__ void kslice_cols_kernel(const int32_t* __restrict__ Ec, const unsigned long long* __restrict__ Sc,
                                   const int32_t* __restrict__ bad, int64_t n, int nch,
                                   const int32_t* __restrict__ Eg, int32_t* __restrict__ E_out,
                                   unsigned long long* __restrict__ S_out) {
    const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (j >= n) return;
    if (!Eg) {
        int E = INT32_MIN;
        for (int c = 0; c < nch; c++) E = max(E, Ec[(int64_t)c * n + j]);
        E_out[j] = bad[j] ? KS_EMAX_MARK : E;
    } else {
        const int E = Eg[j];
        uint64_t S = 0;
        if (E != INT32_MIN && E != KS_EMAX_MARK)
            for (int c = 0; c < nch; c++) {
                const int e = Ec[(int64_t)c * n + j];
                if (e != INT32_MIN) S += ceil_shift(Sc[(int64_t)c * n + j], 2 * (E - e));
            }
        S_out[j] = S;
    }
}

template <int MODE>
__global__ void exponents_from_stats_kernel(const int32_t* __restrict__ E, const unsigned long long* __restrict__ S,
                                            int64_t cnt, int Tb, int kstar, int32_t* __restrict__ e) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= cnt) return;
    const int Ei = E[i];
    if (Ei == KS_EMAX_MARK) { e[i] = OZ2_EXP_NONFINITE_DEV; return; }
    if (Ei == INT32_MIN) { e[i] = 0; return; }
    e[i] = MODE == 0 ? Tb + 15 - Ei - log4_ceil(S[i]) : kstar - 1 - Ei;
}

// lines 7-10 for G partial products: c''_t = (sum_g R[g][t][i][j]) mod m_t, then
// the CRT and scaling (crt_from_packed).  R[g] at R + g * part_stride, [N][m][n].
// One thread per row i and 4 consecutive columns: one 4-byte load per plane
// (coalesced rows), no 64-bit index division; G = 1 (the single-GPU small-problem
// path) needs no reduction at all -- the planes already hold c''_t.
template <int NM>
__global__ void __launch_bounds__(256)
crt_sum_kernel(const uint8_t* __restrict__ R, int G, int64_t part_stride, int64_t m, int64_t n,
               const int32_t* __restrict__ e, const int32_t* __restrict__ f, double* __restrict__ C, int64_t ldc) {
    constexpr int G4 = (NM + 3) / 4;
    const int64_t c0 = 4 * ((int64_t)blockIdx.x * blockDim.x + threadIdx.x);
    if (c0 >= n) return;
    const bool full = c0 + 4 <= n && (n & 3) == 0;
    for (int64_t i = blockIdx.y; i < m; i += gridDim.y) {
        uint32_t wt[NM];                                   // byte j of wt[t] = c''_t of column c0 + j
        #pragma unroll
        for (int t = 0; t < NM; t++) {
            const uint8_t* base = R + ((int64_t)t * m + i) * n + c0;
            if (G == 1) {
                if (full) {
                    wt[t] = *reinterpret_cast<const uint32_t*>(base);
                } else {
                    uint32_t w = 0;
                    for (int j = 0; j < 4; j++) if (c0 + j < n) w |= (uint32_t)base[j] << (8 * j);
                    wt[t] = w;
                }
            } else {
                int32_t s4[4] = {0, 0, 0, 0};
                for (int g = 0; g < G; g++) {
                    const uint8_t* b = base + (int64_t)g * part_stride;
                    #pragma unroll
                    for (int j = 0; j < 4; j++) if (c0 + j < n) s4[j] += b[j];
                }
                uint32_t w = 0;
                #pragma unroll
                for (int j = 0; j < 4; j++) w |= reduce_line7<NM>(s4[j], t) << (8 * j);
                wt[t] = w;
            }
        }
        uint32_t P[4][G4];
        #pragma unroll
        for (int g = 0; g < G4; g++) {
            uint32_t o[4];
            transpose4x4(wt[4 * g], 4 * g + 1 < NM ? wt[4 * g + 1] : 0u, 4 * g + 2 < NM ? wt[4 * g + 2] : 0u,
                         4 * g + 3 < NM ? wt[4 * g + 3] : 0u, o);
            #pragma unroll
            for (int j = 0; j < 4; j++) P[j][g] = o[j];
        }
        const int ei = e[i];
        double* crow = C + i * ldc + c0;
        #pragma unroll
        for (int j = 0; j < 4; j++)
            if (c0 + j < n) crow[j] = crt_from_packed<NM>(P[j], ei, __ldg(f + c0 + j));
    }
}

void launch_kslice_rows(const double* A, int64_t m, int64_t k, int64_t lda, int mode, const int32_t* Eg,
                        int32_t* E_out, unsigned long long* S_out, cudaStream_t st) {
    if (m <= 0) return;
    const size_t smem = row_smem_bytes(k);
    auto kern = mode == 0 ? kslice_rows_kernel<0> : kslice_rows_kernel<1>;
    if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    (kern<<<(unsigned)m, 256, smem, st>>>(A, m, k, lda, Eg, E_out, S_out), count_launch());
}

void launch_kslice_cols(const double* B, int64_t k, int64_t n, int64_t ldb, int mode, const int32_t* Eg,
                        int32_t* E_out, unsigned long long* S_out, void* scratch, cudaStream_t st) {
    if (n <= 0) return;
    const int64_t nch = (k + KC - 1) / KC;
    unsigned long long* Sc = reinterpret_cast<unsigned long long*>(scratch);
    int32_t* Ec = reinterpret_cast<int32_t*>(Sc + nch * n);
    int32_t* bad = Ec + nch * n;
    cudaMemsetAsync(bad, 0, sizeof(int32_t) * n, st);
    if (nch > 0) {
        dim3 grid((unsigned)((n + 31) / 32), (unsigned)nch);
        if (mode == 0) (cols_stats_kernel<0><<<grid, 32 * CS_WARPS, 0, st>>>(B, k, n, ldb, Ec, Sc, bad), count_launch());
        else (cols_stats_kernel<1><<<grid, 32 * CS_WARPS, 0, st>>>(B, k, n, ldb, Ec, Sc, bad), count_launch());
    }
    (kslice_cols_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(Ec, Sc, bad, n, (int)nch, Eg, E_out, S_out), count_launch());
}

void launch_exponents_from_stats(const int32_t* E, const unsigned long long* S, int64_t cnt, int N, int mode,
                                 int kstar, int32_t* e, cudaStream_t st) {
    if (cnt <= 0) return;
    const unsigned g = (unsigned)((cnt + 255) / 256);
    if (mode == 0) (exponents_from_stats_kernel<0><<<g, 256, 0, st>>>(E, S, cnt, host_T(N), kstar, e), count_launch());
    else (exponents_from_stats_kernel<1><<<g, 256, 0, st>>>(E, S, cnt, host_T(N), kstar, e), count_launch());
}

// FAST exponents from the statistics with an explicit bound exponent T (the FP64
// prime regime's M, fp64mod.cu)
void launch_exponents_T(const int32_t* E, const unsigned long long* S, int64_t cnt, int T, int32_t* e,
                        cudaStream_t st) {
    if (cnt <= 0) return;
    (exponents_from_stats_kernel<0><<<(unsigned)((cnt + 255) / 256), 256, 0, st>>>(E, S, cnt, T, 0, e), count_launch());
}

template <int NM>
static void launch_crt_sum_nm(const uint8_t* R, int G, int64_t part_stride, int64_t m, int64_t n, const int32_t* e,
                              const int32_t* f, double* C, int64_t ldc, cudaStream_t st) {
    dim3 grid((unsigned)((n + 4 * 64 - 1) / (4 * 64)), (unsigned)(m < 65535 ? m : 65535));
    (crt_sum_kernel<NM><<<grid, 64, 0, st>>>(R, G, part_stride, m, n, e, f, C, ldc), count_launch());
}

void launch_crt_sum(const uint8_t* R, int G, int64_t part_stride, int64_t m, int64_t n, const int32_t* e,
                    const int32_t* f, int N, double* C, int64_t ldc, cudaStream_t st) {
    if (m * n == 0) return;
    OZ2_DISPATCH_N(N, launch_crt_sum_nm, R, G, part_stride, m, n, e, f, C, ldc, st);
}

}  // namespace oz2
