// gemm.cu -- Part 2 of Ozaki scheme II on the sm_100a INT8 tensor cores:
// C'_t = A'_t B'_t for t = 1..N (Alg. 1 line 6), exact in int32
// for k < 2^17, and -- in the FUSED mode used by
// oz2_dgemm -- lines 7-10 in the epilogue, so no int32 product leaves the chip.
//
// One persistent kernel, warp-specialised:
//   warp 0       TMA producer: 3-D tensor maps over the residue planes
//                [N][rows][ld_res] (K-major, 128-byte swizzle) into a
//                STAGES-deep mbarrier ring of (A 128 x 128 B, B 256 x 128 B);
//   warp 1       MMA issuer: one thread issues tcgen05.mma.cta_group::1.kind::i8
//                (M = 128, N = 256, K = 32) into int32 TMEM accumulators,
//                double-buffered (2 x 256 of the 512 TMEM columns);
//   warp 2       TMEM allocator;
//   warps 4..11  epilogue (2 warps per TMEM lane quadrant, 4 column chunks each):
//                RAW:   tcgen05.ld -> int32 C'_t to global (split API);
//                FUSED: tcgen05.ld -> c''_t = C'_t mod m_t (line 7) -> uint8
//                scratch; at t = N-1 the tile's N residues are combined by the
//                exact CRT (lines 8-9) and scaled (line 10) straight into C.
//
// Schedule ("modulus-outer groups"): output tiles are grouped by GROUP_TM tile
// rows; for each group, for t = 1..N, the CTAs sweep the group's tiles (tile j
// -> CTA j mod grid, every t).  All CTAs therefore work on the same modulus at
// the same time, the group's A_t panels stay in L2 across the sweep, and every
// tile is finalised by the CTA (and the threads) that wrote its residues.
#include "oz2_device.cuh"
#include "oz2_kernels.h"

#include <algorithm>
#include <stdlib.h>

namespace oz2 {
namespace gemm {

constexpr int BM = 128;             // UMMA M (one CTA)
constexpr int BN = 256;             // UMMA N
constexpr int BK = 128;             // bytes = int8 elements per stage (one 128B swizzle row)
constexpr int UK = 32;              // K per tcgen05.mma kind::i8
constexpr int STAGES = 4;
constexpr int A_BYTES = BM * BK;    // 16 KB
constexpr int B_BYTES = BN * BK;    // 32 KB
constexpr int EPI_WARPS = 8;
constexpr int THREADS = 128 + 32 * EPI_WARPS;
constexpr int EPI_WARP0 = 4;
constexpr int GROUP_TM = 16;        // tile rows per schedule group (2048 rows of A)
constexpr uint32_t TMEM_COLS = 512;
constexpr int TILE_BYTES = BM * BN; // one uint8 residue tile

struct __align__(1024) Smem {
    uint8_t a[STAGES][A_BYTES];
    uint8_t b[STAGES][B_BYTES];
    uint64_t full[STAGES];
    uint64_t empty[STAGES];
    uint64_t tfull[2];
    uint64_t tempty[2];
    uint32_t tmem_base;
};

struct Params {
    int m, n, k, N;
    int num_tm, num_tn, num_kb;
    int max_slots;                  // tiles per CTA per group (scratch slots)
    int group_tm;                   // tile rows per schedule group
    int tile_major;                 // 1: all N moduli of a tile back to back
    int32_t* cprod;                 // RAW: [N][m][n]
    uint8_t* scratch;               // FUSED: [grid][max_slots][N][BM*BN]
    double* C;                      // FUSED
    int64_t ldc;
    const int32_t* e;
    const int32_t* f;
};

// Visit every work unit (tm, tn, t, slot) of this CTA in schedule order.
//  modulus-outer (default): for each group of group_tm tile rows, for t, for the
//    group's tiles j = blockIdx.x + i * gridDim.x (slot i);
//  tile-major: for each tile j = blockIdx.x + i * gridDim.x (grouped raster), for t (slot 0).
template <typename F>
__device__ __forceinline__ void for_each_unit(const Params& p, F&& fn) {
    if (p.tile_major) {
        const int tiles = p.num_tm * p.num_tn;
        for (int j = blockIdx.x; j < tiles; j += gridDim.x) {
            const int gsz = p.group_tm * p.num_tn;
            const int g0 = (j / gsz) * p.group_tm;
            const int gtm = min(p.group_tm, p.num_tm - g0);
            const int jj = j % gsz;
            for (int t = 0; t < p.N; t++) fn(g0 + jj % gtm, jj / gtm, t, 0);
        }
        return;
    }
    for (int g0 = 0; g0 < p.num_tm; g0 += p.group_tm) {
        const int gtm = min(p.group_tm, p.num_tm - g0);
        const int gtiles = gtm * p.num_tn;
        for (int t = 0; t < p.N; t++) {
            int slot = 0;
            for (int j = blockIdx.x; j < gtiles; j += gridDim.x, slot++) {
                const int tm = g0 + j % gtm;        // consecutive CTAs share the B panel (tn)
                const int tn = j / gtm;
                fn(tm, tn, t, slot);
            }
        }
    }
}

// --------------------------------------------------------------------------
// FUSED epilogue helpers
// --------------------------------------------------------------------------
// 32 reduced residues (bytes) of one modulus -> 8 words
template <int NM>
__device__ __forceinline__ void reduce32(const uint32_t (&v)[32], int t, uint32_t (&w)[8]) {
    #pragma unroll
    for (int q = 0; q < 8; q++) {
        uint32_t r0 = reduce_line7<NM>((int32_t)v[4 * q + 0], t);
        uint32_t r1 = reduce_line7<NM>((int32_t)v[4 * q + 1], t);
        uint32_t r2 = reduce_line7<NM>((int32_t)v[4 * q + 2], t);
        uint32_t r3 = reduce_line7<NM>((int32_t)v[4 * q + 3], t);
        w[q] = r0 | (r1 << 8) | (r2 << 16) | (r3 << 24);
    }
}

template <int NM>
__global__ void __launch_bounds__(THREADS, 1)
modmul_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
              const Params p) {
    constexpr bool FUSED = NM > 0;
    extern __shared__ uint8_t smem_raw[];
    Smem& s = *reinterpret_cast<Smem*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tmA);
        tma_prefetch_desc(&tmB);
        for (int i = 0; i < STAGES; i++) { mbar_init(smem_u32(&s.full[i]), 1); mbar_init(smem_u32(&s.empty[i]), 1); }
        for (int i = 0; i < 2; i++) { mbar_init(smem_u32(&s.tfull[i]), 1); mbar_init(smem_u32(&s.tempty[i]), EPI_WARPS); }
        fence_barrier_init();
    }
    if (warp == 2) tmem_alloc(smem_u32(&s.tmem_base), TMEM_COLS);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = s.tmem_base;

    if (warp == 0) {
        // ===================== TMA producer =====================
        if (lane == 0) {
            int stage = 0; uint32_t ph = 0;
            for_each_unit(p, [&](int tm, int tn, int t, int) {
                for (int kb = 0; kb < p.num_kb; kb++) {
                    mbar_wait(smem_u32(&s.empty[stage]), ph ^ 1);
                    const uint32_t fb = smem_u32(&s.full[stage]);
                    mbar_expect_tx(fb, A_BYTES + B_BYTES);
                    tma_load_3d(smem_u32(s.a[stage]), &tmA, fb, kb * BK, tm * BM, t);
                    tma_load_3d(smem_u32(s.b[stage]), &tmB, fb, kb * BK, tn * BN, t);
                    if (++stage == STAGES) { stage = 0; ph ^= 1; }
                }
            });
        }
    } else if (warp == 1) {
        // ===================== MMA issuer =====================
        if (lane == 0) {
            const uint32_t idesc = idesc_i8(BM, BN);
            int stage = 0; uint32_t ph = 0;
            int acc = 0; uint32_t aph = 0;
            for_each_unit(p, [&](int, int, int, int) {
                mbar_wait(smem_u32(&s.tempty[acc]), aph ^ 1);
                tc_fence_after();
                const uint32_t d = tmem + (uint32_t)(acc * BN);
                for (int kb = 0; kb < p.num_kb; kb++) {
                    mbar_wait(smem_u32(&s.full[stage]), ph);
                    tc_fence_after();
                    const uint32_t a0 = smem_u32(s.a[stage]), b0 = smem_u32(s.b[stage]);
                    #pragma unroll
                    for (int kk = 0; kk < BK / UK; kk++)
                        mma_i8(d, sw128_desc(a0 + kk * UK), sw128_desc(b0 + kk * UK), idesc, (kb | kk) != 0);
                    mma_commit(smem_u32(&s.empty[stage]));       // stage reusable when these MMAs finish
                    if (++stage == STAGES) { stage = 0; ph ^= 1; }
                }
                mma_commit(smem_u32(&s.tfull[acc]));             // accumulator ready
                if (++acc == 2) { acc = 0; aph ^= 1; }
            });
        }
    } else if (warp >= EPI_WARP0) {
        // ===================== epilogue =====================
        const int q = warp & 3;                           // TMEM lane quadrant
        const int half = (warp - EPI_WARP0) >> 2;         // column chunks [4*half, 4*half+4)
        const int r = q * 32 + lane;                      // row within the tile
        int acc = 0; uint32_t aph = 0;
        for_each_unit(p, [&](int tm, int tn, int t, int slot) {
            mbar_wait(smem_u32(&s.tfull[acc]), aph);
            tc_fence_after();
            const int row = tm * BM + r;
            const uint32_t tbase = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * BN);
            if constexpr (!FUSED) {
                #pragma unroll 1
                for (int cc = 0; cc < 4; cc++) {
                    const int c = half * 4 + cc;
                    uint32_t v[32];
                    tmem_ld_32x32b_x32(tbase + (uint32_t)(c * 32), v);
                    tmem_ld_wait();
                    const int col0 = tn * BN + c * 32;
                    if (row < p.m) {
                        int32_t* dst = p.cprod + ((int64_t)t * p.m + row) * p.n + col0;
                        if (col0 + 32 <= p.n && (p.n & 3) == 0) {
                            #pragma unroll
                            for (int j = 0; j < 32; j += 4)
                                *reinterpret_cast<int4*>(dst + j) =
                                    make_int4((int)v[j], (int)v[j + 1], (int)v[j + 2], (int)v[j + 3]);
                        } else {
                            #pragma unroll
                            for (int j = 0; j < 32; j++) if (col0 + j < p.n) dst[j] = (int)v[j];
                        }
                    }
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(smem_u32(&s.tempty[acc]));
            } else {
                // line 7 for the 4 chunks -> uint8 residues in this tile's scratch slot
                uint8_t* tile_scr = p.scratch + (((size_t)blockIdx.x * p.max_slots + slot) * NM) * TILE_BYTES;
                #pragma unroll
                for (int cc = 0; cc < 4; cc++) {
                    const int c = half * 4 + cc;
                    uint32_t v[32], w[8];
                    tmem_ld_32x32b_x32(tbase + (uint32_t)(c * 32), v);
                    tmem_ld_wait();
                    reduce32<NM>(v, t, w);
                    uint4* d4 = reinterpret_cast<uint4*>(tile_scr + (size_t)t * TILE_BYTES + ((size_t)(c * BM + r)) * 32);
                    d4[0] = make_uint4(w[0], w[1], w[2], w[3]);
                    d4[1] = make_uint4(w[4], w[5], w[6], w[7]);
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(smem_u32(&s.tempty[acc]));   // TMEM buffer free
                if (t == NM - 1 && row < p.m) {
                    // lines 8-10: exact CRT of the tile's N residues, scaled into C
                    const int ei = __ldg(p.e + row);
                    #pragma unroll 1
                    for (int cc = 0; cc < 4; cc++) {
                        const int c = half * 4 + cc;
                        const int col0 = tn * BN + c * 32;
                        if (col0 >= p.n) continue;
                        #pragma unroll 1
                        for (int hh = 0; hh < 4; hh++) {           // 8 columns at a time
                            uint32_t wt[NM][2];
                            #pragma unroll
                            for (int tt = 0; tt < NM; tt++) {
                                const uint2 x = *reinterpret_cast<const uint2*>(
                                    tile_scr + (size_t)tt * TILE_BYTES + ((size_t)(c * BM + r)) * 32 + hh * 8);
                                wt[tt][0] = x.x; wt[tt][1] = x.y;
                            }
                            double* crow = p.C + (int64_t)row * p.ldc + col0 + hh * 8;
                            const int ncol = p.n - (col0 + hh * 8);
                            const bool vec = ncol >= 8 && ((reinterpret_cast<uintptr_t>(crow) & 15) == 0);
                            #pragma unroll
                            for (int j = 0; j < 8; j += 2) {
                                double o[2];
                                #pragma unroll
                                for (int jj = 0; jj < 2; jj++) {
                                    uint32_t res[NM];
                                    #pragma unroll
                                    for (int tt = 0; tt < NM; tt++)
                                        res[tt] = (wt[tt][(j + jj) >> 2] >> (8 * ((j + jj) & 3))) & 0xffu;
                                    const int col = col0 + hh * 8 + j + jj;
                                    const int fj = col < p.n ? __ldg(p.f + col) : 0;
                                    o[jj] = crt_from_residues<NM>(res, ei, fj);
                                }
                                if (vec) {
                                    *reinterpret_cast<double2*>(crow + j) = make_double2(o[0], o[1]);
                                } else {
                                    if (j < ncol) crow[j] = o[0];
                                    if (j + 1 < ncol) crow[j + 1] = o[1];
                                }
                            }
                        }
                    }
                }
            }
            if (++acc == 2) { acc = 0; aph ^= 1; }
        });
    }

    tc_fence_before();
    __syncthreads();
    if (warp == 2) tmem_dealloc(tmem, TMEM_COLS);
}

template <int NM>
static int launch_nm(const CUtensorMap* tmA, const CUtensorMap* tmB, const Params& p, int grid, cudaStream_t st) {
    const size_t smem = sizeof(Smem) + 1024;
    static bool attr_done[64] = {false};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 64 && !attr_done[dev]) {
        cudaError_t e = cudaFuncSetAttribute(modmul_kernel<NM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return (int)e;
        attr_done[dev] = true;
    }
    modmul_kernel<NM><<<grid, THREADS, smem, st>>>(*tmA, *tmB, p);
    return (int)cudaGetLastError();
}

}  // namespace gemm

static int env_int(const char* name, int dflt) {
    const char* v = getenv(name);
    return v && *v ? atoi(v) : dflt;
}

static gemm::Params make_params(int64_t m, int64_t n, int64_t k, int N, int num_sms, int* grid_out) {
    using namespace gemm;
    Params p{};
    p.m = (int)m; p.n = (int)n; p.k = (int)k; p.N = N;
    p.num_tm = (int)((m + BM - 1) / BM);
    p.num_tn = (int)((n + BN - 1) / BN);
    p.num_kb = (int)((k + BK - 1) / BK);
    p.group_tm = std::max(1, env_int("OZ2_GROUP_TM", GROUP_TM));     // tuning knobs (experiments)
    p.tile_major = env_int("OZ2_TILE_MAJOR", 0);
    const int gtiles = p.tile_major ? p.num_tm * p.num_tn : std::min(p.group_tm, p.num_tm) * p.num_tn;
    const int grid = gtiles < num_sms ? gtiles : num_sms;
    p.max_slots = p.tile_major ? 1 : (gtiles + grid - 1) / grid;
    *grid_out = grid;
    return p;
}

size_t fused_scratch_bytes(int64_t m, int64_t n, int N, int num_sms) {
    int grid;
    gemm::Params p = make_params(m, n, 1, N, num_sms, &grid);
    return (size_t)grid * p.max_slots * N * gemm::TILE_BYTES;
}

int launch_modmul(const CUtensorMap* tmA, const CUtensorMap* tmB, int64_t m, int64_t n, int64_t k,
                  int N, int32_t* cprod, int num_sms, cudaStream_t st) {
    int grid;
    gemm::Params p = make_params(m, n, k, N, num_sms, &grid);
    p.cprod = cprod;
    return gemm::launch_nm<0>(tmA, tmB, p, grid, st);
}

int launch_modmul_fused(const CUtensorMap* tmA, const CUtensorMap* tmB, int64_t m, int64_t n, int64_t k,
                        int N, uint8_t* scratch, const int32_t* e, const int32_t* f, double* C, int64_t ldc,
                        int num_sms, cudaStream_t st) {
    int grid;
    gemm::Params p = make_params(m, n, k, N, num_sms, &grid);
    p.scratch = scratch; p.e = e; p.f = f; p.C = C; p.ldc = ldc;
    switch (N) {
#define OZ2_CASE(NN) case NN: return gemm::launch_nm<NN>(tmA, tmB, p, grid, st);
        OZ2_CASE(2) OZ2_CASE(3) OZ2_CASE(4) OZ2_CASE(5) OZ2_CASE(6) OZ2_CASE(7) OZ2_CASE(8)
        OZ2_CASE(9) OZ2_CASE(10) OZ2_CASE(11) OZ2_CASE(12) OZ2_CASE(13) OZ2_CASE(14) OZ2_CASE(15)
        OZ2_CASE(16) OZ2_CASE(17) OZ2_CASE(18) OZ2_CASE(19) OZ2_CASE(20)
#undef OZ2_CASE
        default: return (int)cudaErrorInvalidValue;
    }
}

}  // namespace oz2
