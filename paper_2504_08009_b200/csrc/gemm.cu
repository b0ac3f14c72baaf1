// gemm.cu -- Part 2-b of Ozaki scheme II on the sm_100a INT8 tensor cores:
// C'_t = A'_t B'_t for t = 1..N (Alg. 1 line 6), exact in int32
// for k < 2^17.
//
// One persistent kernel walks (output tile) x (all N moduli):
//   warp 0      TMA producer: 3-D tensor maps over the residue planes
//               [N][rows][ld_res] (K-major, 128-byte swizzle), a STAGES-deep
//               mbarrier ring of (A 128 x 128 B, B 256 x 128 B) stages;
//   warp 1      MMA issuer: one thread issues tcgen05.mma.cta_group::1.kind::i8
//               (M = 128, N = 256, K = 32), int32 accumulators in TMEM,
//               double-buffered (2 x 256 of the 512 TMEM columns);
//   warp 2      TMEM allocator;
//   warps 4..7  epilogue: tcgen05.ld 32x32b -> registers -> output.
#include "oz2_device.cuh"
#include "oz2_kernels.h"

namespace oz2 {
namespace gemm {

constexpr int BM = 128;             // UMMA M (one CTA)
constexpr int BN = 256;             // UMMA N
constexpr int BK = 128;             // bytes = int8 elements per stage (one 128B swizzle row)
constexpr int UK = 32;              // K per tcgen05.mma kind::i8
constexpr int STAGES = 4;
constexpr int A_BYTES = BM * BK;    // 16 KB
constexpr int B_BYTES = BN * BK;    // 32 KB
constexpr int THREADS = 256;
constexpr int EPI_WARP0 = 4;
constexpr int GROUP_M = 16;         // tile rasterisation: 16 tile-rows per group (L2 reuse of B panels)
constexpr uint32_t TMEM_COLS = 512;

struct __align__(1024) Smem {
    uint8_t a[STAGES][A_BYTES];
    uint8_t b[STAGES][B_BYTES];
    uint64_t full[STAGES];
    uint64_t empty[STAGES];
    uint64_t tfull[2];
    uint64_t tempty[2];
    uint32_t tmem_base;
};

__device__ __forceinline__ void tile_coords(int tile, int num_tm, int num_tn, int& tm, int& tn) {
    const int group = GROUP_M * num_tn;
    const int g = tile / group;
    const int first = g * GROUP_M;
    const int gm = min(num_tm - first, GROUP_M);
    const int r = tile % group;
    tm = first + r % gm;
    tn = r / gm;
}

__global__ void __launch_bounds__(THREADS, 1)
modmul_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
              int m, int n, int k, int N, int32_t* __restrict__ cprod) {
    extern __shared__ uint8_t smem_raw[];
    Smem& s = *reinterpret_cast<Smem*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    const int num_tm = (m + BM - 1) / BM, num_tn = (n + BN - 1) / BN;
    const int num_tiles = num_tm * num_tn;
    const int num_kb = (k + BK - 1) / BK;

    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tmA);
        tma_prefetch_desc(&tmB);
        for (int i = 0; i < STAGES; i++) { mbar_init(smem_u32(&s.full[i]), 1); mbar_init(smem_u32(&s.empty[i]), 1); }
        for (int i = 0; i < 2; i++) { mbar_init(smem_u32(&s.tfull[i]), 1); mbar_init(smem_u32(&s.tempty[i]), 4); }
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
            for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
                int tm, tn; tile_coords(tile, num_tm, num_tn, tm, tn);
                for (int t = 0; t < N; t++) {
                    for (int kb = 0; kb < num_kb; kb++) {
                        mbar_wait(smem_u32(&s.empty[stage]), ph ^ 1);
                        uint32_t fb = smem_u32(&s.full[stage]);
                        mbar_expect_tx(fb, A_BYTES + B_BYTES);
                        tma_load_3d(smem_u32(s.a[stage]), &tmA, fb, kb * BK, tm * BM, t);
                        tma_load_3d(smem_u32(s.b[stage]), &tmB, fb, kb * BK, tn * BN, t);
                        if (++stage == STAGES) { stage = 0; ph ^= 1; }
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ===================== MMA issuer =====================
        if (lane == 0) {
            const uint32_t idesc = idesc_i8(BM, BN);
            int stage = 0; uint32_t ph = 0;
            int acc = 0; uint32_t aph = 0;
            for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
                for (int t = 0; t < N; t++) {
                    mbar_wait(smem_u32(&s.tempty[acc]), aph ^ 1);
                    tc_fence_after();
                    const uint32_t d = tmem + (uint32_t)(acc * BN);
                    for (int kb = 0; kb < num_kb; kb++) {
                        mbar_wait(smem_u32(&s.full[stage]), ph);
                        tc_fence_after();
                        const uint32_t a0 = smem_u32(s.a[stage]), b0 = smem_u32(s.b[stage]);
                        #pragma unroll
                        for (int kk = 0; kk < BK / UK; kk++) {
                            mma_i8(d, sw128_desc(a0 + kk * UK), sw128_desc(b0 + kk * UK), idesc,
                                   (kb | kk) != 0);
                        }
                        mma_commit(smem_u32(&s.empty[stage]));      // stage free when these MMAs finish
                        if (++stage == STAGES) { stage = 0; ph ^= 1; }
                    }
                    mma_commit(smem_u32(&s.tfull[acc]));            // accumulator ready
                    if (++acc == 2) { acc = 0; aph ^= 1; }
                }
            }
        }
    } else if (warp >= EPI_WARP0) {
        // ===================== epilogue =====================
        const int q = warp & 3;                 // TMEM lane quadrant of this warp
        int acc = 0; uint32_t aph = 0;
        for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
            int tm, tn; tile_coords(tile, num_tm, num_tn, tm, tn);
            const int row = tm * BM + q * 32 + lane;
            for (int t = 0; t < N; t++) {
                mbar_wait(smem_u32(&s.tfull[acc]), aph);
                tc_fence_after();
                #pragma unroll 1
                for (int c = 0; c < BN / 32; c++) {
                    uint32_t v[32];
                    tmem_ld_32x32b_x32(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * BN + c * 32), v);
                    tmem_ld_wait();
                    const int col0 = tn * BN + c * 32;
                    if (row < m) {
                        int32_t* dst = cprod + ((int64_t)t * m + row) * n + col0;
                        if (col0 + 32 <= n && (n & 3) == 0) {
                            #pragma unroll
                            for (int j = 0; j < 32; j += 4)
                                *reinterpret_cast<int4*>(dst + j) = make_int4((int)v[j], (int)v[j + 1], (int)v[j + 2], (int)v[j + 3]);
                        } else {
                            #pragma unroll
                            for (int j = 0; j < 32; j++) if (col0 + j < n) dst[j] = (int)v[j];
                        }
                    }
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(smem_u32(&s.tempty[acc]));
                if (++acc == 2) { acc = 0; aph ^= 1; }
            }
        }
    }

    tc_fence_before();
    __syncthreads();
    if (warp == 2) tmem_dealloc(tmem, TMEM_COLS);
}

}  // namespace gemm

int launch_modmul(const CUtensorMap* tmA, const CUtensorMap* tmB, int64_t m, int64_t n, int64_t k,
                  int N, int32_t* cprod, int num_sms, cudaStream_t st) {
    using namespace gemm;
    const size_t smem = sizeof(Smem) + 1024;
    static bool attr_done[64] = {false};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 64 && !attr_done[dev]) {
        cudaError_t e = cudaFuncSetAttribute(modmul_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return (int)e;
        attr_done[dev] = true;
    }
    const int64_t tiles = ((m + BM - 1) / BM) * ((n + BN - 1) / BN);
    const int grid = (int)(tiles < num_sms ? tiles : num_sms);
    modmul_kernel<<<grid, THREADS, smem, st>>>(*tmA, *tmB, (int)m, (int)n, (int)k, N, cprod);
    return (int)cudaGetLastError();
}

}  // namespace oz2
