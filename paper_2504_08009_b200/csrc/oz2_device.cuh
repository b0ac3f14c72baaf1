// oz2_device.cuh -- device-side helpers shared by the sm_100a kernels:
// the __constant__ tables, exponent extraction, mbarrier / TMA / tcgen05 PTX.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "oz2_tables.h"

#define OZ2_EXP_NONFINITE_DEV INT32_MIN
#define OZ2_EXP_ZERO_DEV (INT32_MIN + 1)     // accu-internal: max exponent of an all-zero row/column

// per-N constants, filled once per device by api.cu; one copy per translation
// unit (static): api.cu uploads every TU's copy
static __constant__ Oz2Table c_tab[OZ2_MAX_MODULI + 1];

namespace oz2 {

// kernel launches issued by the library since load (oz2_kernel_launches):
// every launch site increments it, so a caller can count the library's own
// kernels in a timed region (bench.py's gpu_launches)
unsigned long long& launch_counter_ref();
inline void count_launch() { __atomic_add_fetch(&launch_counter_ref(), 1ull, __ATOMIC_RELAXED); }

// ---------------------------------------------------------------------------
// binary64 decomposition: x = mant * 2^ex with integer mant (exact), and
// ilogb(x) = floor(log2|x|) (correct for subnormals).  class: 0 zero,
// 1 finite non-zero, 2 Inf/NaN.
// ---------------------------------------------------------------------------
struct Dec { uint64_t mant; int ex; int ilogb; int cls; };

__device__ __forceinline__ Dec decompose(double x) {
    uint64_t b = (uint64_t)__double_as_longlong(x);
    int ef = (int)((b >> 52) & 0x7ff);
    uint64_t fr = b & 0xfffffffffffffull;
    Dec d;
    if (ef == 0x7ff) { d.cls = 2; d.mant = 0; d.ex = 0; d.ilogb = 0; return d; }
    if (ef == 0) {
        d.mant = fr; d.ex = -1074;
        d.cls = fr ? 1 : 0;
        d.ilogb = fr ? (63 - __clzll((long long)fr)) - 1074 : INT32_MIN;
    } else {
        d.mant = fr | (1ull << 52); d.ex = ef - 1075; d.cls = 1; d.ilogb = ef - 1023;
    }
    return d;
}

// x * 2^e exactly when the result is >= 1 in magnitude (two steps outside the
// normal exponent range so the first step never rounds).
__device__ __forceinline__ double scale_pow2(double x, int e) {
    if (e > 1023) {
        x *= __longlong_as_double((long long)(1023 + 1023) << 52);
        e -= 1023;
    } else if (e < -1022) {
        x *= __longlong_as_double((long long)(1) << 52);        // 2^-1022
        e += 1022;
        if (e < -1022) return 0.0 * x;                            // |result| < 1 (see R12 note)
    }
    return x * __longlong_as_double((long long)(e + 1023) << 52);
}

// ---------------------------------------------------------------------------
// shared-memory addresses, mbarriers
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_barrier_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}"
        :: "r"(bar), "r"(parity) : "memory");
}

// non-blocking: has the phase with this parity completed?
__device__ __forceinline__ bool mbar_test(uint32_t bar, uint32_t parity) {
    uint32_t done;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done) : "r"(bar), "r"(parity) : "memory");
    return done != 0;
}

// ---------------------------------------------------------------------------
// TMA (cp.async.bulk.tensor) 3-D tile load, completion on an mbarrier
// ---------------------------------------------------------------------------
__device__ __forceinline__ void tma_load_3d(uint32_t dst, const void* tmap, uint32_t bar,
                                            int c0, int c1, int c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4}], [%5];"
        :: "r"(dst), "l"((uint64_t)tmap), "r"(c0), "r"(c1), "r"(c2), "r"(bar) : "memory");
}
// bring a 3-D tile into L2 only (no shared memory, no completion)
__device__ __forceinline__ void tma_prefetch_3d(const void* tmap, int c0, int c1, int c2) {
    asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global.tile [%0, {%1, %2, %3}];"
                 :: "l"((uint64_t)tmap), "r"(c0), "r"(c1), "r"(c2) : "memory");
}
__device__ __forceinline__ void tma_prefetch_desc(const void* tmap) {
    asm volatile("prefetch.tensormap [%0];" :: "l"((uint64_t)tmap) : "memory");
}

// ---------------------------------------------------------------------------
// tcgen05: TMEM allocation, MMA, commit, loads, fences
// ---------------------------------------------------------------------------
__device__ __forceinline__ void tmem_alloc(uint32_t dst_smem, uint32_t ncols) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                 :: "r"(dst_smem), "r"(ncols) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(taddr), "r"(ncols) : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
// D[tmem] (+)= A[smem] * B[smem]^T, int8 x int8 -> int32 (kind::i8)
__device__ __forceinline__ void mma_i8(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc,
                                       uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}"
        :: "r"(d_tmem), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate) : "memory");
}
// arrive on an mbarrier when all prior tcgen05.mma of this thread complete
__device__ __forceinline__ void mma_commit(uint32_t bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                 :: "r"(bar) : "memory");
}
// 32 lanes x 32 bit, 32 consecutive columns per thread
__device__ __forceinline__ void tmem_ld_32x32b_x32(uint32_t taddr, uint32_t (&v)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
          "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]),
          "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]),
          "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
          "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]),
          "=r"(v[31])
        : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld_wait() {
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
// compiler-only fence binding registers of a tcgen05.ld already covered by a
// preceding tmem_ld_wait_regs (no instruction): their uses stay after the wait
__device__ __forceinline__ void tmem_regs_fence(uint32_t (&v)[32]) {
    asm volatile(""
                 : "+r"(v[0]), "+r"(v[1]), "+r"(v[2]), "+r"(v[3]), "+r"(v[4]), "+r"(v[5]), "+r"(v[6]),
                   "+r"(v[7]), "+r"(v[8]), "+r"(v[9]), "+r"(v[10]), "+r"(v[11]), "+r"(v[12]),
                   "+r"(v[13]), "+r"(v[14]), "+r"(v[15]), "+r"(v[16]), "+r"(v[17]), "+r"(v[18]),
                   "+r"(v[19]), "+r"(v[20]), "+r"(v[21]), "+r"(v[22]), "+r"(v[23]), "+r"(v[24]),
                   "+r"(v[25]), "+r"(v[26]), "+r"(v[27]), "+r"(v[28]), "+r"(v[29]), "+r"(v[30]),
                   "+r"(v[31])
                 :: "memory");
}
// the same wait, with the registers of an in-flight tcgen05.ld as operands so
// that no use of them can be scheduled before it (tcgen05.ld is asynchronous)
__device__ __forceinline__ void tmem_ld_wait_regs(uint32_t (&v)[32]) {
    asm volatile("tcgen05.wait::ld.sync.aligned;"
                 : "+r"(v[0]), "+r"(v[1]), "+r"(v[2]), "+r"(v[3]), "+r"(v[4]), "+r"(v[5]), "+r"(v[6]),
                   "+r"(v[7]), "+r"(v[8]), "+r"(v[9]), "+r"(v[10]), "+r"(v[11]), "+r"(v[12]),
                   "+r"(v[13]), "+r"(v[14]), "+r"(v[15]), "+r"(v[16]), "+r"(v[17]), "+r"(v[18]),
                   "+r"(v[19]), "+r"(v[20]), "+r"(v[21]), "+r"(v[22]), "+r"(v[23]), "+r"(v[24]),
                   "+r"(v[25]), "+r"(v[26]), "+r"(v[27]), "+r"(v[28]), "+r"(v[29]), "+r"(v[30]),
                   "+r"(v[31])
                 :: "memory");
}

// UMMA shared-memory descriptor, K-major, 128-byte swizzle: 8-row x 128-byte
// swizzle atoms stacked at SBO = 1024 bytes (tile base 1024-aligned).
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr & 0x3FFFFu) >> 4);          // start address  [0,14)
    d |= (uint64_t)1 << 16;                              // LBO (unused for SW128 K-major)
    d |= (uint64_t)(1024 >> 4) << 32;                    // SBO            [32,46)
    d |= (uint64_t)1 << 46;                              // version = 1    [46,48)
    d |= (uint64_t)2 << 61;                              // SWIZZLE_128B   [61,64)
    return d;
}
// K-major operand with a BK-byte swizzled row: 128B (SBO 1024) or 64B (SBO 512, layout type 4)
template <int BKB>
__device__ __forceinline__ uint64_t sw_desc(uint32_t saddr) {
    if constexpr (BKB == 128) {
        return sw128_desc(saddr);
    } else {
        static_assert(BKB == 64, "BK is 128 or 64");
        uint64_t d = 0;
        d |= (uint64_t)((saddr & 0x3FFFFu) >> 4);      // start address
        d |= (uint64_t)1 << 16;                          // LBO (unused for swizzled K-major)
        d |= (uint64_t)(512 >> 4) << 32;                 // SBO: 8 rows x 64 B
        d |= (uint64_t)1 << 46;                          // version = 1
        d |= (uint64_t)4 << 61;                          // SWIZZLE_64B
        return d;
    }
}
// instruction descriptor, kind::i8: s8 x s8 -> s32, both K-major, M x N
__host__ __device__ constexpr uint32_t idesc_i8(int M, int N, bool is_signed = true) {
    return (2u << 4)                 // c_format = S32
         | ((is_signed ? 1u : 0u) << 7)    // a_format: signed / unsigned int8
         | ((is_signed ? 1u : 0u) << 10)   // b_format: signed / unsigned int8
         | ((uint32_t)(N >> 3) << 17)
         | ((uint32_t)(M >> 4) << 24);
}

// ---------------------------------------------------------------------------
// clusters / CTA pairs (cta_group::2)
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t cluster_ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// shared::cta address -> the same variable's shared::cluster address in CTA `rank`
__device__ __forceinline__ uint32_t mapa_shared(uint32_t addr, uint32_t rank) {
    uint32_t d;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(d) : "r"(addr), "r"(rank));
    return d;
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" :: "r"(cluster_addr) : "memory");
}
// TMA load whose completion is signalled on the pair leader's mbarrier
__device__ __forceinline__ void tma_load_3d_cg2(uint32_t dst, const void* tmap, uint32_t bar_cluster,
                                                int c0, int c1, int c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4}], [%5];"
        :: "r"(dst), "l"((uint64_t)tmap), "r"(c0), "r"(c1), "r"(c2), "r"(bar_cluster) : "memory");
}
__device__ __forceinline__ void tmem_alloc_cg2(uint32_t dst_smem, uint32_t ncols) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;"
                 :: "r"(dst_smem), "r"(ncols) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc_cg2(uint32_t taddr, uint32_t ncols) {
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" :: "r"(taddr), "r"(ncols) : "memory");
}
// D[tmem, both CTAs] (+)= A[smem, both CTAs] * B[smem, both CTAs]^T  (M = 256)
__device__ __forceinline__ void mma_i8_cg2(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc,
                                           uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}"
        :: "r"(d_tmem), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate) : "memory");
}
// arrive on the mbarrier at this offset in every CTA of `mask` when the MMAs complete
__device__ __forceinline__ void mma_commit_cg2(uint32_t bar, uint16_t mask) {
    asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                 :: "r"(bar), "h"(mask) : "memory");
}

// ---------------------------------------------------------------------------
// global progress counter (keeps persistent CTAs in step for L2 reuse)
// ---------------------------------------------------------------------------
__device__ __forceinline__ void red_add_release_gpu(uint32_t* p, uint32_t v) {
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_gpu(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ uint32_t dp4a_uu(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t d;
    asm("dp4a.u32.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
    uint32_t d;
    asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(sel));
    return d;
}
// Legacy warp-level INT8 MMA (IMMA.16832.U8.U8): D = A B + C, A 16 x 32 u8
// (row), B 32 x 8 u8 (col), int32 C / D, fragment layout per the PTX ISA
// (groupID g = lane / 4, t = lane % 4): a0 = A[g][4t..4t+3], a1 = A[g+8][4t..],
// a2 = A[g][16+4t..], a3 = A[g+8][16+4t..]; b0 = B[4t..4t+3][g], b1 =
// B[16+4t..][g]; c0, c1 = C[g][2t, 2t+1], c2, c3 = C[g+8][2t, 2t+1].
// Used for the residue byte dot products (scale.cu), not for the GEMM.
__device__ __forceinline__ void imma_u8(uint32_t (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                        uint32_t b0, uint32_t b1, uint32_t c0, uint32_t c1, uint32_t c2,
                                        uint32_t c3) {
    asm("mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%10,%11,%12,%13};"
        : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1), "r"(c0), "r"(c1), "r"(c2), "r"(c3));
}

// low bytes of four 32-bit values -> one word (byte i from v_i)
__device__ __forceinline__ uint32_t pack_lo_bytes(uint32_t v0, uint32_t v1, uint32_t v2, uint32_t v3) {
    uint32_t a = prmt(v0, v1, 0x0040u);
    uint32_t b = prmt(v2, v3, 0x0040u);
    return prmt(a, b, 0x5410u);
}

}  // namespace oz2
