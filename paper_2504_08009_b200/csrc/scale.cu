// scale.cu -- Part 1 and Part 2-a of Ozaki scheme II on sm_100a:
// Alg. 1 lines 1-5: exponent vectors e (rows of A) and f
// (columns of B), A' = trunc(D A), B' = trunc(B E), and the N symmetric int8
// residue planes (Eq. 11).
//
// Exponent rule FAST (reading R4): for each chunk of KC = 256
// consecutive inner indices, E_c = max ilogb|x| and S_c = sum u^2 with
// u = ceil(|x| 2^(15-E_c)) (>= 1 for x != 0); then E = max E_c,
// S = sum ceil(S_c / 4^(E-E_c)), h = min{h : S <= 4^h}, e = T + 15 - E - h.
// All integer, so the result does not depend on the reduction order.
//
// Residues: x = trunc(2^e a) as a 64-bit (N <= 16) or 96-bit (N > 16) two's
// complement integer; for odd m_t, y = sum_b byte_b(x) (2^(8b) mod m_t) with
// dp4a (+ (-2^64) mod m_t when x < 0), q = floor((y + h_t)/m_t) by a magic
// multiply, r = y - q m_t in [-h_t, h_t] (Eq. 1 for odd m); for m_1 = 256 the
// residue is the low byte of x (Eq. 1 tie 128 -> -128 = int8 wrap).
#include "oz2_device.cuh"
#include "oz2_kernels.h"

#include <stdlib.h>

#include <algorithm>

namespace oz2 {

constexpr int KC = 256;            // FAST chunk length (reading R4)
constexpr int MAX_CHUNKS = 4096;   // k < 2^20 (OZ2 max k; chunk statistics live in shared memory)

__device__ __forceinline__ uint64_t ceil_shift(uint64_t S, int sh) {
    if (S == 0) return 0;
    if (sh >= 64) return 1;
    return (S + ((1ull << sh) - 1)) >> sh;
}

// h = min{h >= 0 : S <= 4^h}
__device__ __forceinline__ int log4_ceil(uint64_t S) {
    if (S <= 1) return 0;
    int bl = 64 - __clzll((long long)(S - 1));
    return (bl + 1) / 2;
}

__device__ __forceinline__ int warp_max(int v) {
    #pragma unroll
    for (int o = 16; o; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ uint64_t warp_sum64(uint64_t v) {
    #pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// ---------------------------------------------------------------------------
// Residues of one integer x, |x| < 2^62 (WORDS = 2) or < 2^94 (WORDS = 3),
// held as U = x + 2^63 (resp. 2^95) in 32-bit words: the bias makes U >= 0, so
// y = G_t + sum_b byte_b(U) (2^(8b) mod m_t) == x (mod m_t) with the per-modulus
// constant G_t = (-2^63) mod m_t, 0 <= y < 2^20; then the symmetric residue of
// Eq. (1) is y - m_t floor((y + h_t) / m_t) in [-h_t, h_t], where the floor is
// one 64-bit multiply-add ((y magic_t + h_t magic_t) >> 32, exact since
// (y + h_t)(magic_t m_t - 2^32) < 2^32).  The low byte is the int8 residue.
// ---------------------------------------------------------------------------
//
// q = rint(y / m_t) (= floor((y + h_t) / m_t) for odd m_t) is formed on the
// full-rate FP32 pipe instead of a quarter-rate IMAD.HI (measured on sm_100a,
// tools/mb/op_rates.cu: IDP, IMAD 2 cycles per warp instruction and SMSP,
// IMAD.HI 4, FFMA / FADD 1): the dp4a addend carries 0x4B000000, so the bits
// of y' = 0x4B000000 + y are the binary32 2^23 + y (y < 2^20), f = y' - 2^23
// is y exactly, and one FMA f * RN(1/m_t) + 1.5 2^23 rounds to 1.5 2^23 +
// rint(y / m_t): the product's error is below y 2^-24 / m_t < 2^-4 / m_t,
// while y / m_t lies at least 1 / (2 m_t) from every half-integer (m_t odd).
// Then y - q m_t = y' + qb (2^32 - m_t) - (0x4B000000 - 0x4B400000 m_t), and
// that constant is 0 mod 256, so the low byte is the residue.
// (tools/mb/residue_pipes.cu: 114 vs 145 cycles per warp-element at N = 14,
// bitwise equal.)
template <int NM, int WORDS>
__device__ __forceinline__ uint32_t residue_odd(int t, const uint32_t (&w)[3]) {
    const Oz2Table& T = c_tab[NM];
    uint32_t y = dp4a_uu(w[0], T.cw[0][t], WORDS == 2 ? T.G63f[t] : T.G95f[t]);
    y = dp4a_uu(w[1], T.cw[1][t], y);
    if (WORDS == 3) y = dp4a_uu(w[2], T.cw[2][t], y);
    const float f = __fsub_rn(__uint_as_float(y), 8388608.0f);                      // y, exact
    const uint32_t qb = __float_as_uint(__fmaf_rn(f, T.invm[t], 12582912.0f));      // 1.5 2^23 + q
    return qb * T.negm[t] + y;                                  // low byte: y - q m_t (mod 256)
}

// ---------------------------------------------------------------------------
// The same residues with the byte dot products on the (otherwise idle) tensor
// cores: one legacy warp-level IMMA (m16n8k32, u8 x u8 -> s32) computes, for 64
// elements of a warp (2 per thread) and 2 moduli, y = G_t + sum_b byte_b(U)
// c_(t,b).  Fragment mapping (imma_u8): thread (g, tq) puts its element E0's
// words into A row g and E1's into row g + 8, at K slot tq (bytes 0-3 at K =
// 4 tq.., bytes 4-7 at K = 16 + 4 tq..) -- exactly the a0..a3 registers, no
// data movement.  Column n = 2 slot + mm of B holds c_(t_mm, b) at the K
// positions of `slot` and 0 elsewhere, so C[g][2 tq + mm] is y of this
// thread's own element and modulus t_mm: the accumulator fragment c0..c3 holds
// (E0, t0), (E0, t1), (E1, t0), (E1, t1).  C (the bias G_t) enters as the MMA's
// addend.  96-bit inputs (N > 16) chain a second IMMA over bytes 8-11.
// One IMMA replaces 4 dp4a per thread (8 for 96-bit); the symmetric reduction
// and the byte packing stay on the integer pipes.
// ---------------------------------------------------------------------------
constexpr int MAX_PAIRS = OZ2_MAX_MODULI / 2;

// Integer widths of the residue inputs x = trunc(2^e a) (the launcher picks the
// narrowest that holds the line-1 rule's bound on |x|):
//   BW_7:  |x| < 2^55: U = x + 2^55 in bytes 0-6, byte 7 := 1, and B carries the
//          bias correction (-2^55 mod m_t) at byte 7 -- the MMA's addend is 0, so
//          no accumulator set-up per MMA (FAST / EQ17 with N <= 14: T <= 54);
//   BW_8:  |x| < 2^63: U = x + 2^63, the correction G63_t as the MMA's addend;
//   BW_12: |x| < 2^95: U = x + 2^95 in 12 bytes (two chained MMAs), G95_t.
constexpr int BW_7 = 7, BW_8 = 8, BW_12 = 12;
template <int BW> struct BwWords { static constexpr int value = BW == BW_12 ? 3 : 2; };

// B fragments of every (N, width class, modulus pair (t0, t1) = (1 + 2p, 2 + 2p),
// lane): the same for every warp and CTA, built once per device by
// init_bfrag_kernel (api.cu, after the tables) and read with one cached 8- or
// 12-byte load per pair and lane
static __device__ uint32_t g_bfrag[OZ2_MAX_MODULI + 1][2][MAX_PAIRS][32][3];

__device__ __forceinline__ uint32_t pow2_mod(int e, uint32_t m) {
    uint32_t r = 1 % m;
    for (int i = 0; i < e; i++) r = (r * 2u) % m;
    return r;
}

__global__ void init_bfrag_kernel() {
    const int NM = blockIdx.x, b7 = blockIdx.y;
    if (NM < 2) return;
    const Oz2Table& T = c_tab[NM];
    for (int x = threadIdx.x; x < (NM / 2) * 32; x += blockDim.x) {
        const int p = x >> 5, l = x & 31, g = l >> 2, tq = l & 3;
        const int t = 1 + 2 * p + (g & 1);
        const bool sel = tq == (g >> 1) && t < NM;
        uint32_t v[3] = {0u, 0u, 0u};
        if (sel) {
            for (int w = 0; w < 3; w++) v[w] = T.cw[w][t];
            if (b7) {                                      // BW_7: byte 7 of U is 1, its weight is the bias term
                const uint32_t m = (uint32_t)T.m[t];
                const uint32_t g55 = (m - pow2_mod(55, m)) % m;
                v[1] = (v[1] & 0x00ffffffu) | (g55 << 24);
            }
        }
        for (int w = 0; w < 3; w++) g_bfrag[NM][b7][p][l][w] = v[w];
    }
}

void launch_init_bfrag(cudaStream_t st) {
    (init_bfrag_kernel<<<dim3(OZ2_MAX_MODULI + 1, 2), 128, 0, st>>>(), count_launch());
}

template <int NM>
__device__ __forceinline__ uint32_t sym_residue(uint32_t y, int t) {
    const Oz2Table& T = c_tab[NM];
    const uint32_t q = (uint32_t)(((uint64_t)y * T.magic[t] + T.hmagic[t]) >> 32);
    return q * T.negm[t] + y;                                   // y - q m_t (mod 2^32)
}

// The IMMA A operand of element pair (E0, E1) as one register quad, in the
// fragment order {bytes 0-3 of E0, of E1, bytes 4-7 of E0, of E1} (plus, for
// 12-byte inputs, {bytes 8-11 of E0, of E1, 0, 0}): built once by to_quad and
// reused by every modulus pair.
template <int BW>
struct EQuad {
    uint32_t a[4];
    uint32_t b[4];          // BW_12 only
};

// One A quad (two elements, fragment order as residues_imma) against NP modulus
// pairs' B fragments in ONE asm statement: the quad stays in its registers for
// all NP MMAs (separate statements let ptxas copy it before every MMA), the
// accumulator addend is RZ (the 7-byte width puts the bias into B).
template <int NP>
__device__ __forceinline__ void imma_block(uint32_t (&d)[4 * NP], const uint32_t (&a)[4], const uint32_t (&b)[2 * NP]) {
    if constexpr (NP == 1) {
        asm(
        "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {0,0,0,0};\n\t"
            : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3])
            : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
    } else if constexpr (NP == 2) {
        asm(
        "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%8,%9,%10,%11}, {%12,%13}, {0,0,0,0};\n\t"
        "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%4,%5,%6,%7}, {%8,%9,%10,%11}, {%14,%15}, {0,0,0,0};\n\t"
            : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3]), "=r"(d[4]), "=r"(d[5]), "=r"(d[6]), "=r"(d[7])
            : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]), "r"(b[2]), "r"(b[3]));
    } else if constexpr (NP == 3) {
        asm(
        "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%12,%13,%14,%15}, {%16,%17}, {0,0,0,0};\n\t"
        "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%4,%5,%6,%7}, {%12,%13,%14,%15}, {%18,%19}, {0,0,0,0};\n\t"
        "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%8,%9,%10,%11}, {%12,%13,%14,%15}, {%20,%21}, {0,0,0,0};\n\t"
            : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3]), "=r"(d[4]), "=r"(d[5]), "=r"(d[6]), "=r"(d[7]), "=r"(d[8]), "=r"(d[9]), "=r"(d[10]), "=r"(d[11])
            : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]), "r"(b[2]), "r"(b[3]), "r"(b[4]), "r"(b[5]));
    } else if constexpr (NP == 4) {
        asm(
        "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%16,%17,%18,%19}, {%20,%21}, {0,0,0,0};\n\t"
        "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%4,%5,%6,%7}, {%16,%17,%18,%19}, {%22,%23}, {0,0,0,0};\n\t"
        "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%8,%9,%10,%11}, {%16,%17,%18,%19}, {%24,%25}, {0,0,0,0};\n\t"
        "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%12,%13,%14,%15}, {%16,%17,%18,%19}, {%26,%27}, {0,0,0,0};\n\t"
            : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3]), "=r"(d[4]), "=r"(d[5]), "=r"(d[6]), "=r"(d[7]), "=r"(d[8]), "=r"(d[9]), "=r"(d[10]), "=r"(d[11]), "=r"(d[12]), "=r"(d[13]), "=r"(d[14]), "=r"(d[15])
            : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]), "r"(b[2]), "r"(b[3]), "r"(b[4]), "r"(b[5]), "r"(b[6]), "r"(b[7]));
    } else if constexpr (NP == 5) {
        asm(
        "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%20,%21,%22,%23}, {%24,%25}, {0,0,0,0};\n\t"
        "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%4,%5,%6,%7}, {%20,%21,%22,%23}, {%26,%27}, {0,0,0,0};\n\t"
        "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%8,%9,%10,%11}, {%20,%21,%22,%23}, {%28,%29}, {0,0,0,0};\n\t"
        "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%12,%13,%14,%15}, {%20,%21,%22,%23}, {%30,%31}, {0,0,0,0};\n\t"
        "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%16,%17,%18,%19}, {%20,%21,%22,%23}, {%32,%33}, {0,0,0,0};\n\t"
            : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3]), "=r"(d[4]), "=r"(d[5]), "=r"(d[6]), "=r"(d[7]), "=r"(d[8]), "=r"(d[9]), "=r"(d[10]), "=r"(d[11]), "=r"(d[12]), "=r"(d[13]), "=r"(d[14]), "=r"(d[15]), "=r"(d[16]), "=r"(d[17]), "=r"(d[18]), "=r"(d[19])
            : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]), "r"(b[2]), "r"(b[3]), "r"(b[4]), "r"(b[5]), "r"(b[6]), "r"(b[7]), "r"(b[8]), "r"(b[9]));
    } else if constexpr (NP == 6) {
        asm(
        "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%24,%25,%26,%27}, {%28,%29}, {0,0,0,0};\n\t"
        "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%4,%5,%6,%7}, {%24,%25,%26,%27}, {%30,%31}, {0,0,0,0};\n\t"
        "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%8,%9,%10,%11}, {%24,%25,%26,%27}, {%32,%33}, {0,0,0,0};\n\t"
        "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%12,%13,%14,%15}, {%24,%25,%26,%27}, {%34,%35}, {0,0,0,0};\n\t"
        "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%16,%17,%18,%19}, {%24,%25,%26,%27}, {%36,%37}, {0,0,0,0};\n\t"
        "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%20,%21,%22,%23}, {%24,%25,%26,%27}, {%38,%39}, {0,0,0,0};\n\t"
            : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3]), "=r"(d[4]), "=r"(d[5]), "=r"(d[6]), "=r"(d[7]), "=r"(d[8]), "=r"(d[9]), "=r"(d[10]), "=r"(d[11]), "=r"(d[12]), "=r"(d[13]), "=r"(d[14]), "=r"(d[15]), "=r"(d[16]), "=r"(d[17]), "=r"(d[18]), "=r"(d[19]), "=r"(d[20]), "=r"(d[21]), "=r"(d[22]), "=r"(d[23])
            : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]), "r"(b[2]), "r"(b[3]), "r"(b[4]), "r"(b[5]), "r"(b[6]), "r"(b[7]), "r"(b[8]), "r"(b[9]), "r"(b[10]), "r"(b[11]));
    } else if constexpr (NP == 7) {
        asm(
        "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%28,%29,%30,%31}, {%32,%33}, {0,0,0,0};\n\t"
        "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%4,%5,%6,%7}, {%28,%29,%30,%31}, {%34,%35}, {0,0,0,0};\n\t"
        "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%8,%9,%10,%11}, {%28,%29,%30,%31}, {%36,%37}, {0,0,0,0};\n\t"
        "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%12,%13,%14,%15}, {%28,%29,%30,%31}, {%38,%39}, {0,0,0,0};\n\t"
        "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%16,%17,%18,%19}, {%28,%29,%30,%31}, {%40,%41}, {0,0,0,0};\n\t"
        "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%20,%21,%22,%23}, {%28,%29,%30,%31}, {%42,%43}, {0,0,0,0};\n\t"
        "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%24,%25,%26,%27}, {%28,%29,%30,%31}, {%44,%45}, {0,0,0,0};\n\t"
            : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3]), "=r"(d[4]), "=r"(d[5]), "=r"(d[6]), "=r"(d[7]), "=r"(d[8]), "=r"(d[9]), "=r"(d[10]), "=r"(d[11]), "=r"(d[12]), "=r"(d[13]), "=r"(d[14]), "=r"(d[15]), "=r"(d[16]), "=r"(d[17]), "=r"(d[18]), "=r"(d[19]), "=r"(d[20]), "=r"(d[21]), "=r"(d[22]), "=r"(d[23]), "=r"(d[24]), "=r"(d[25]), "=r"(d[26]), "=r"(d[27])
            : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]), "r"(b[2]), "r"(b[3]), "r"(b[4]), "r"(b[5]), "r"(b[6]), "r"(b[7]), "r"(b[8]), "r"(b[9]), "r"(b[10]), "r"(b[11]), "r"(b[12]), "r"(b[13]));
    }
}

// residues for t = 1..NM-1 of the 2 * NQ elements held as quads q[0..NQ) (NQ
// even); store(t, pw[NQ/2]) receives the int8 residues of modulus t packed 4 per
// word in element order (element 2i, 2i+1 of quad i).  Every lane of the warp
// must call it (mma.sync).  Loop order: for each group of 4 elements (2 quads)
// all modulus pairs back to back, so each A quad feeds its NM/2 MMAs in a row
// and stays in its registers (the other order made ptxas copy the quads into
// fresh registers before every MMA).
template <int NM, int BW, int NQ, typename Store>
__device__ __forceinline__ void residues_imma(const EQuad<BW> (&q)[NQ], Store&& store) {
    static_assert(NQ % 2 == 0, "4 elements per packed word");
    constexpr int NP = NM / 2;
    const Oz2Table& T = c_tab[NM];
    const int lane = threadIdx.x & 31;
    const uint32_t* bf = &g_bfrag[NM][BW == BW_7 ? 1 : 0][0][lane][0];
    if constexpr (BW == BW_7) {
        // all NP pairs of one quad in one asm statement (imma_block); the B
        // fragments stay live in registers for the thread's NQ quads
        uint32_t b[2 * NP];
        #pragma unroll
        for (int p = 0; p < NP; p++) { b[2 * p] = __ldg(bf + p * 96); b[2 * p + 1] = __ldg(bf + p * 96 + 1); }
        uint32_t pw[NM][NQ / 2];
        #pragma unroll
        for (int u = 0; u < NQ / 2; u++) {
            uint32_t half[NM];                             // modulus t: bytes of elements 4u, 4u + 1
            #pragma unroll
            for (int h = 0; h < 2; h++) {
                uint32_t d[4 * NP];
                imma_block<NP>(d, q[2 * u + h].a, b);
                #pragma unroll
                for (int p = 0; p < NP; p++) {
                    const int t0 = 1 + 2 * p, t1 = t0 + 1;
                    const uint32_t r0a = sym_residue<NM>(d[4 * p], t0), r0b = sym_residue<NM>(d[4 * p + 2], t0);
                    if (h == 0) half[t0] = prmt(r0a, r0b, 0x0040u);
                    else pw[t0][u] = prmt(half[t0], prmt(r0a, r0b, 0x0040u), 0x5410u);
                    if (t1 < NM) {
                        const uint32_t r1a = sym_residue<NM>(d[4 * p + 1], t1), r1b = sym_residue<NM>(d[4 * p + 3], t1);
                        if (h == 0) half[t1] = prmt(r1a, r1b, 0x0040u);
                        else pw[t1][u] = prmt(half[t1], prmt(r1a, r1b, 0x0040u), 0x5410u);
                    }
                }
            }
        }
        #pragma unroll
        for (int t = 1; t < NM; t++) store(t, pw[t]);
        return;
    }
    uint32_t pw[NM][NQ / 2];                           // pw[t][u]: modulus t, elements 4u..4u+3
    #pragma unroll
    for (int u = 0; u < NQ / 2; u++) {
        #pragma unroll
        for (int p = 0; p < NP; p++) {
            const int t0 = 1 + 2 * p, t1 = t0 + 1;
            const bool two = t1 < NM;
            const uint32_t b0 = __ldg(bf + p * 96), b1 = __ldg(bf + p * 96 + 1);
            const uint32_t b2 = BW == BW_12 ? __ldg(bf + p * 96 + 2) : 0u;
            const uint32_t g0 = BW == BW_7 ? 0u : (BW == BW_8 ? T.G63[t0] : T.G95[t0]);
            const uint32_t g1 = BW == BW_7 || !two ? 0u : (BW == BW_8 ? T.G63[t1] : T.G95[t1]);
            uint32_t r0[4], r1[4];
            #pragma unroll
            for (int h = 0; h < 2; h++) {
                const EQuad<BW>& e = q[2 * u + h];
                uint32_t d[4];
                imma_u8(d, e.a[0], e.a[1], e.a[2], e.a[3], b0, b1, g0, g1, g0, g1);
                if (BW == BW_12) {
                    uint32_t d2[4];
                    imma_u8(d2, e.b[0], e.b[1], e.b[2], e.b[3], b2, 0u, d[0], d[1], d[2], d[3]);
                    #pragma unroll
                    for (int x = 0; x < 4; x++) d[x] = d2[x];
                }
                r0[2 * h] = sym_residue<NM>(d[0], t0);
                r0[2 * h + 1] = sym_residue<NM>(d[2], t0);
                if (two) {
                    r1[2 * h] = sym_residue<NM>(d[1], t1);
                    r1[2 * h + 1] = sym_residue<NM>(d[3], t1);
                }
            }
            pw[t0][u] = pack_lo_bytes(r0[0], r0[1], r0[2], r0[3]);
            if (two) pw[t1][u] = pack_lo_bytes(r1[0], r1[1], r1[2], r1[3]);
        }
    }
    #pragma unroll
    for (int t = 1; t < NM; t++) store(t, pw[t]);
}

// 2^e as the product s1 * s2 of two doubles (the two multiplications of
// scale_pow2, hoisted out of the per-element loops: x s1 s2 is bitwise
// scale_pow2(x, e) for every finite x)
__device__ __forceinline__ void pow2_factors(int e, double& s1, double& s2) {
    if (e > 1023) {
        s1 = __longlong_as_double((long long)(1023 + 1023) << 52);    // 2^1023
        s2 = __longlong_as_double((long long)(e - 1023 + 1023) << 52);
    } else if (e < -1022) {
        s1 = __longlong_as_double((long long)1 << 52);                // 2^-1022
        s2 = e + 1022 < -1022 ? 0.0 : __longlong_as_double((long long)(e + 1022 + 1023) << 52);
    } else {
        s1 = __longlong_as_double((long long)(e + 1023) << 52);
        s2 = 1.0;
    }
}

// U = trunc(2^e a) + 2^63 (WORDS = 2) or + 2^95 (WORDS = 3) as words, with
// 2^e = s1 s2 (pow2_factors); a = 0 for rows / columns of the exponent sentinel
template <int WORDS>
__device__ __forceinline__ void to_words(double a, double s1, double s2, uint32_t (&w)[3]) {
    double v = (a * s1) * s2;
    if (WORDS == 2) {
        const long long x = __double2ll_rz(v);                  // trunc
        w[0] = (uint32_t)x;
        w[1] = (uint32_t)((unsigned long long)x >> 32) ^ 0x80000000u;
        w[2] = 0;
    } else {
        v = trunc(v);
        const double hi = floor(v * 0x1p-32);                   // exact
        const double lo = fma(-hi, 0x1p32, v);                  // exact, in [0, 2^32)
        const long long h = __double2ll_rz(hi);
        w[0] = __double2uint_rz(lo);
        w[1] = (uint32_t)h;
        w[2] = (uint32_t)((unsigned long long)h >> 32) ^ 0x80000000u;
    }
}

// elements a0, a1 -> their IMMA quad (BW_8 / BW_12: the words of to_words;
// BW_7: U = x + 2^55 with byte 7 set to 1, x in [-2^55, 2^55))
template <int BW>
__device__ __forceinline__ void to_quad(double a0, double a1, double s1, double s2, EQuad<BW>& q) {
    if (BW == BW_7) {
        const long long x0 = __double2ll_rz((a0 * s1) * s2), x1 = __double2ll_rz((a1 * s1) * s2);
        q.a[0] = (uint32_t)x0;
        q.a[1] = (uint32_t)x1;
        q.a[2] = (uint32_t)((unsigned long long)x0 >> 32) + 0x01800000u;   // + 2^23 (the bias), byte 7 := 1
        q.a[3] = (uint32_t)((unsigned long long)x1 >> 32) + 0x01800000u;
        return;
    }
    constexpr int W = BwWords<BW>::value;
    uint32_t w0[3], w1[3];
    to_words<W>(a0, s1, s2, w0);
    to_words<W>(a1, s1, s2, w1);
    q.a[0] = w0[0]; q.a[1] = w1[0]; q.a[2] = w0[1]; q.a[3] = w1[1];
    if (BW == BW_12) { q.b[0] = w0[2]; q.b[1] = w1[2]; q.b[2] = 0u; q.b[3] = 0u; }
}

// ---------------------------------------------------------------------------
// memory helpers: L2 eviction-priority policies, streaming stores
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint64_t l2_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t l2_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ double2 ld2_hint(const double* a, uint64_t pol) {
    double2 v;
    asm volatile("ld.global.nc.L2::cache_hint.v2.f64 {%0,%1}, [%2], %3;" : "=d"(v.x), "=d"(v.y) : "l"(a), "l"(pol));
    return v;
}
__device__ __forceinline__ double ld1_hint(const double* a, uint64_t pol) {
    double v;
    asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(a), "l"(pol));
    return v;
}
__device__ __forceinline__ void st_cs_v2(void* a, uint32_t x, uint32_t y) {
    asm volatile("st.global.cs.v2.b32 [%0], {%1, %2};" :: "l"(a), "r"(x), "r"(y) : "memory");
}
// predicated forms (no branch around the store)
__device__ __forceinline__ void st_cs_b32_if(bool p, void* a, uint32_t x) {
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q st.global.cs.b32 [%0], %1;\n\t}"
                 :: "l"(a), "r"(x), "r"((int)p) : "memory");
}
__device__ __forceinline__ void st_cs_v2_if(bool p, void* a, uint32_t x, uint32_t y) {
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %3, 0;\n\t@q st.global.cs.v2.b32 [%0], {%1, %2};\n\t}"
                 :: "l"(a), "r"(x), "r"(y), "r"((int)p) : "memory");
}
__device__ __forceinline__ void st_cs_v4_if(bool p, void* a, uint32_t x, uint32_t y, uint32_t z, uint32_t w) {
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %5, 0;\n\t@q st.global.cs.v4.b32 [%0], {%1, %2, %3, %4};\n\t}"
                 :: "l"(a), "r"(x), "r"(y), "r"(z), "r"(w), "r"((int)p) : "memory");
}
__device__ __forceinline__ void st_cs_v4(void* a, uint32_t x, uint32_t y, uint32_t z, uint32_t w) {
    asm volatile("st.global.cs.v4.b32 [%0], {%1, %2, %3, %4};" :: "l"(a), "r"(x), "r"(y), "r"(z), "r"(w) : "memory");
}

// ---------------------------------------------------------------------------
// FAST-rule chunk statistics
//   E_c = ilogb(max |x|): |x| orders like its bit pattern, so take the max of
//   the sign-cleared bits (Inf/NaN patterns are larger than every finite one);
//   S_c = sum u^2, u = ceil(|x| 2^(15-E_c)) (>= 1 for x != 0) in FP64: every u
//   <= 2^16, so u^2 <= 2^32 and a 256-term sum <= 2^40 are exact.
// ---------------------------------------------------------------------------
#ifndef OZ2_ROW_CU
#define OZ2_ROW_CU 2             // KC-chunks per warp step in the rows' pass 1 (loads in flight)
#endif
constexpr uint64_t ABS_MASK = 0x7fffffffffffffffull;
constexpr uint64_t INF_BITS = 0x7ff0000000000000ull;

__device__ __forceinline__ int ilogb_bits(uint64_t b) {      // b != 0, finite, sign clear
    const int ef = (int)(b >> 52);
    return ef ? ef - 1023 : (63 - __clzll((long long)b)) - 1074;
}
__device__ __forceinline__ uint64_t warp_max64(uint64_t v) {
    #pragma unroll
    for (int o = 16; o; o >>= 1) {
        const uint64_t w = __shfl_xor_sync(0xffffffffu, v, o);
        v = w > v ? w : v;
    }
    return v;
}
__device__ __forceinline__ double warp_sumd(double v) {
    #pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
// 2^(15 - Ec) as s1 * s2 (s2 != 1 only for chunks of subnormals)
__device__ __forceinline__ void u_scale(int Ec, double& s1, double& s2) {
    const int sh = 15 - Ec;
    if (sh <= 1000) { s1 = __longlong_as_double((long long)(sh + 1023) << 52); s2 = 1.0; }
    else { s1 = 0x1p1000; s2 = __longlong_as_double((long long)(sh - 1000 + 1023) << 52); }
}
// u^2 as an exact integer: u = ceil(|x| 2^(15-E_c)) with the product rounded
// UPWARD (exact whenever it is >= 2^-1022; a nonzero product that underflows
// stays > 0), then ceil to an integer in one conversion (cvt.rpi.u32.f64): so
// u >= 1 for every x != 0 and u = 0 for x = 0, which is the rule's
// max(1, ceil(.)) without a compare; u <= 2^16, u^2 <= 2^32 in 64-bit integers
__device__ __forceinline__ uint64_t u_sq(double x, double s1, double s2) {
    const uint32_t u = __double2uint_ru(__dmul_ru(__dmul_ru(fabs(x), s1), s2));
    return (uint64_t)u * u;
}
// the same for s2 = 1 (every chunk whose maximum is a normal number >= 2^-1008)
__device__ __forceinline__ uint64_t u_sq1(double x, double s1) {
    const uint32_t u = __double2uint_ru(__dmul_ru(fabs(x), s1));
    return (uint64_t)u * u;
}

// per-row chunk statistics in dynamic shared memory: Sc[nch], Ec[nch], then bad, e
struct RowSmem {
    unsigned long long* Sc;
    int* Ec;
    int* misc;                        // [0] = bad, [1] = e
};
__host__ __device__ inline size_t row_smem_bytes(int64_t k) {
    const int64_t nch = (k + KC - 1) / KC;
    return (size_t)(nch > 0 ? nch : 1) * (sizeof(unsigned long long) + sizeof(int)) + 2 * sizeof(int);
}

// combine chunk statistics (warp 0): e = T + 15 - E - h, or EQ17 / zero / non-finite
template <int MODE>
__device__ __forceinline__ int combine_chunks(const int* Ec, const unsigned long long* Sc, int nch, int bad,
                                              int Tb, int kstar) {
    const int lane = threadIdx.x & 31;
    int E = INT32_MIN;
    for (int c = lane; c < nch; c += 32) E = max(E, Ec[c]);
    E = warp_max(E);
    int e;
    if (E == INT32_MIN) {
        e = 0;                                                // zero row / column
    } else if (MODE == 0) {
        uint64_t S = 0;
        for (int c = lane; c < nch; c += 32)
            if (Ec[c] != INT32_MIN) S += ceil_shift(Sc[c], 2 * (E - Ec[c]));
        S = warp_sum64(S);
        e = Tb + 15 - E - log4_ceil(S);
    } else {
        e = kstar - 1 - E;                                    // EQ17 (reading R5)
    }
    return bad ? OZ2_EXP_NONFINITE_DEV : e;
}

// chunk statistics of one row (CTA-wide) into sm (E_c, S_c per chunk, the
// non-finite flag); loads keep the row in L2 (evict_last) for the residue pass
template <int MODE>
__device__ void row_chunk_stats(const double* __restrict__ X, int64_t k, RowSmem& sm) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nwarps = blockDim.x >> 5;
    const int nch = (int)((k + KC - 1) / KC);
    const bool vec = ((reinterpret_cast<uintptr_t>(X) & 15) == 0);
    const uint64_t pol = l2_evict_last();
    if (threadIdx.x == 0) sm.misc[0] = 0;
    __syncthreads();
    // CU chunks per warp and step (c, c + nwarps, ...): all their loads are in
    // flight before the first reduction.  The chunk maximum comes from the high
    // words of |x| (exponent field; >= 0x7ff00000 flags Inf/NaN); a chunk whose
    // maximum is subnormal or zero takes the full 64-bit patterns (warp-uniform)
    constexpr int CU = OZ2_ROW_CU, VP = KC / 32;
    for (int c0 = warp; c0 < nch; c0 += CU * nwarps) {
        double v[CU][VP];
        #pragma unroll
        for (int u = 0; u < CU; u++) {
            const int c = c0 + u * nwarps;
            const int64_t base = (int64_t)c * KC;
            if (c < nch && vec && base + KC <= k) {
                #pragma unroll
                for (int j = 0; j < VP / 2; j++) {
                    const double2 p = ld2_hint(X + base + 2 * lane + 64 * j, pol);
                    v[u][2 * j] = p.x; v[u][2 * j + 1] = p.y;
                }
            } else {
                #pragma unroll
                for (int j = 0; j < VP; j++) {
                    const int64_t l = base + lane + 32 * j;
                    v[u][j] = (c < nch && l < k) ? ld1_hint(X + l, pol) : 0.0;
                }
            }
        }
        uint32_t mh[CU];
        #pragma unroll
        for (int u = 0; u < CU; u++) {
            mh[u] = 0;
            #pragma unroll
            for (int j = 0; j < VP; j++) mh[u] = max(mh[u], (uint32_t)__double2hiint(v[u][j]) & 0x7fffffffu);
        }
        #pragma unroll
        for (int o = 16; o; o >>= 1) {
            #pragma unroll
            for (int u = 0; u < CU; u++) mh[u] = max(mh[u], __shfl_xor_sync(0xffffffffu, mh[u], o));
        }
        int Ec[CU];
        uint64_t S[CU];
        #pragma unroll
        for (int u = 0; u < CU; u++) {
            S[u] = 0;
            if (mh[u] >= (uint32_t)(INF_BITS >> 32)) {
                Ec[u] = INT32_MIN;
                if (lane == 0 && c0 + u * nwarps < nch) sm.misc[0] = 1;
            } else if (mh[u] >= 0x00100000u) {
                Ec[u] = (int)(mh[u] >> 20) - 1023;
            } else {
                uint64_t mb = 0;
                #pragma unroll
                for (int j = 0; j < VP; j++) {
                    const uint64_t b = (uint64_t)__double_as_longlong(v[u][j]) & ABS_MASK;
                    mb = b > mb ? b : mb;
                }
                mb = warp_max64(mb);
                Ec[u] = mb != 0 ? ilogb_bits(mb) : INT32_MIN;
            }
            if (MODE == 0 && Ec[u] != INT32_MIN) {
                double s1, s2;
                u_scale(Ec[u], s1, s2);
                if (s2 == 1.0) {                              // warp-uniform (one chunk per warp)
                    #pragma unroll
                    for (int j = 0; j < VP; j++) S[u] += u_sq1(v[u][j], s1);
                } else {
                    #pragma unroll
                    for (int j = 0; j < VP; j++) S[u] += u_sq(v[u][j], s1, s2);
                }
            }
        }
        if (MODE == 0) {
            #pragma unroll
            for (int o = 16; o; o >>= 1) {
                #pragma unroll
                for (int u = 0; u < CU; u++) S[u] += __shfl_xor_sync(0xffffffffu, S[u], o);
            }
        }
        #pragma unroll
        for (int u = 0; u < CU; u++) {
            const int c = c0 + u * nwarps;
            if (lane == 0 && c < nch) { sm.Ec[c] = Ec[u]; sm.Sc[c] = S[u]; }
        }
    }
    __syncthreads();
}

// exponent of one row (CTA-wide), first pass over the row
template <int MODE>
__device__ int row_exponent(const double* __restrict__ X, int64_t k, int Tb, int kstar, RowSmem& sm) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    row_chunk_stats<MODE>(X, k, sm);
    if (warp == 0) {
        const int e = combine_chunks<MODE>(sm.Ec, sm.Sc, (int)((k + KC - 1) / KC), sm.misc[0], Tb, kstar);
        if (lane == 0) sm.misc[1] = e;
    }
    __syncthreads();
    return sm.misc[1];
}

// residues of one row for all N moduli: planes out[t][l], RV elements per
// thread per step (RV = 16: 128 B of loads, one 16-byte streaming store per
// modulus; the plane row stride is a multiple of 16, so the last step may write
// residues of zeros into [k, round_up(k, 16)), inside the row's ld_res bytes)
constexpr int RV = 16;
template <int NM, int WORDS>
__device__ void row_residues(const double* __restrict__ X, int64_t k, int e, int8_t* __restrict__ out,
                             int64_t plane_stride) {
    const bool vec = ((reinterpret_cast<uintptr_t>(X) & 15) == 0);
    const uint64_t pol = l2_evict_first();
    const int64_t step = RV * (int64_t)blockDim.x;
    if (e == OZ2_EXP_NONFINITE_DEV) {                 // x = 0: every residue is 0
        for (int64_t l0 = RV * (int64_t)threadIdx.x; l0 < k; l0 += step)
            #pragma unroll 1
            for (int t = 0; t < NM; t++) st_cs_v4(out + t * plane_stride + l0, 0u, 0u, 0u, 0u);
        return;
    }
    double s1, s2;
    pow2_factors(e, s1, s2);
    for (int64_t l0 = RV * (int64_t)threadIdx.x; l0 < k; l0 += step) {
        double a[RV];
        if (vec && l0 + RV <= k) {
            #pragma unroll
            for (int j = 0; j < RV / 2; j++) {
                const double2 p = ld2_hint(X + l0 + 2 * j, pol);
                a[2 * j] = p.x; a[2 * j + 1] = p.y;
            }
        } else {
            #pragma unroll
            for (int j = 0; j < RV; j++) a[j] = (l0 + j < k) ? ld1_hint(X + l0 + j, pol) : 0.0;
        }
        uint32_t w[RV][3];
        #pragma unroll
        for (int j = 0; j < RV; j++) to_words<WORDS>(a[j], s1, s2, w[j]);
        int8_t* o = out + l0;
        // t = 0: m = 256, the low byte of x
        st_cs_v4(o, pack_lo_bytes(w[0][0], w[1][0], w[2][0], w[3][0]), pack_lo_bytes(w[4][0], w[5][0], w[6][0], w[7][0]),
                 pack_lo_bytes(w[8][0], w[9][0], w[10][0], w[11][0]), pack_lo_bytes(w[12][0], w[13][0], w[14][0], w[15][0]));
        #pragma unroll
        for (int t = 1; t < NM; t++) {
            uint32_t r[RV];
            #pragma unroll
            for (int j = 0; j < RV; j++) r[j] = residue_odd<NM, WORDS>(t, w[j]);
            o += plane_stride;
            st_cs_v4(o, pack_lo_bytes(r[0], r[1], r[2], r[3]), pack_lo_bytes(r[4], r[5], r[6], r[7]),
                     pack_lo_bytes(r[8], r[9], r[10], r[11]), pack_lo_bytes(r[12], r[13], r[14], r[15]));
        }
    }
}

#ifndef OZ2_RES_IMMA
// 1: the byte dot products of the 7-byte width on the legacy IMMA path.  Measured
// (round 2, tools/gpu/ab_conv.sh, 16384^2, N = 14): bitwise-correct, rows equal
// to dp4a (1.87 vs 1.87-1.90 ms, 93 instructions per element either way: the
// dp4a savings go to register moves that ptxas inserts around every MMA), the
// column kernel slower (2.03 vs 1.73 ms: 80 registers, lower occupancy on a
// latency-bound kernel).  Default 0 (dp4a); kept as a build option.
#define OZ2_RES_IMMA 0
#endif
// the byte dot products on the IMMA path for the 7-byte width (the headline N
// <= 14 with FAST / EQ17 exponents), dp4a otherwise (OZ2_RES_IMMA=0: always dp4a)
template <int BW>
struct UseImma { static constexpr bool value = OZ2_RES_IMMA && BW == BW_7; };
#ifndef OZ2_COLS_IMMA
#define OZ2_COLS_IMMA 0          // the column kernel on the IMMA path too (measured slower: see section 7)
#endif
template <int BW>
struct UseImmaCols { static constexpr bool value = OZ2_COLS_IMMA && UseImma<BW>::value; };

// residues of RPT elements a[] of this thread (scale 2^e = s1 s2) for all NM
// moduli; put(t, pw[RPT/4]) receives modulus t's bytes packed 4 per word.  On
// the IMMA path every lane of the warp must call it.
template <int NM, int BW, int RPT, typename Put>
__device__ __forceinline__ void thread_residues(const double (&a)[RPT], double s1, double s2, Put&& put) {
    if constexpr (UseImmaCols<BW>::value) {
        EQuad<BW> eq[RPT / 2];
        #pragma unroll
        for (int q = 0; q < RPT / 2; q++) to_quad<BW>(a[2 * q], a[2 * q + 1], s1, s2, eq[q]);
        uint32_t pw[RPT / 4];                                     // t = 0: m = 256, the low byte
        #pragma unroll
        for (int u = 0; u < RPT / 4; u++)
            pw[u] = pack_lo_bytes(eq[2 * u].a[0], eq[2 * u].a[1], eq[2 * u + 1].a[0], eq[2 * u + 1].a[1]);
        put(0, pw);
        residues_imma<NM, BW, RPT / 2>(eq, put);
    } else {
        constexpr int WORDS = BwWords<BW>::value;
        uint32_t w[RPT][3];
        #pragma unroll
        for (int q = 0; q < RPT; q++) to_words<WORDS>(a[q], s1, s2, w[q]);
        {
            uint32_t pw[RPT / 4];                                 // t = 0: m = 256, the low byte
            #pragma unroll
            for (int u = 0; u < RPT / 4; u++)
                pw[u] = pack_lo_bytes(w[4 * u][0], w[4 * u + 1][0], w[4 * u + 2][0], w[4 * u + 3][0]);
            put(0, pw);
        }
        #pragma unroll
        for (int t = 1; t < NM; t++) {
            uint32_t pw[RPT / 4];
            #pragma unroll
            for (int u = 0; u < RPT / 4; u++)
                pw[u] = pack_lo_bytes(residue_odd<NM, WORDS>(t, w[4 * u]), residue_odd<NM, WORDS>(t, w[4 * u + 1]),
                                      residue_odd<NM, WORDS>(t, w[4 * u + 2]), residue_odd<NM, WORDS>(t, w[4 * u + 3]));
            put(t, pw);
        }
    }
}

// row_residues with the IMMA byte dots: the same output; RVI elements per thread
// and step; the loop runs while any lane of the warp has elements left (mma.sync
// needs the whole warp), lanes past the row convert zeros and do not store
#ifndef OZ2_ROW_RVI
#define OZ2_ROW_RVI 8
#endif
template <int NM, int BW>
__device__ void row_residues_imma(const double* __restrict__ X, int64_t k, int e, int8_t* __restrict__ out,
                                  int64_t plane_stride) {
    constexpr int RVI = OZ2_ROW_RVI;
    static_assert(RVI == 4 || RVI == 8 || RVI == 16, "4, 8 or 16 elements per thread");
    const bool vec = ((reinterpret_cast<uintptr_t>(X) & 15) == 0);
    const uint64_t pol = l2_evict_first();
    const int64_t step = RVI * (int64_t)blockDim.x;
    const int64_t warp0 = RVI * (int64_t)(threadIdx.x & ~31);
    const int64_t ldr = (k + 15) & ~(int64_t)15;
    if (e == OZ2_EXP_NONFINITE_DEV) {                 // x = 0: every residue is 0
        for (int64_t l0 = RV * (int64_t)threadIdx.x; l0 < k; l0 += RV * (int64_t)blockDim.x)
            #pragma unroll 1
            for (int t = 0; t < NM; t++) st_cs_v4(out + t * plane_stride + l0, 0u, 0u, 0u, 0u);
        return;
    }
    double s1, s2;
    pow2_factors(e, s1, s2);
    #pragma unroll 1
    for (int64_t base = warp0; base < k; base += step) {
        const int64_t l0 = base + RVI * (int64_t)(threadIdx.x & 31);
        double a[RVI];
        if (vec && l0 + RVI <= k) {
            #pragma unroll
            for (int j = 0; j < RVI / 2; j++) {
                const double2 p = ld2_hint(X + l0 + 2 * j, pol);
                a[2 * j] = p.x; a[2 * j + 1] = p.y;
            }
        } else {
            #pragma unroll
            for (int j = 0; j < RVI; j++) a[j] = (l0 + j < k) ? ld1_hint(X + l0 + j, pol) : 0.0;
        }
        EQuad<BW> q[RVI / 2];
        if (s2 == 1.0) {                              // block-uniform (one exponent per row)
            #pragma unroll
            for (int j = 0; j < RVI / 2; j++) to_quad<BW>(a[2 * j], a[2 * j + 1], s1, 1.0, q[j]);
        } else {
            #pragma unroll
            for (int j = 0; j < RVI / 2; j++) to_quad<BW>(a[2 * j], a[2 * j + 1], s1, s2, q[j]);
        }
        const bool live = l0 < ldr;                   // l0 is a multiple of RVI: whole pieces
        int8_t* o = out + l0;                          // walks the planes: t = 0, 1, 2, ... in order
        auto put = [&](int t, const uint32_t (&pw)[RVI / 4]) {
            if (t) o += plane_stride;
            if constexpr (RVI == 16) st_cs_v4_if(live, o, pw[0], pw[1], pw[2], pw[3]);
            else if constexpr (RVI == 8) st_cs_v2_if(live, o, pw[0], pw[1]);
            else st_cs_b32_if(live, o, pw[0]);
        };
        {                                              // t = 0: m = 256, the low byte of x
            uint32_t pw[RVI / 4];
            #pragma unroll
            for (int u = 0; u < RVI / 4; u++)
                pw[u] = pack_lo_bytes(q[2 * u].a[0], q[2 * u].a[1], q[2 * u + 1].a[0], q[2 * u + 1].a[1]);
            put(0, pw);
        }
        residues_imma<NM, BW, RVI / 2>(q, put);
    }
}

// ---------------------------------------------------------------------------
// Row kernels (A: m x k, row-major, lda); one CTA per row
// ---------------------------------------------------------------------------
// what: 1 = exponents, 2 = residues (given e), 3 = both
#ifndef OZ2_ROW_THREADS
#define OZ2_ROW_THREADS 256      // threads per row CTA (256 or 512)
#endif
#ifndef OZ2_ROW_MINB
#define OZ2_ROW_MINB 4          // resident 256-thread row CTAs per SM for N <= 16 (64 registers; A/B round 2: 1.58 -> 1.55 ms vs 3); 96-bit inputs (N > 16) keep 3
#endif
template <int NM, int BW, int MODE, int THREADS>
__global__ void __launch_bounds__(THREADS, (THREADS == 256 ? (NM <= 16 ? OZ2_ROW_MINB : 3) : (NM <= 16 ? 2 : 1)))
rows_kernel(const double* __restrict__ A, int64_t m, int64_t k, int64_t lda, int what, int kstar,
            int32_t* __restrict__ e_io, int8_t* __restrict__ res, int64_t ldr, int64_t pstride) {
    constexpr int WORDS = BwWords<BW>::value;
    extern __shared__ __align__(16) unsigned char row_smem[];
    const int64_t nch = (k + KC - 1) / KC;
    RowSmem sm;
    sm.Sc = reinterpret_cast<unsigned long long*>(row_smem);
    sm.Ec = reinterpret_cast<int*>(row_smem + sizeof(unsigned long long) * (nch > 0 ? nch : 1));
    sm.misc = sm.Ec + (nch > 0 ? nch : 1);
    // rows blockIdx.x, + gridDim.x, ...: a grid of a few CTAs per SM keeps the
    // rows in flight (x 8k bytes) small enough that pass 2 re-reads them from L2
    for (int64_t i = blockIdx.x; i < m; i += gridDim.x) {
        const double* X = A + i * lda;
        int e;
        if (what & 1) {
            e = row_exponent<MODE>(X, k, c_tab[NM].T, kstar, sm);
            if (threadIdx.x == 0) e_io[i] = e;
        } else {
            e = e_io[i];
        }
        if constexpr (UseImma<BW>::value) {
            if (what & 2) row_residues_imma<NM, BW>(X, k, e, res + i * ldr, pstride);
        } else {
            if (what & 2) row_residues<NM, WORDS>(X, k, e, res + i * ldr, pstride);
        }
    }
}

// A' = trunc(D A) as FP64 (split API)
__global__ void trunc_rows_kernel(const double* __restrict__ A, int64_t m, int64_t k, int64_t lda,
                                  const int32_t* __restrict__ e, double* __restrict__ out) {
    int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (idx >= m * k) return;
    int64_t i = idx / k, l = idx % k;
    int ei = e[i];
    out[idx] = ei == OZ2_EXP_NONFINITE_DEV ? 0.0 : trunc(scale_pow2(A[i * lda + l], ei));
}

// ---------------------------------------------------------------------------
// Column kernels (B: k x n, row-major, ldb)
// ---------------------------------------------------------------------------
// chunk statistics: block = 32 columns x one KC chunk; 16 warps x 16 rows.
// The chunk maximum is taken over the high words of |x| (one 32-bit max per
// element): they order like |x| and carry the exponent field, so they give E_c
// and the Inf/NaN flag directly; only a column chunk whose maximum is subnormal
// (or zero) needs the full 64-bit patterns (ilogb of a subnormal depends on its
// leading mantissa bit), which a second, block-uniform pass supplies.
#ifndef OZ2_CS_WARPS
#define OZ2_CS_WARPS 8           // warps per column-statistics CTA, 32 rows per thread (A/B round 2: 0.465 -> 0.368 ms vs 16, 0.434 with 4)
#endif
constexpr int CS_WARPS = OZ2_CS_WARPS;
constexpr int CS_RPT = KC / CS_WARPS;
template <int MODE>
__global__ void __launch_bounds__(32 * CS_WARPS)
cols_stats_kernel(const double* __restrict__ B, int64_t k, int64_t n, int64_t ldb,
                  int32_t* __restrict__ Ec_out, unsigned long long* __restrict__ Sc_out,
                  int32_t* __restrict__ bad_out) {
    __shared__ uint32_t sHi[CS_WARPS][32];
    __shared__ unsigned long long sMax[CS_WARPS][32];
    __shared__ unsigned long long sS[CS_WARPS][32];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t j = (int64_t)blockIdx.x * 32 + lane;
    const int64_t c = blockIdx.y;
    const int64_t r0 = c * KC + warp * CS_RPT;
    const uint64_t pol = l2_evict_first();
    const double* src = B + r0 * ldb + j;
    double v[CS_RPT];
    if (j < n && r0 + CS_RPT <= k) {
        #pragma unroll
        for (int q = 0; q < CS_RPT; q++) v[q] = ld1_hint(src + q * ldb, pol);
    } else {
        #pragma unroll
        for (int q = 0; q < CS_RPT; q++) v[q] = (j < n && r0 + q < k) ? ld1_hint(src + q * ldb, pol) : 0.0;
    }
    uint32_t mh = 0;
    #pragma unroll
    for (int q = 0; q < CS_RPT; q++) mh = max(mh, (uint32_t)__double2hiint(v[q]) & 0x7fffffffu);
    sHi[warp][lane] = mh;
    __syncthreads();
    uint32_t ch = 0;
    #pragma unroll
    for (int w = 0; w < CS_WARPS; w++) ch = max(ch, sHi[w][lane]);
    int Ec;
    bool bad = false;
    if (ch >= (uint32_t)(INF_BITS >> 32)) {
        bad = true; Ec = INT32_MIN;
    } else if (ch >= 0x00100000u) {
        Ec = (int)(ch >> 20) - 1023;                          // normal maximum
    } else {
        Ec = INT32_MIN;                                       // zero or subnormal: below
    }
    // block-uniform: some column's chunk maximum is subnormal (or the chunk is zero)
    if (__syncthreads_or(ch < 0x00100000u)) {
        uint64_t mb = 0;
        #pragma unroll
        for (int q = 0; q < CS_RPT; q++) {
            const uint64_t b = (uint64_t)__double_as_longlong(v[q]) & ABS_MASK;
            mb = b > mb ? b : mb;
        }
        sMax[warp][lane] = mb;
        __syncthreads();
        if (ch < 0x00100000u) {
            uint64_t cm = 0;
            #pragma unroll
            for (int w = 0; w < CS_WARPS; w++) cm = sMax[w][lane] > cm ? sMax[w][lane] : cm;
            Ec = cm != 0 ? ilogb_bits(cm) : INT32_MIN;
        }
    }
    uint64_t S = 0;
    double s1 = 1.0, s2 = 1.0;
    if (Ec != INT32_MIN) u_scale(Ec, s1, s2);
    const bool one = __all_sync(0xffffffffu, s2 == 1.0);      // every lane votes (zero chunks too)
    if (MODE == 0 && Ec != INT32_MIN) {
        if (one) {
            #pragma unroll
            for (int q = 0; q < CS_RPT; q++) S += u_sq1(v[q], s1);
        } else {
            #pragma unroll
            for (int q = 0; q < CS_RPT; q++) S += u_sq(v[q], s1, s2);
        }
    }
    sS[warp][lane] = S;
    __syncthreads();
    if (warp == 0 && j < n) {
        uint64_t St = 0;
        #pragma unroll
        for (int w = 0; w < CS_WARPS; w++) St += sS[w][lane];
        Ec_out[c * n + j] = Ec;
        Sc_out[c * n + j] = St;
        if (bad) atomicOr(bad_out + j, 1);
    }
}

template <int MODE>
__global__ void cols_finalize_kernel(const int32_t* __restrict__ Ec, const unsigned long long* __restrict__ Sc,
                                     const int32_t* __restrict__ bad, int64_t n, int nch, int Tb, int kstar,
                                     int32_t* __restrict__ f) {
    int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (j >= n) return;
    int E = INT32_MIN;
    for (int c = 0; c < nch; c++) E = max(E, Ec[(int64_t)c * n + j]);
    int e;
    if (MODE == 2) {                                  // accu: the raw max exponent (zero column marked)
        f[j] = bad[j] ? OZ2_EXP_NONFINITE_DEV : (E == INT32_MIN ? OZ2_EXP_ZERO_DEV : E);
        return;
    }
    if (E == INT32_MIN) {
        e = 0;
    } else if (MODE == 0) {
        uint64_t S = 0;
        for (int c = 0; c < nch; c++) {
            int Ecc = Ec[(int64_t)c * n + j];
            if (Ecc != INT32_MIN) S += ceil_shift(Sc[(int64_t)c * n + j], 2 * (E - Ecc));
        }
        e = Tb + 15 - E - log4_ceil(S);
    } else {
        e = kstar - 1 - E;
    }
    f[j] = bad[j] ? OZ2_EXP_NONFINITE_DEV : e;
}

// residues of B columns into K-major planes out[t][j][l].  Block = 32 columns
// x CR_ROWS = 128 rows of B: thread (warp w, lane) converts column j0+lane,
// rows l0+16w .. l0+16w+15 (coalesced 256-byte row loads across the warp, 16
// independent loads in flight per thread); its 16 residue bytes per modulus go
// to shared memory as one 16-byte store ([t][col][128 bytes of k], 16-byte
// chunks XOR-swizzled by (col & 7): conflict-free), then every 128-byte plane
// row segment is written by 8 consecutive threads with 16-byte stores (full
// sectors, no partial-sector read-modify-write in L2).
// resident CTAs per SM the register budget allows: the kernel is latency-bound
// on its loads, so occupancy matters (4 CTAs = 64 registers; N > 14 needs 80)
#ifndef OZ2_CR_ROWS
#define OZ2_CR_ROWS 128          // rows of B per column-residue CTA, 16 per thread (A/B round 2: 1.56 -> 1.33 ms vs 64)
#endif
#ifndef OZ2_COLS_MINB
#define OZ2_COLS_MINB 3          // resident CTAs per SM (register cap 85; 16 loads in flight per thread)
#endif
template <int NM, int BW, int CR_ROWS>
__global__ void __launch_bounds__(256, UseImmaCols<BW>::value ? 3 : OZ2_COLS_MINB)
cols_residues_kernel(const double* __restrict__ B, int64_t k, int64_t n, int64_t ldb,
                     const int32_t* __restrict__ f, int8_t* __restrict__ out, int64_t ldr, int64_t pstride) {
    constexpr int WORDS = BwWords<BW>::value;
    constexpr int CR_RPT = CR_ROWS / 8;             // rows per thread (8 warps)
    constexpr int NPC = CR_ROWS / 16;               // 16-byte pieces per (t, col) segment
    extern __shared__ __align__(16) uint8_t sres[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t j0 = (int64_t)blockIdx.x * 32;
    const int64_t l0 = (int64_t)blockIdx.y * CR_ROWS;
    const int64_t j = j0 + lane;
    const uint64_t pol = l2_evict_first();
    {
        // the element loads do not wait for the exponent: they are issued with the
        // load of f[j] (one memory round trip per CTA, not two), and a sentinel
        // column's values are replaced by zeros afterwards
        const int64_t lw = l0 + warp * CR_RPT;
        const double* src = B + lw * ldb + j;
        double a[CR_RPT];
        if (j < n && lw + CR_RPT <= k) {
            #pragma unroll
            for (int q = 0; q < CR_RPT; q++) { a[q] = ld1_hint(src, pol); src += ldb; }
        } else {
            #pragma unroll
            for (int q = 0; q < CR_RPT; q++) a[q] = (j < n && lw + q < k) ? ld1_hint(src + q * ldb, pol) : 0.0;
        }
        const int e = j < n ? __ldg(f + j) : 0;
        const bool live = j < n && e != OZ2_EXP_NONFINITE_DEV;     // sentinel column: x = 0
        double s1, s2;
        pow2_factors(e, s1, s2);
        if (!live) {
            #pragma unroll
            for (int q = 0; q < CR_RPT; q++) a[q] = 0.0;
        }
        // 16-byte chunks XOR-swizzled within the segment (conflict-free stores and loads)
        auto put = [&](int t, const uint32_t (&pw)[CR_RPT / 4]) {
            uint8_t* seg = sres + (size_t)(t * 32 + lane) * CR_ROWS;
            if constexpr (CR_RPT == 16) {
                *reinterpret_cast<uint4*>(seg + ((warp ^ (lane & 7)) * 16)) = make_uint4(pw[0], pw[1], pw[2], pw[3]);
            } else {
                // 8 bytes (rows 8 warp .. 8 warp + 7) at the 8-byte slot warp ^ ((lane >> 1) & 7):
                // the 16 lanes of each parity hit 8 distinct slots, 2 lanes per bank
                // pair (2 wavefronts, the minimum for 256 bytes; the chunk-level XOR
                // of round 1 gave 8-way conflicts)
                const int slot = warp ^ ((lane >> 1) & 7);
                *reinterpret_cast<uint2*>(seg + slot * 8) = make_uint2(pw[0], pw[1]);
            }
        };
        // one multiplication per element when every lane's scale is a normal number
        if (__all_sync(0xffffffffu, s2 == 1.0)) thread_residues<NM, BW, CR_RPT>(a, s1, 1.0, put);
        else thread_residues<NM, BW, CR_RPT>(a, s1, s2, put);
    }
    __syncthreads();
    // write out: NPC threads per (t, col) row segment of CR_ROWS bytes, 16 bytes
    // each; a thread keeps its column and piece and walks t in steps of TSTEP
    constexpr int TSTEP = 256 / NPC / 32;
    const int piece = threadIdx.x % NPC;
    const int col = (threadIdx.x / NPC) & 31;
    const int t0 = (threadIdx.x / NPC) >> 5;
    const int64_t l = l0 + 16 * piece;
    if (l >= ldr || j0 + col >= n) return;                   // ldr % 16 == 0: pieces are whole
    int8_t* gp = out + (int64_t)t0 * pstride + (j0 + col) * ldr + l;
    const int64_t gstep = (int64_t)TSTEP * pstride;
    if constexpr (CR_RPT == 16) {
        const uint8_t* sp = sres + (size_t)(t0 * 32 + col) * CR_ROWS + ((piece ^ (col & (NPC - 1))) * 16);
        #pragma unroll 4
        for (int t = t0; t < NM; t += TSTEP) {
            *reinterpret_cast<uint4*>(gp) = *reinterpret_cast<const uint4*>(sp);
            sp += TSTEP * 32 * CR_ROWS;
            gp += gstep;
        }
    } else {
        // piece = rows 16 piece .. + 15 = the slots of warps 2 piece, 2 piece + 1
        const int sw = (col >> 1) & 7;
        const uint8_t* sp0 = sres + (size_t)(t0 * 32 + col) * CR_ROWS + (((2 * piece) ^ sw) * 8);
        const uint8_t* sp1 = sres + (size_t)(t0 * 32 + col) * CR_ROWS + (((2 * piece + 1) ^ sw) * 8);
        #pragma unroll 4
        for (int t = t0; t < NM; t += TSTEP) {
            const uint2 lo = *reinterpret_cast<const uint2*>(sp0), hi = *reinterpret_cast<const uint2*>(sp1);
            *reinterpret_cast<uint4*>(gp) = make_uint4(lo.x, lo.y, hi.x, hi.y);
            sp0 += TSTEP * 32 * CR_ROWS;
            sp1 += TSTEP * 32 * CR_ROWS;
            gp += gstep;
        }
    }
}

__global__ void trunc_cols_kernel(const double* __restrict__ B, int64_t k, int64_t n, int64_t ldb,
                                  const int32_t* __restrict__ f, double* __restrict__ out) {
    int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;   // over k x n, B order
    if (idx >= k * n) return;
    int64_t l = idx / n, j = idx % n;
    int fj = f[j];
    out[j * k + l] = fj == OZ2_EXP_NONFINITE_DEV ? 0.0 : trunc(scale_pow2(B[l * ldb + j], fj));
}

// ---------------------------------------------------------------------------
// host launchers
// ---------------------------------------------------------------------------
// The residue kernels' integer width for N moduli and a bound |x| < 2^xbits on
// the scaled integers (xbits = T + 1 for FAST, k* for EQ17, 62 / 94 otherwise)
template <int NM>
constexpr int pick_bw(int xbits) {
    return OZ2_RES_IMMA && NM <= 14 && xbits <= 55 ? BW_7 : (NM <= 16 ? BW_8 : BW_12);
}

template <int NM, int BW>
static void launch_rows_bw(const double* A, int64_t m, int64_t k, int64_t lda, int what, int mode,
                           int kstar, int32_t* e, int8_t* res, int64_t ldr, int64_t pstride, cudaStream_t st) {
    // OZ2_ROW_CTAS_PER_SM = R > 0: a persistent grid of R CTAs per SM (rows in
    // flight R * SMs, each 8k bytes, sized against the L2); 0: one CTA per row
    static const int per_sm = [] { const char* v = getenv("OZ2_ROW_CTAS_PER_SM"); return v && *v ? atoi(v) : 0; }();
    int64_t g = m;
    if (per_sm > 0) {
        int dev = 0, sms = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        g = std::min<int64_t>(m, (int64_t)sms * per_sm);
    }
    dim3 grid((unsigned)g), block(OZ2_ROW_THREADS);
    const size_t smem = row_smem_bytes(k);
    auto kern = mode == 0 ? rows_kernel<NM, BW, 0, OZ2_ROW_THREADS> : rows_kernel<NM, BW, 1, OZ2_ROW_THREADS>;
    if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    (kern<<<grid, block, smem, st>>>(A, m, k, lda, what, kstar, e, res, ldr, pstride), count_launch());
}

template <int NM>
static void launch_rows_nm(const double* A, int64_t m, int64_t k, int64_t lda, int what, int mode,
                           int kstar, int32_t* e, int8_t* res, int64_t ldr, int64_t pstride, cudaStream_t st,
                           int xbits) {
    // exponents only: any width (no residues are formed)
    const int bw = (what & 2) ? pick_bw<NM>(xbits) : pick_bw<NM>(64);
    if constexpr (NM <= 14 && OZ2_RES_IMMA) {
        if (bw == BW_7) return launch_rows_bw<NM, BW_7>(A, m, k, lda, what, mode, kstar, e, res, ldr, pstride, st);
    }
    launch_rows_bw<NM, pick_bw<NM>(64)>(A, m, k, lda, what, mode, kstar, e, res, ldr, pstride, st);
}

template <int NM, int BW>
static void launch_cols_res_bw(const double* B, int64_t k, int64_t n, int64_t ldb, const int32_t* f,
                               int8_t* res, int64_t ldr, int64_t pstride, cudaStream_t st) {
    constexpr int ROWS = OZ2_CR_ROWS;
    dim3 grid((unsigned)((n + 31) / 32), (unsigned)((k + ROWS - 1) / ROWS)), block(256);
    const size_t smem = (size_t)NM * 32 * ROWS;
    static bool attr_done[64] = {false};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 64 && !attr_done[dev]) {
        cudaFuncSetAttribute(cols_residues_kernel<NM, BW, ROWS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attr_done[dev] = true;
    }
    (cols_residues_kernel<NM, BW, ROWS><<<grid, block, smem, st>>>(B, k, n, ldb, f, res, ldr, pstride), count_launch());
}

template <int NM>
static void launch_cols_res_nm(const double* B, int64_t k, int64_t n, int64_t ldb, const int32_t* f,
                               int8_t* res, int64_t ldr, int64_t pstride, cudaStream_t st, int xbits) {
    if constexpr (NM <= 14 && OZ2_RES_IMMA) {
        if (pick_bw<NM>(xbits) == BW_7) return launch_cols_res_bw<NM, BW_7>(B, k, n, ldb, f, res, ldr, pstride, st);
    }
    launch_cols_res_bw<NM, pick_bw<NM>(64)>(B, k, n, ldb, f, res, ldr, pstride, st);
}

#define OZ2_DISPATCH_N(N, FN, ...)                                                   \
    switch (N) {                                                                     \
        case 2: FN<2>(__VA_ARGS__); break;   case 3: FN<3>(__VA_ARGS__); break;      \
        case 4: FN<4>(__VA_ARGS__); break;   case 5: FN<5>(__VA_ARGS__); break;      \
        case 6: FN<6>(__VA_ARGS__); break;   case 7: FN<7>(__VA_ARGS__); break;      \
        case 8: FN<8>(__VA_ARGS__); break;   case 9: FN<9>(__VA_ARGS__); break;      \
        case 10: FN<10>(__VA_ARGS__); break; case 11: FN<11>(__VA_ARGS__); break;    \
        case 12: FN<12>(__VA_ARGS__); break; case 13: FN<13>(__VA_ARGS__); break;    \
        case 14: FN<14>(__VA_ARGS__); break; case 15: FN<15>(__VA_ARGS__); break;    \
        case 16: FN<16>(__VA_ARGS__); break; case 17: FN<17>(__VA_ARGS__); break;    \
        case 18: FN<18>(__VA_ARGS__); break; case 19: FN<19>(__VA_ARGS__); break;    \
        case 20: FN<20>(__VA_ARGS__); break; default: break;                         \
    }

void launch_rows(const double* A, int64_t m, int64_t k, int64_t lda, int N, int what, int mode,
                 int kstar, int32_t* e, int8_t* res, int64_t ldr, cudaStream_t st, int64_t pstride, int xbits) {
    if (m == 0) return;
    if (pstride <= 0) pstride = m * ldr;
    OZ2_DISPATCH_N(N, launch_rows_nm, A, m, k, lda, what, mode, kstar, e, res, ldr, pstride, st, xbits);
}

void launch_trunc_rows(const double* A, int64_t m, int64_t k, int64_t lda, const int32_t* e,
                       double* out, cudaStream_t st) {
    int64_t tot = m * k;
    if (!tot) return;
    (trunc_rows_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(A, m, k, lda, e, out), count_launch());
}

size_t cols_stats_bytes(int64_t k, int64_t n) {
    int64_t nch = (k + KC - 1) / KC;
    return (size_t)(nch * n) * (sizeof(int32_t) + sizeof(unsigned long long)) + (size_t)n * sizeof(int32_t) + 256;
}

void launch_cols_exponents(const double* B, int64_t k, int64_t n, int64_t ldb, int N, int mode,
                           int kstar, int32_t* f, void* scratch, cudaStream_t st) {
    if (n == 0) return;
    int64_t nch = (k + KC - 1) / KC;
    if (nch == 0) {                       // k == 0: zero columns
        cudaMemsetAsync(f, 0, sizeof(int32_t) * n, st);
        return;
    }
    unsigned long long* Sc = reinterpret_cast<unsigned long long*>(scratch);
    int32_t* Ec = reinterpret_cast<int32_t*>(Sc + nch * n);
    int32_t* bad = Ec + nch * n;
    cudaMemsetAsync(bad, 0, sizeof(int32_t) * n, st);
    dim3 grid((unsigned)((n + 31) / 32), (unsigned)nch);
    if (mode == 0) (cols_stats_kernel<0><<<grid, 32 * CS_WARPS, 0, st>>>(B, k, n, ldb, Ec, Sc, bad), count_launch());
    else (cols_stats_kernel<1><<<grid, 32 * CS_WARPS, 0, st>>>(B, k, n, ldb, Ec, Sc, bad), count_launch());
    unsigned g2 = (unsigned)((n + 255) / 256);
    if (mode == 0) (cols_finalize_kernel<0><<<g2, 256, 0, st>>>(Ec, Sc, bad, n, (int)nch, host_T(N), kstar, f), count_launch());
    else if (mode == 1) (cols_finalize_kernel<1><<<g2, 256, 0, st>>>(Ec, Sc, bad, n, (int)nch, host_T(N), kstar, f), count_launch());
    else (cols_finalize_kernel<2><<<g2, 256, 0, st>>>(Ec, Sc, bad, n, (int)nch, host_T(N), kstar, f), count_launch());
}

void launch_cols_residues(const double* B, int64_t k, int64_t n, int64_t ldb, const int32_t* f, int N,
                          int8_t* res, int64_t ldr, cudaStream_t st, int64_t pstride, int xbits) {
    if (n == 0 || k == 0) return;
    if (pstride <= 0) pstride = n * ldr;
    OZ2_DISPATCH_N(N, launch_cols_res_nm, B, k, n, ldb, f, res, ldr, pstride, st, xbits);
}

void launch_trunc_cols(const double* B, int64_t k, int64_t n, int64_t ldb, const int32_t* f,
                       double* out, cudaStream_t st) {
    int64_t tot = k * n;
    if (!tot) return;
    (trunc_cols_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(B, k, n, ldb, f, out), count_launch());
}

}  // namespace oz2
