// oz2_tables.h -- per-N constants of Algorithm 1 as the kernels consume them.
//
// Built on the host by tables.cpp (independent of oracle/) and copied to
// __constant__ memory once per device.  Indexed by N (2..20).
#pragma once
#include <stdint.h>

#define OZ2_MAX_MODULI 20
#define OZ2_MAX_BYTES 20    // bytes of M (and of every w_t < M): M < 2^156 for N <= 20
#define OZ2_MAX_GROUPS 5    // groups of 4 moduli (one dp4a per group and byte)
#define OZ2_MAX_WORDS 5     // 32-bit words of X in [-3M/2, 3M/2), two's complement

struct Oz2Table {
    int32_t N;           // number of moduli
    int32_t JB;          // bytes of M (1..20)
    int32_t WS;          // 32-bit words of S = sum_t c''_t w_t < 2^13 M (1..6)
    int32_t WX;          // 32-bit words that hold X in [-3M/2, 3M/2) (1..5)
    int32_t L;           // floor(log2(M/2 - 1))        (Eq. 16 with q dropped)
    int32_t T;           // floor(L/2): FAST bound ||2^e a||_2 <= 2^T   (reading R4)
    int32_t m[OZ2_MAX_MODULI];        // moduli, Eq. (18) + reading R1
    uint32_t magic[OZ2_MAX_MODULI];   // ceil(2^32 / m): floor(y/m) = umulhi(y, magic) for y < 2^24
    int32_t h[OZ2_MAX_MODULI];        // (m - 1) / 2 (odd m): symmetric offset
    uint32_t negm[OZ2_MAX_MODULI];    // 2^32 - m: y - q m as one multiply-add
    uint32_t cw[3][OZ2_MAX_MODULI];   // byte b of cw[w][t] = 2^(8(4w+b)) mod m_t
    uint32_t k16[OZ2_MAX_MODULI];     // 2^16 mod m_t
    int32_t k16s[OZ2_MAX_MODULI];     // 2^16 mod m_t, symmetric representative (|k16s| <= m_t / 2)
    uint32_t off7[OZ2_MAX_MODULI];    // m_t * ceil(2^22 / m_t): keeps the line-7 value non-negative
    uint32_t g32[OZ2_MAX_MODULI];     // (-2^32) mod m_t in [0, m_t)
    int32_t g64[OZ2_MAX_MODULI];      // (-2^64) mod m_t in [0, m_t)
    int32_t g96[OZ2_MAX_MODULI];      // (-2^96) mod m_t in [0, m_t)
    uint32_t G63[OZ2_MAX_MODULI];     // (-2^63) mod m_t: undoes the 2^63 bias of 64-bit residue inputs
    uint32_t G95[OZ2_MAX_MODULI];     // (-2^95) mod m_t: same for 96-bit inputs
    uint64_t hmagic[OZ2_MAX_MODULI];  // h_t * magic_t: floor((y + h)/m) = (y * magic + hmagic) >> 32
    // w_t = M y_t / m_t (Alg. 1 line 8) as bytes, packed for dp4a: byte i of
    // Wb[j][g] is byte j of w_(4g+i) (0 beyond N), so that
    // sum_t c''_t byte_j(w_t) = sum_g dp4a(c''_(4g..4g+3), Wb[j][g])
    uint32_t Wb[OZ2_MAX_BYTES][OZ2_MAX_GROUPS];
    uint32_t w32[OZ2_MAX_MODULI][OZ2_MAX_WORDS];  // w_t as 32-bit words (host export / tests)
    uint32_t M32[OZ2_MAX_WORDS];      // M, 32-bit words, little endian
    uint32_t Mh32[OZ2_MAX_WORDS];     // M / 2, same
    float qscale;                     // 2^(32 (WS - 2)) / M (WS >= 2), 1 / M (WS = 1)
    int32_t y[OZ2_MAX_MODULI];        // least positive inverse of M_t mod m_t (host only)
    // residue kernels, q = rint(y / m_t) on the FP32 pipe: the dp4a addend
    // 0x4B000000 + G makes y's bits the binary32 2^23 + y (y < 2^20)
    uint32_t G63f[OZ2_MAX_MODULI];    // 0x4B000000 + G63
    uint32_t G95f[OZ2_MAX_MODULI];    // 0x4B000000 + G95
    float invm[OZ2_MAX_MODULI];       // RN_binary32(1 / m_t)
    // GEMM drain (line 7) on the FP32 pipe: c' = hi 2^18 + lo
    int32_t k18s[OZ2_MAX_MODULI];     // 2^18 mod m_t, |k18s| <= m_t / 2
    uint32_t k18k[OZ2_MAX_MODULI];    // -8 k18s mod 2^32 (cancels the 2^21 offset of the lo bits)
    float h23f[OZ2_MAX_MODULI];       // 2^23 + (m_t - 1) / 2 (odd m_t; exact in binary32)
};

// Fill tabs[2..20]; tabs[0], tabs[1] are zeroed.  Returns 0 on success.
int oz2_build_tables(Oz2Table tabs[OZ2_MAX_MODULI + 1]);
// Eq. (17): max{kappa : q 4^kappa <= M/2 - 1} or -1.
int oz2_host_eq17_k(int N, int64_t q);
