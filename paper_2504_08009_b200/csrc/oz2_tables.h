// oz2_tables.h -- per-N constants of Algorithm 1 as the kernels consume them.
//
// Built on the host by tables.cpp (independent of oracle/) and copied to
// __constant__ memory once per device.  Indexed by N (2..20).
#pragma once
#include <stdint.h>

#define OZ2_MAX_MODULI 20
#define OZ2_PIECE_BITS 38   // CRT weights and M are split into 38-bit FP64 pieces
#define OZ2_MAX_PIECES 5

struct Oz2Table {
    int32_t N;           // number of moduli
    int32_t P;           // number of 38-bit pieces of M (1..5)
    int32_t L;           // floor(log2(M/2 - 1))        (Eq. 16 with q dropped)
    int32_t T;           // floor(L/2): FAST bound ||2^e a||_2 <= 2^T   (reading R4)
    int32_t m[OZ2_MAX_MODULI];        // moduli, Eq. (18) + reading R1
    uint32_t magic[OZ2_MAX_MODULI];   // ceil(2^32 / m): floor(y/m) = umulhi(y, magic) for y < 2^24
    int32_t h[OZ2_MAX_MODULI];        // (m - 1) / 2 (odd m): symmetric offset
    uint32_t cw[3][OZ2_MAX_MODULI];   // byte b of cw[w][t] = 2^(8(4w+b)) mod m_t
    uint32_t k16[OZ2_MAX_MODULI];     // 2^16 mod m_t
    uint32_t g32[OZ2_MAX_MODULI];     // (-2^32) mod m_t in [0, m_t)
    int32_t g64[OZ2_MAX_MODULI];      // (-2^64) mod m_t in [0, m_t)
    int32_t g96[OZ2_MAX_MODULI];      // (-2^96) mod m_t in [0, m_t)
    uint32_t G63[OZ2_MAX_MODULI];     // (-2^63) mod m_t: undoes the 2^63 bias of 64-bit residue inputs
    uint32_t G95[OZ2_MAX_MODULI];     // (-2^95) mod m_t: same for 96-bit inputs
    uint64_t hmagic[OZ2_MAX_MODULI];  // h_t * magic_t: floor((y + h)/m) = (y * magic + hmagic) >> 32
    double W[OZ2_MAX_PIECES][OZ2_MAX_MODULI];  // w_t = M y_t / m_t = sum_p W[p][t] 2^(38p), W < 2^38
    double Mp[OZ2_MAX_PIECES];        // M = sum_p Mp[p] 2^(38p)
    double invM;                      // 2^(38(P-2)) / M  (P >= 2),  1/M  (P == 1)
    uint64_t bias[3];                 // (0x4338000000000000 * sum_p 2^(38p)) mod 2^192 (piece-extraction bias)
    double inv_m[OZ2_MAX_MODULI];     // 1.0 / m_t
    uint64_t Mw[3];                   // M, 192-bit little endian
    uint64_t Mhalf[3];                // M / 2
    int32_t y[OZ2_MAX_MODULI];        // least positive inverse of M_t mod m_t (host only)
};

// Fill tabs[2..20]; tabs[0], tabs[1] are zeroed.  Returns 0 on success.
int oz2_build_tables(Oz2Table tabs[OZ2_MAX_MODULI + 1]);
// Eq. (17): max{kappa : q 4^kappa <= M/2 - 1} or -1.
int oz2_host_eq17_k(int N, int64_t q);
