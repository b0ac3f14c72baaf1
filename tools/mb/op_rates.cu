// Microbenchmark: reciprocal throughput (cycles per warp-instruction per SMSP)
// of single SASS instruction forms on sm_100a: 8 independent loop-carried
// chains per thread, 32 warps per SM.  Each probe is one instruction per
// chain step (checked in the SASS with cuobjdump).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/opr tools/mb/op_rates.cu && /tmp/opr
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t dp4a_r(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t d; asm volatile("dp4a.u32.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c)); return d;
}
__device__ __forceinline__ uint32_t dp4a_i(uint32_t a, uint32_t c) {
    uint32_t d; asm volatile("dp4a.u32.u32 %0, %1, 0x01020304, %2;" : "=r"(d) : "r"(a), "r"(c)); return d;
}
__device__ __forceinline__ uint32_t mulhi_i(uint32_t a) {
    uint32_t d; asm volatile("mul.hi.u32 %0, %1, 0x9e3779b9;" : "=r"(d) : "r"(a)); return d;
}
__device__ __forceinline__ uint32_t madhi_i(uint32_t a, uint32_t c) {
    uint32_t d; asm volatile("mad.hi.u32 %0, %1, 0x9e3779b9, %2;" : "=r"(d) : "r"(a), "r"(c)); return d;
}
__device__ __forceinline__ uint32_t mad_i(uint32_t a, uint32_t c) {
    uint32_t d; asm volatile("mad.lo.u32 %0, %1, 0x9e3779b9, %2;" : "=r"(d) : "r"(a), "r"(c)); return d;
}
__device__ __forceinline__ uint32_t mad_r(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t d; asm volatile("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c)); return d;
}
__device__ __forceinline__ uint64_t madwide_i(uint32_t a, uint64_t c) {
    uint64_t d; asm volatile("mad.wide.u32 %0, %1, 0x9e3779b9, %2;" : "=l"(d) : "r"(a), "l"(c)); return d;
}
__device__ __forceinline__ float ffma_i(float a, float c) {
    float d; asm volatile("fma.rn.f32 %0, %1, 0f3F7FBE77, %2;" : "=f"(d) : "f"(a), "f"(c)); return d;
}
__device__ __forceinline__ float ffma_r(float a, float b, float c) {
    float d; asm volatile("fma.rn.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c)); return d;
}
__device__ __forceinline__ float fadd_i(float a) {
    float d; asm volatile("add.rn.f32 %0, %1, 0f4B400000;" : "=f"(d) : "f"(a)); return d;
}
__device__ __forceinline__ double dfma_i(double a, double c) {
    double d; asm volatile("fma.rn.f64 %0, %1, 0d3FEFFFFFFFFFFFFF, %2;" : "=d"(d) : "d"(a), "d"(c)); return d;
}
__device__ __forceinline__ uint32_t lea_i(uint32_t a, uint32_t b) {
    uint32_t d; asm volatile("{.reg .u32 t; shl.b32 t, %1, 3; add.u32 %0, t, %2;}" : "=r"(d) : "r"(a), "r"(b)); return d;
}
__device__ __forceinline__ uint32_t iadd3(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t d; asm volatile("{.reg .u32 t; add.u32 t, %1, %2; add.u32 %0, t, %3;}" : "=r"(d) : "r"(a), "r"(b), "r"(c)); return d;
}
__device__ __forceinline__ uint32_t prmt_r(uint32_t a, uint32_t b) {
    uint32_t d; asm volatile("prmt.b32 %0, %1, %2, 0x5140;" : "=r"(d) : "r"(a), "r"(b)); return d;
}
__device__ __forceinline__ uint32_t lop3(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t d; asm volatile("lop3.b32 %0, %1, %2, %3, 0x96;" : "=r"(d) : "r"(a), "r"(b), "r"(c)); return d;
}
__device__ __forceinline__ float i2f_trick(uint32_t a) {   // LOP3 + FADD
    return __uint_as_float(a | 0x4B000000u) - 8388608.0f;
}

template <int OP>
__global__ void __launch_bounds__(256, 4) kop(uint32_t* out, int iters, uint32_t s) {
    uint32_t u[8]; float f[8]; double d[8]; uint64_t w[8];
    #pragma unroll
    for (int j = 0; j < 8; j++) { u[j] = threadIdx.x * 7 + j + s; f[j] = (float)u[j]; d[j] = u[j]; w[j] = u[j]; }
    for (int it = 0; it < iters; it++) {
        #pragma unroll
        for (int j = 0; j < 8; j++) {
            if (OP == 0) u[j] = dp4a_r(u[j], s, u[j]);
            if (OP == 1) u[j] = dp4a_i(u[j], u[j]);
            if (OP == 2) u[j] = madhi_i(u[j], u[j]);
            if (OP == 3) u[j] = mad_i(u[j], u[j]);
            if (OP == 4) u[j] = mad_r(u[j], s, u[j]);
            if (OP == 5) w[j] = madwide_i((uint32_t)w[j], w[j]);
            if (OP == 6) f[j] = ffma_i(f[j], f[j]);
            if (OP == 7) f[j] = ffma_r(f[j], __uint_as_float(s), f[j]);
            if (OP == 8) f[j] = fadd_i(f[j]);
            if (OP == 9) d[j] = dfma_i(d[j], d[j]);
            if (OP == 10) u[j] = lea_i(u[j], u[j]);
            if (OP == 11) u[j] = iadd3(u[j], s, u[j]);
            if (OP == 12) u[j] = prmt_r(u[j], u[(j + 1) & 7]);
            if (OP == 13) u[j] = lop3(u[j], s, u[(j + 3) & 7]);
            if (OP == 14) u[j] = mulhi_i(u[j]);
        }
    }
    uint32_t acc = 0;
    #pragma unroll
    for (int j = 0; j < 8; j++) acc ^= u[j] ^ __float_as_uint(f[j]) ^ (uint32_t)__double2loint(d[j]) ^ (uint32_t)w[j];
    out[blockIdx.x * 256 + threadIdx.x] = acc;
}

int main() {
    int sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const int blocks = sms * 4 * 4;
    uint32_t* out;
    cudaMalloc(&out, blocks * 256 * 4);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    auto timeit = [&](auto kern, const char* name) {
        const int iters = 4096;
        kern<<<blocks, 256>>>(out, 16, 3u);
        cudaDeviceSynchronize();
        float best = 1e30f;
        for (int r = 0; r < 5; r++) {
            cudaEventRecord(e0);
            kern<<<blocks, 256>>>(out, iters, 3u);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            best = ms < best ? ms : best;
        }
        const double n = (double)blocks * 256 * iters * 8;
        const double cyc = best * 1e-3 * clk * 1e3 * sms * 4 / (n / 32);
        printf("%-28s %6.2f cyc per warp-instr per SMSP (max clock %d MHz assumed)\n", name, cyc, clk / 1000);
    };
    timeit(kop<0>, "IDP reg");
    timeit(kop<1>, "IDP imm");
    timeit(kop<2>, "IMAD.HI imm + addend");
    timeit(kop<14>, "IMAD.HI imm (mul.hi)");
    timeit(kop<3>, "IMAD imm");
    timeit(kop<4>, "IMAD reg");
    timeit(kop<5>, "IMAD.WIDE imm");
    timeit(kop<6>, "FFMA imm");
    timeit(kop<7>, "FFMA reg");
    timeit(kop<8>, "FADD imm");
    timeit(kop<9>, "DFMA imm");
    timeit(kop<10>, "LEA (shl+add)");
    timeit(kop<11>, "IADD3");
    timeit(kop<12>, "PRMT");
    timeit(kop<13>, "LOP3");
    return 0;
}
