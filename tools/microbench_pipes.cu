// Throughput of the ALU pipes the CRT epilogue could use (DFMA, IMAD.WIDE.U32,
// IMAD, FFMA, I2F.F64) on this GPU: 148 x 4 CTAs of 256 threads, 8 independent
// chains per thread, CUDA-event timed.  Design input for the CRT.
#include <cstdio>
#include <cstdint>
#define ITERS 4096
__global__ void k_dfma(double* out, double s) {
    double a[8]; for (int i = 0; i < 8; i++) a[i] = threadIdx.x + i;
    for (int it = 0; it < ITERS; it++)
        #pragma unroll
        for (int i = 0; i < 8; i++) a[i] = fma(a[i], s, 1.0);
    double r = 0; for (int i = 0; i < 8; i++) r += a[i];
    if (r == 12345.0) out[0] = r;
}
__global__ void k_imadwide(uint64_t* out, uint32_t s) {
    uint64_t a[8]; for (int i = 0; i < 8; i++) a[i] = threadIdx.x + i;
    for (int it = 0; it < ITERS; it++)
        #pragma unroll
        for (int i = 0; i < 8; i++) a[i] = (uint64_t)(uint32_t)(a[i] >> 7) * s + a[i];
    uint64_t r = 0; for (int i = 0; i < 8; i++) r += a[i];
    if (r == 12345) out[0] = r;
}
__global__ void k_imad(uint32_t* out, uint32_t s) {
    uint32_t a[8]; for (int i = 0; i < 8; i++) a[i] = threadIdx.x + i;
    for (int it = 0; it < ITERS; it++)
        #pragma unroll
        for (int i = 0; i < 8; i++) a[i] = a[i] * s + 0x9e3779b9u;
    uint32_t r = 0; for (int i = 0; i < 8; i++) r += a[i];
    if (r == 12345) out[0] = r;
}
__global__ void k_ffma(float* out, float s) {
    float a[8]; for (int i = 0; i < 8; i++) a[i] = threadIdx.x + i;
    for (int it = 0; it < ITERS; it++)
        #pragma unroll
        for (int i = 0; i < 8; i++) a[i] = fmaf(a[i], s, 1.0f);
    float r = 0; for (int i = 0; i < 8; i++) r += a[i];
    if (r == 12345.f) out[0] = r;
}
__global__ void k_i2f64(double* out, uint64_t s) {
    uint64_t a[8]; double acc = 0; for (int i = 0; i < 8; i++) a[i] = threadIdx.x * s + i;
    for (int it = 0; it < ITERS; it++)
        #pragma unroll
        for (int i = 0; i < 8; i++) { double d = __ull2double_rn(a[i]); a[i] ^= (uint64_t)__double_as_longlong(d); }
    for (int i = 0; i < 8; i++) acc += (double)a[i];
    if (acc == 12345.0) out[0] = acc;
}
template <typename F, typename... A>
void run(const char* name, F f, A... args) {
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    dim3 g(sms * 4), b(256);
    f<<<g, b>>>(args...); cudaDeviceSynchronize();
    cudaEventRecord(e0); f<<<g, b>>>(args...); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double ops = (double)g.x * b.x * ITERS * 8;
    printf("%-10s %8.3f ms  %8.2f Gop/s  %6.1f lane-ops/clk/SM @1.9GHz\n", name, ms, ops / ms / 1e6,
           ops / (ms * 1e-3) / sms / 1.9e9);
}
int main() {
    void* buf; cudaMalloc(&buf, 64);
    run("DFMA", k_dfma, (double*)buf, 1.0000001);
    run("IMAD.WIDE", k_imadwide, (uint64_t*)buf, 12345u);
    run("IMAD", k_imad, (uint32_t*)buf, 12345u);
    run("FFMA", k_ffma, (float*)buf, 1.0000001f);
    run("I2F.F64", k_i2f64, (double*)buf, (uint64_t)0x12345);
    return 0;
}
