// Microbenchmark: legacy warp-level int8 MMA (mma.sync m16n8k32 u8.u8 -> IMMA)
// vs dp4a issue throughput on sm_100a.  Design input for the residue kernels'
// byte dot products.
#include <cstdio>
#include <cstdint>
__global__ void kmma(uint32_t* out, int iters) {
  uint32_t a0=threadIdx.x, a1=a0*3, a2=a0*5, a3=a0*7, b1=0x05060708;
  int c[8][4] = {};
  for (int i = 0; i < iters; i++) {
    #pragma unroll
    for (int j = 0; j < 8; j++)
    asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+r"(c[j][0]),"+r"(c[j][1]),"+r"(c[j][2]),"+r"(c[j][3]) : "r"(a0),"r"(a1),"r"(a2),"r"(a3),"r"(0x01020304u+j),"r"(b1));
  }
  int s=0; for(int j=0;j<8;j++) s+=c[j][0]+c[j][1]+c[j][2]+c[j][3];
  out[blockIdx.x*blockDim.x+threadIdx.x]=s;
}
__global__ void kdp4a(uint32_t* out, int iters) {
  uint32_t a = threadIdx.x * 0x01010101u;
  uint32_t c[16] = {};
  for (int i = 0; i < iters; i++) {
    #pragma unroll
    for (int j = 0; j < 16; j++) c[j] = __dp4a(a + j, 0x01020304u, c[j]);
  }
  uint32_t s=0; for(int j=0;j<16;j++) s+=c[j];
  out[blockIdx.x*blockDim.x+threadIdx.x]=s;
}
int main(){ uint32_t* o; cudaMalloc(&o, 148*8*1024*4);
 cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
 int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
 for (int w=1; w<=32; w*=2) {
   int iters=2048; kmma<<<148, 32*w>>>(o, 16); cudaDeviceSynchronize();
   cudaEventRecord(e0); kmma<<<148*2, 32*w>>>(o, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
   float ms; cudaEventElapsedTime(&ms,e0,e1);
   double n = 148.0*2*w*iters*8;
   printf("mma.sync u8 warps/cta %2d: %.3f ms, %.3f IMMA/clk/SM (at %d MHz), %.1f TOPS\n", w, ms, n/(ms*1e-3)/148/(clk*1e3), clk/1000, n*16*8*32*2/(ms*1e-3)/1e12);
 }
 for (int w=1; w<=32; w*=2) {
   int iters=4096; kdp4a<<<148, 32*w>>>(o, 16); cudaDeviceSynchronize();
   cudaEventRecord(e0); kdp4a<<<148*2, 32*w>>>(o, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
   float ms; cudaEventElapsedTime(&ms,e0,e1);
   double n = 148.0*2*w*iters*16;
   printf("dp4a warps/cta %2d: %.3f ms, %.3f warp-dp4a/clk/SM\n", w, ms, n/(ms*1e-3)/148/(clk*1e3));
 }
 return 0; }
