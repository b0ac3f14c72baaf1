// liboz2_gemm.cu -- translation unit 2 of liboz2.so: the persistent tcgen05
// GEMM with the fused CRT epilogue (gemm.cu).
#include "gemm.cu"
