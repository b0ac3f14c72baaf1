// liboz2.cu -- the library is compiled as one translation unit so that the
// __constant__ tables are shared by every kernel without relocatable device code.
#include "oz2_device.cuh"
#include "scale.cu"
#include "crt.cu"
#include "accu.cu"
#include "kslice.cu"
#include "gemm.cu"
#include "api.cu"
