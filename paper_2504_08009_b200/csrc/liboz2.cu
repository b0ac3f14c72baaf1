// liboz2.cu -- translation unit 1 of liboz2.so: conversion, CRT, accu, K-split,
// certificate kernels and the C ABI.  The persistent GEMM is translation unit 2
// (liboz2_gemm.cu).  Each unit has its own copy of the __constant__ tables;
// api.cu uploads both.
#include "oz2_device.cuh"
#include "scale.cu"
#include "crt.cu"
#include "accu.cu"
#include "kslice.cu"
#include "certify.cu"
#include "fp64mod.cu"
#include "api.cu"
