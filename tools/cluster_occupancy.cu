// How many thread-block clusters of size 1/2/4/8 fit at once with the GEMM's
// footprint (384 threads, ~194 KB dynamic smem): GPC granularity decides
// whether a 4-CTA (two CTA pairs, TMA multicast) design can keep all SMs busy.
#include <cstdio>
__global__ void dummy() {}
int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaFuncSetAttribute(dummy, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(dummy, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    for (int cs : {1, 2, 4, 8, 16}) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(cs * 64); cfg.blockDim = dim3(384); cfg.dynamicSmemBytes = 198 * 1024;
        cudaLaunchAttribute a[1]; a[0].id = cudaLaunchAttributeClusterDimension;
        a[0].val.clusterDim.x = cs; a[0].val.clusterDim.y = 1; a[0].val.clusterDim.z = 1;
        cfg.attrs = a; cfg.numAttrs = 1;
        int n = -1; cudaError_t e = cudaOccupancyMaxActiveClusters(&n, dummy, &cfg);
        printf("cluster %2d: max active clusters %3d -> %3d of %d SMs (%s)\n", cs, n, n * cs, sms, cudaGetErrorString(e));
    }
    return 0;
}
