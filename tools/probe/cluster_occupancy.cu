// How many thread-block clusters of 2 / 4 / 8 / 16 CTAs (one ~227 KB CTA per SM, as
// the b2b / du kernels) a B200 runs at once: cudaOccupancyMaxActiveClusters.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k() {}
int main() {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    for (int cs : {1, 2, 4, 6, 8, 12, 16}) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(cs * 64);
        cfg.blockDim = dim3(384);
        cfg.dynamicSmemBytes = 220 * 1024;
        cudaLaunchAttribute a[1];
        a[0].id = cudaLaunchAttributeClusterDimension;
        a[0].val.clusterDim.x = cs;
        a[0].val.clusterDim.y = 1;
        a[0].val.clusterDim.z = 1;
        cfg.attrs = a;
        cfg.numAttrs = 1;
        int n = 0;
        cudaError_t e = cudaOccupancyMaxActiveClusters(&n, k, &cfg);
        printf("cluster %2d CTAs: %3d clusters = %3d CTAs (%s)\n", cs, n, n * cs, cudaGetErrorString(e));
    }
    return 0;
}
