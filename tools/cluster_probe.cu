// How many clusters of each size can be co-resident with one 768-thread, ~200 KB CTA per SM.
// nvcc -gencode arch=compute_100a,code=sm_100a -o tools/cluster_probe tools/cluster_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k(int* out) {
    extern __shared__ int s[];
    if (threadIdx.x == 0 && out) { s[0] = 1; out[blockIdx.x] = s[0]; }
}

int main() {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    printf("SMs %d\n", nsm);
    for (int cs = 1; cs <= 16; ++cs) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(cs * 16);
        cfg.blockDim = dim3(768);
        cfg.dynamicSmemBytes = 200 * 1024;
        cudaLaunchAttribute a[1];
        a[0].id = cudaLaunchAttributeClusterDimension;
        a[0].val.clusterDim.x = cs;
        a[0].val.clusterDim.y = 1;
        a[0].val.clusterDim.z = 1;
        cfg.attrs = a;
        cfg.numAttrs = 1;
        int n = -1;
        cudaError_t e = cudaOccupancyMaxActiveClusters(&n, k, &cfg);
        printf("cluster %2d: max active clusters %3d -> %3d CTAs (%s)\n", cs, n, n * cs, cudaGetErrorString(e));
    }
    return 0;
}
