// FP64 vs FP32 FMA throughput per SM (sm_100a).  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mb_fp64 tools/mb_fp64.cu
#include <cstdio>
#include <cuda_runtime.h>
template <typename Tp>
__global__ void k(Tp* out, int iters) {
    Tp a[8];
    for (int i = 0; i < 8; ++i) a[i] = (Tp)(threadIdx.x + i) * (Tp)1e-3;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = a[i] * (Tp)1.0000001 + (Tp)1e-7;
    }
    Tp s = 0;
    for (int i = 0; i < 8; ++i) s += a[i];
    if (s == (Tp)12345.678) out[0] = s;
}
int main() {
    int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    double* od; float* of; cudaMalloc(&od, 8); cudaMalloc(&of, 8);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int iters = 4096;
    for (int rep = 0; rep < 2; ++rep) {
        k<double><<<nsm * 4, 256>>>(od, 16); cudaDeviceSynchronize();
        cudaEventRecord(e0); k<double><<<nsm * 4, 256>>>(od, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
        float msd; cudaEventElapsedTime(&msd, e0, e1);
        cudaEventRecord(e0); k<float><<<nsm * 4, 256>>>(of, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
        float msf; cudaEventElapsedTime(&msf, e0, e1);
        double ops = (double)nsm * 4 * 256 * iters * 8;
        printf("FP64 FMA: %.1f lanes/clk/SM (%.2f TFLOP/s) | FP32 FMA: %.1f lanes/clk/SM (%.2f TFLOP/s)\n",
               ops / (msd * 1e-3) / nsm / (clk * 1e3), 2 * ops / (msd * 1e-3) / 1e12,
               ops / (msf * 1e-3) / nsm / (clk * 1e3), 2 * ops / (msf * 1e-3) / 1e12);
    }
    return 0;
}
