// mb_ops.cu -- per-SM throughput of the instructions on the pass-1 path (sm_100a):
// bf16x2 max (HMNMX2), f32 max (FMNMX), FADD2/FFMA2, FFMA, shuffles, LDS.128, EX2.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb_ops mb_ops.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define N 8
template <int OP>
__global__ void k(uint32_t* out, int iters) {
    __shared__ uint4 sm[1024];
    uint32_t a[N];
    float f[N];
    float2 g[N];
    for (int i = 0; i < N; ++i) { a[i] = threadIdx.x * 77 + i; f[i] = threadIdx.x + i; g[i] = make_float2(f[i], f[i] + 1); }
    if (OP == 5) for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = make_uint4(i, i, i, i);
    __syncthreads();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < N; ++i) {
            if (OP == 0) asm volatile("max.NaN.bf16x2 %0, %0, %1;" : "+r"(a[i]) : "r"(0xF149F149u));
            if (OP == 1) asm volatile("max.NaN.f32 %0, %0, %1;" : "+f"(f[i]) : "f"(-1e30f));
            if (OP == 2) g[i] = __ffma2_rn(g[i], make_float2(1.0001f, 0.9999f), make_float2(0.5f, 0.25f));
            if (OP == 3) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(f[i]) : "f"(1.0001f), "f"(0.5f));
            if (OP == 4) a[i] = __shfl_xor_sync(0xffffffffu, a[i], 1 + (i & 15));
            if (OP == 5) { uint4 v = sm[(threadIdx.x + i * 32 + it) & 1023]; a[i] += v.x ^ v.w; }
            if (OP == 6) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(f[i]));
            if (OP == 7) asm volatile("max.s32 %0, %0, %1;" : "+r"(a[i]) : "r"(7));
            if (OP == 8) asm volatile("{.reg .b32 t; shl.b32 t, %0, 16; and.b32 %0, %0, 0xffff0000; or.b32 %0, %0, t;}" : "+r"(a[i]));
            if (OP == 9) asm volatile("max.f32 %0, %0, %1;" : "+f"(f[i]) : "f"(-1e30f));
        }
    }
    uint32_t s = 0;
    for (int i = 0; i < N; ++i) s += a[i] + __float_as_uint(f[i]) + __float_as_uint(g[i].x) + __float_as_uint(g[i].y);
    if (s == 0x1234567) out[0] = s;
}
template <int OP>
void run(const char* name, int nsm, int clk_khz, uint32_t* out) {
    int iters = 4096;
    k<OP><<<nsm * 4, 256>>>(out, 16);
    cudaDeviceSynchronize();
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    k<OP><<<nsm * 4, 256>>>(out, iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    double ops = (double)nsm * 4 * 256 * iters * N;   // thread-ops
    printf("%-22s %7.1f thread-ops/clk/SM (%5.2f warp-instr/clk/SM)\n", name, ops / (ms * 1e-3) / nsm / (clk_khz * 1e3),
           ops / 32 / (ms * 1e-3) / nsm / (clk_khz * 1e3));
}
int main() {
    int nsm, clk; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    uint32_t* out; cudaMalloc(&out, 64);
    run<0>("max.NaN.bf16x2", nsm, clk, out);
    run<1>("max.NaN.f32", nsm, clk, out);
    run<9>("max.f32", nsm, clk, out);
    run<2>("ffma2 (pairs)", nsm, clk, out);
    run<3>("ffma", nsm, clk, out);
    run<4>("shfl.bfly", nsm, clk, out);
    run<5>("lds.128", nsm, clk, out);
    run<6>("ex2.approx", nsm, clk, out);
    run<7>("max.s32", nsm, clk, out);
    run<8>("shl/and/or (3 ops)", nsm, clk, out);
    return 0;
}
