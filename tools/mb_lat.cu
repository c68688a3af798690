// mb_lat.cu -- dependent-chain latencies (SM cycles) of the pass-1 instructions on sm_100a.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
template <int OP>
__global__ void k(uint32_t* out, long long* cyc, int iters) {
    __shared__ uint32_t sm[1024];
    __shared__ uint64_t bar;
    __shared__ uint32_t taddr;
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = (i + 1) & 1023;
    if (OP == 7 && threadIdx.x == 0) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar))); }
    if (OP == 8) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(sa(&taddr)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    uint32_t a = threadIdx.x;
    float f = 0.5f + threadIdx.x * 1e-3f;
    float2 g = make_float2(f, f);
    uint32_t ph = 0;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        if (OP == 0) a = __shfl_xor_sync(0xffffffffu, a, 1);
        if (OP == 1) a = sm[a];
        if (OP == 2) asm volatile("max.NaN.bf16x2 %0, %0, %1;" : "+r"(a) : "r"(0xF149F149u));
        if (OP == 3) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(f));
        if (OP == 4) g = __ffma2_rn(g, make_float2(1.0001f, 0.9999f), make_float2(-0.5f, 0.25f));
        if (OP == 5) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(f) : "f"(1.0001f), "f"(0.5f));
        if (OP == 6) { a = __shfl_xor_sync(0xffffffffu, a, 16); a = __shfl_xor_sync(0xffffffffu, a, 8);
                       a = __shfl_xor_sync(0xffffffffu, a, 4); a = __shfl_xor_sync(0xffffffffu, a, 2);
                       a = __shfl_xor_sync(0xffffffffu, a, 1); }
        if (OP == 7) {
            if (threadIdx.x == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(&bar)) : "memory");
            uint32_t done = 0;
            while (!done)
                asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }"
                             : "=r"(done) : "r"(sa(&bar)), "r"(ph) : "memory");
            ph ^= 1;
        }
        if (OP == 8) {
            asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(taddr), "r"(a) : "memory");
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(a) : "r"(taddr) : "memory");
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        }
        if (OP == 9) { asm volatile("bar.warp.sync 0xffffffff;" ::: "memory"); a += 1; }
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[OP] = (t1 - t0) / iters;
    if (a == 0x1234567 || f == 1234.5f || g.x == 1234.f) out[0] = a;
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (OP == 8) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(taddr));
}
int main() {
    uint32_t* out; long long* cyc; cudaMalloc(&out, 64); cudaMalloc(&cyc, 16 * 8); cudaMemset(cyc, 0, 128);
    k<0><<<1, 32>>>(out, cyc, 1000); k<1><<<1, 32>>>(out, cyc, 1000); k<2><<<1, 32>>>(out, cyc, 1000);
    k<3><<<1, 32>>>(out, cyc, 1000); k<4><<<1, 32>>>(out, cyc, 1000); k<5><<<1, 32>>>(out, cyc, 1000);
    k<6><<<1, 32>>>(out, cyc, 1000); k<7><<<1, 32>>>(out, cyc, 1000); k<8><<<1, 32>>>(out, cyc, 1000);
    k<9><<<1, 32>>>(out, cyc, 1000);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[16]; cudaMemcpy(h, cyc, 128, cudaMemcpyDeviceToHost);
    const char* n[] = {"shfl", "lds.u32 (pointer chase)", "max.bf16x2", "ex2", "ffma2", "ffma", "5x shfl (warp reduce)",
                       "mbarrier arrive+try_wait", "tmem st+wait+ld+wait", "syncwarp+iadd"};
    for (int i = 0; i < 10; ++i) printf("%-28s %lld cycles\n", n[i], h[i]);
    printf("%s\n", cudaGetErrorString(e));
}
