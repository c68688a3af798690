// Streaming-read ceiling of TMA bulk copies on B200 for the grid shapes a cluster-based core
// can use: 1 CTA per SM without clusters, and clusters of 2/4/8/16 CTAs (only as many CTAs as
// can be co-resident).  Optional per-element work: mode 1 = one MUFU ex2 + fp32 add per bf16
// element (the pass-1 exponential), mode 2 = mode 1 + 3 more packed fp32 ops per element pair.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mb_cluster_bw tools/mb_cluster_bw.cu
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); return 1; } } while (0)

constexpr int NCONS = 8;             // consumer warps
constexpr int THREADS = 32 * (1 + NCONS);

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mb_init(uint64_t* b, uint32_t n) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n)); }
__device__ __forceinline__ bool mb_try(uint64_t* b, uint32_t ph) {
    uint32_t d;
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3; selp.u32 %0, 1, 0, p; }"
                 : "=r"(d) : "r"(su32(b)), "r"(ph), "r"(1000000u) : "memory");
    return d != 0;
}
__device__ __forceinline__ bool mb_try_spin(uint64_t* b, uint32_t ph) {
    uint32_t d;
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(d) : "r"(su32(b)), "r"(ph) : "memory");
    return d != 0;
}
template <bool SPIN> __device__ __forceinline__ void mb_wait(uint64_t* b, uint32_t ph) { if (SPIN) { while (!mb_try_spin(b, ph)) {} } else { while (!mb_try(b, ph)) {} } }
__device__ __forceinline__ void mb_arrive(uint64_t* b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory"); }
__device__ __forceinline__ void mb_expect(uint64_t* b, uint32_t n) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(n) : "memory"); }

template <int CHUNK, bool SPIN>
__global__ void __launch_bounds__(THREADS, 1) stream_kernel(const char* src, size_t nchunks, int stages, int mode, float* out) {
    extern __shared__ __align__(128) unsigned char sm[];
    uint64_t* full = reinterpret_cast<uint64_t*>(sm);
    uint64_t* empty = full + 64;
    unsigned char* ring = sm + 1024;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s) { mb_init(&full[s], 1); mb_init(&empty[s], NCONS); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const size_t nct = gridDim.x;
    const size_t my = nchunks / nct + ((size_t)blockIdx.x < nchunks % nct ? 1 : 0);
    if (warp == 0) {
        if (lane == 0) {
            uint64_t pol;
            asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
            for (size_t k = 0; k < my; ++k) {
                const int st = (int)(k % stages);
                const uint32_t ph = (uint32_t)((k / stages) & 1);
                if (k >= (size_t)stages) mb_wait<SPIN>(&empty[st], ph ^ 1);
                mb_expect(&full[st], CHUNK);
                const char* g = src + (blockIdx.x + k * nct) * (size_t)CHUNK;
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
                             ::"r"(su32(ring + (size_t)st * CHUNK)), "l"(g), "r"(CHUNK), "r"(su32(&full[st])), "l"(pol) : "memory");
            }
        }
    } else {
        const int t = threadIdx.x - 32;
        float acc = 0.f;
        uint32_t x = 0;
        for (size_t k = 0; k < my; ++k) {
            const int st = (int)(k % stages);
            mb_wait<SPIN>(&full[st], (uint32_t)((k / stages) & 1));
            const uint4* p = reinterpret_cast<const uint4*>(ring + (size_t)st * CHUNK);
            const uint4 a = p[t], b = p[(t + 256) % (CHUNK / 16)];
            if (mode == 0) {
                x ^= a.x ^ a.y ^ a.z ^ a.w ^ b.x ^ b.y ^ b.z ^ b.w;
            } else {
                const uint32_t w[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
                float2 s2 = make_float2(0.f, 0.f);
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    float lo = __uint_as_float(w[i] << 16), hi = __uint_as_float(w[i] & 0xffff0000u);
                    float2 y = __fmul2_rn(make_float2(lo, hi), make_float2(1.4426950408889634f, 1.4426950408889634f));
                    float e0, e1;
                    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e0) : "f"(y.x));
                    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e1) : "f"(y.y));
                    if (mode == 2) {
                        float2 q = __ffma2_rn(make_float2(e0, e1), y, s2);
                        s2 = __fadd2_rn(q, make_float2(e1, e0));
                    }
                    s2 = __fadd2_rn(s2, make_float2(e0, e1));
                }
                acc += s2.x + s2.y;
            }
            __syncwarp();
            if (lane == 0) mb_arrive(&empty[st]);
        }
        if (acc == 1.2345f || x == 0x12345u) out[threadIdx.x] = acc + (float)x;
    }
}


template <int CHUNK, bool SPIN>
static int run(const char* src, size_t bytes, float* out, int nsm, int mode, int cs, int inflight) {
    const int stages = inflight / CHUNK;
    const size_t nchunks = bytes / CHUNK;
    const size_t smem = 1024 + (size_t)stages * CHUNK;
    auto k = stream_kernel<CHUNK, SPIN>;
    CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    CK(cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    cudaLaunchConfig_t cfg = {};
    cfg.blockDim = dim3(THREADS);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute a[1];
    a[0].id = cudaLaunchAttributeClusterDimension;
    a[0].val.clusterDim.x = cs; a[0].val.clusterDim.y = 1; a[0].val.clusterDim.z = 1;
    cfg.attrs = a; cfg.numAttrs = 1;
    cfg.gridDim = dim3(cs * 8);
    int ncl = 0;
    CK(cudaOccupancyMaxActiveClusters(&ncl, k, &cfg));
    const int grid = cs == 1 ? nsm : ncl * cs;
    cfg.gridDim = dim3(grid);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    float best = 1e30f;
    for (int it = 0; it < 6; ++it) {
        cudaEventRecord(e0);
        CK(cudaLaunchKernelEx(&cfg, k, src, nchunks, stages, mode, out));
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        if (it > 0 && ms < best) best = ms;
    }
    printf("chunk %5d spin %d inflight %3d KB mode %d cluster %2d: %3d CTAs %.3f ms %5.0f GB/s (%.1f GB/s per CTA)\n", CHUNK, (int)SPIN,
           inflight / 1024, mode, cs, grid, best, bytes / (best * 1e-3) / 1e9, bytes / (best * 1e-3) / 1e9 / grid);
    return 0;
}

int main() {
    const size_t bytes = (size_t)3 << 30;
    char* src; float* out;
    CK(cudaMalloc(&src, bytes));
    CK(cudaMemset(src, 0x3c, bytes));
    CK(cudaMalloc(&out, 4096));
    int nsm = 0;
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
    for (int infl : {96 * 1024, 192 * 1024}) {
        run<4096, false>(src, bytes, out, nsm, 0, 1, infl);
        run<8192, false>(src, bytes, out, nsm, 0, 1, infl);
        run<8192, true>(src, bytes, out, nsm, 0, 1, infl);
        run<16384, false>(src, bytes, out, nsm, 0, 1, infl);
        run<32768, false>(src, bytes, out, nsm, 0, 1, infl);
        run<32768, true>(src, bytes, out, nsm, 0, 1, infl);
    }
    for (int cs : {1, 4, 8}) {
        run<32768, false>(src, bytes, out, nsm, 0, cs, 192 * 1024);
        run<16384, false>(src, bytes, out, nsm, 0, cs, 192 * 1024);
        run<16384, false>(src, bytes, out, nsm, 2, cs, 192 * 1024);
    }
    return 0;
}
