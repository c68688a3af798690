// microbench.cu -- B200 (sm_100a) rate probes that fix the design of msd_core:
//   1. read-only HBM bandwidth: persistent CTAs stream a large buffer with
//      cp.async.bulk (TMA) into a shared-memory ring (the K0 probe of SURVEY §7)
//   2. MUFU.EX2 throughput per SM per clock
//   3. TMEM store / load (tcgen05.st / tcgen05.ld) throughput per SM per clock
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o microbench microbench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int STAGES, int CHUNK>
__global__ void __launch_bounds__(128) k_read(const char* buf, size_t bytes, unsigned long long* sink) {
    extern __shared__ __align__(128) char sm[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm + STAGES * CHUNK);
    const size_t nchunks = bytes / CHUNK;
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar[s])));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    auto issue = [&](size_t c, int s) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar[s])), "r"(CHUNK));
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
                     ::"r"(sa(sm + s * CHUNK)), "l"(buf + c * CHUNK), "r"(CHUNK), "r"(sa(&bar[s])), "l"(pol) : "memory");
    };
    size_t j = 0;
    unsigned long long acc = 0;
    if (threadIdx.x == 0)
        for (int s = 0; s < STAGES; ++s) {
            size_t c = blockIdx.x + (size_t)s * gridDim.x;
            if (c < nchunks) issue(c, s);
        }
    for (size_t c = blockIdx.x; c < nchunks; c += gridDim.x, ++j) {
        int s = j % STAGES;
        uint32_t par = (j / STAGES) & 1, done = 0;
        while (!done)
            asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }"
                         : "=r"(done) : "r"(sa(&bar[s])), "r"(par) : "memory");
        acc += reinterpret_cast<const uint32_t*>(sm + s * CHUNK)[threadIdx.x];
        __syncthreads();
        if (threadIdx.x == 0) {
            size_t cn = c + (size_t)STAGES * gridDim.x;
            if (cn < nchunks) issue(cn, s);
        }
    }
    if (acc == 0x12345) sink[0] = acc;
}

__global__ void k_ldg(const uint4* buf, size_t n16, unsigned long long* sink) {
    uint32_t acc = 0;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    for (; i + 3 * stride < n16; i += 4 * stride) {
        uint4 a = __ldcs(buf + i), b = __ldcs(buf + i + stride), c = __ldcs(buf + i + 2 * stride), d = __ldcs(buf + i + 3 * stride);
        acc ^= a.x ^ b.y ^ c.z ^ d.w;
    }
    for (; i < n16; i += stride) acc ^= __ldcs(buf + i).x;
    if (acc == 0x12345) sink[0] = acc;
}

__global__ void k_ex2(float* out, int iters) {
    float x[16];
    for (int i = 0; i < 16; ++i) x[i] = -0.001f * (threadIdx.x + i);
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            float r;
            asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x[i]));
            x[i] = r - 1.0f;
        }
    float s = 0;
    for (int i = 0; i < 16; ++i) s += x[i];
    if (s == 12345.f) out[0] = s;
}

__global__ void k_tmem(float* out, int iters, int do_ld) {
    __shared__ uint32_t taddr_s;
    int warp = threadIdx.x / 32;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(sa(&taddr_s)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    uint32_t base = taddr_s;
    uint32_t ta = base + (((warp & 3) * 32) << 16) + (warp >> 2) * 128;
    float v[16];
    for (int i = 0; i < 16; ++i) v[i] = threadIdx.x + i;
    float s = 0;
    for (int it = 0; it < iters; ++it) {
        uint32_t t = ta + (it & 7) * 16;
        if (!do_ld) {
            asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
                         ::"r"(t), "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]),
                         "f"(v[8]), "f"(v[9]), "f"(v[10]), "f"(v[11]), "f"(v[12]), "f"(v[13]), "f"(v[14]), "f"(v[15]) : "memory");
        } else {
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                         : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7]),
                           "=f"(v[8]), "=f"(v[9]), "=f"(v[10]), "=f"(v[11]), "=f"(v[12]), "=f"(v[13]), "=f"(v[14]), "=f"(v[15])
                         : "r"(t) : "memory");
            if ((it & 3) == 3) asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            s += v[it & 15];
        }
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    if (s == 1234.5f) out[0] = s;
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(base));
}

int main() {
    int nsm, clk;
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
    CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0));
    const size_t bytes = (size_t)4 << 30;
    char* buf;
    CK(cudaMalloc(&buf, bytes));
    CK(cudaMemset(buf, 1, bytes));
    unsigned long long* sink;
    CK(cudaMalloc(&sink, 64));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float ms;
    printf("{\"sms\": %d, \"clock_khz\": %d", nsm, clk);
    // 1a. TMA bulk read
    {
        constexpr int ST = 6, CH = 32768;
        auto k = k_read<ST, CH>;
        size_t smem = ST * CH + 64;
        CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        for (int occ = 1; occ <= 1; ++occ) {
            k<<<nsm * occ, 128, smem>>>(buf, bytes, sink);
            CK(cudaDeviceSynchronize());
            float best = 1e9;
            for (int r = 0; r < 5; ++r) {
                cudaEventRecord(a);
                k<<<nsm * occ, 128, smem>>>(buf, bytes, sink);
                cudaEventRecord(b);
                CK(cudaEventSynchronize(b));
                cudaEventElapsedTime(&ms, a, b);
                if (ms < best) best = ms;
            }
            printf(", \"tma_read_gbs\": %.1f", bytes / (best * 1e-3) / 1e9);
        }
    }
    // 1b. LDG.128 streaming read
    {
        float best = 1e9;
        for (int r = 0; r < 5; ++r) {
            cudaEventRecord(a);
            k_ldg<<<nsm * 8, 512>>>((const uint4*)buf, bytes / 16, sink);
            cudaEventRecord(b);
            CK(cudaEventSynchronize(b));
            cudaEventElapsedTime(&ms, a, b);
            if (ms < best) best = ms;
        }
        printf(", \"ldg_read_gbs\": %.1f", bytes / (best * 1e-3) / 1e9);
    }
    // 2. ex2 throughput
    {
        float* out;
        CK(cudaMalloc(&out, 64));
        int iters = 4096;
        k_ex2<<<nsm * 4, 512>>>(out, 16);
        CK(cudaDeviceSynchronize());
        cudaEventRecord(a);
        k_ex2<<<nsm * 4, 512>>>(out, iters);
        cudaEventRecord(b);
        CK(cudaEventSynchronize(b));
        cudaEventElapsedTime(&ms, a, b);
        double n = (double)nsm * 4 * 512 * iters * 16;
        printf(", \"ex2_per_s\": %.4g, \"ex2_per_clk_per_sm_at_max_clock\": %.2f", n / (ms * 1e-3),
               n / (ms * 1e-3) / nsm / (clk * 1e3));
    }
    // 3. TMEM st / ld
    for (int ld = 0; ld < 2; ++ld) {
        float* out;
        CK(cudaMalloc(&out, 64));
        int iters = 1 << 16;
        k_tmem<<<nsm, 256>>>(out, 64, ld);
        CK(cudaDeviceSynchronize());
        cudaEventRecord(a);
        k_tmem<<<nsm, 256>>>(out, iters, ld);
        cudaEventRecord(b);
        CK(cudaEventSynchronize(b));
        cudaEventElapsedTime(&ms, a, b);
        double byt = (double)nsm * 256 * iters * 64;
        printf(", \"tmem_%s_bytes_per_clk_per_sm\": %.1f", ld ? "ld" : "st", byt / (ms * 1e-3) / nsm / (clk * 1e3));
    }
    printf("}\n");
    return 0;
}
