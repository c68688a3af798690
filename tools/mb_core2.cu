// mb_core2.cu -- feasibility probe of a cluster-exchange core design (not the product):
// grid = U units x P parts, clusters of P CTAs (one unit), 2 CTAs per SM.  Each CTA streams its
// share of the unit's L rows through a TMA ring (pass 1: online max / sum / KL numerator, loads
// kept in L2 with evict_last), exchanges the row (max, sum) records through DSMEM (cluster
// barriers), then re-streams the share from L2 (pass 2: normalised p, pair terms) -- no on-chip
// window across the exchange.  Prints the achieved logit GB/s (one HBM read per byte).
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/mb_core2 tools/mb_core2.cu
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

constexpr int L = 3, TH = 256, CH = 2048, S = 8;   // rows, threads, chunk entries, ring stages
constexpr float LOG2E = 1.4426950408889634f;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(n));
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes));
}
__device__ __forceinline__ bool mbar_try(uint64_t* b, uint32_t ph) {
    uint32_t ok;
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(ok) : "r"(smem_u32(b)), "r"(ph) : "memory");
    return ok;
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) { while (!mbar_try(b, ph)) {} }
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
                 ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol) : "memory");
}
__device__ __forceinline__ uint64_t pol_last() { uint64_t p; asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p)); return p; }
__device__ __forceinline__ uint64_t pol_first() { uint64_t p; asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p)); return p; }
__device__ __forceinline__ float ex2f(float x) { float r; asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x)); return r; }
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ float ld_peer(const float* p, uint32_t rank) {
    uint32_t a = smem_u32(p), r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
    float v;
    asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(r));
    return v;
}

struct __align__(128) Sm {
    __nv_bfloat16 ring[S][L][CH];
    uint64_t full[S];
    float rec_m[L], rec_s[L];
    float red[TH / 32][2 * L + 2];
};

__global__ void __launch_bounds__(TH, 2) core2(const __nv_bfloat16* z, int64_t V, int P, float* out, int mode) {
    extern __shared__ __align__(128) unsigned char smraw[];
    Sm& sm = *reinterpret_cast<Sm*>(smraw);
    uint32_t rank;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    const int64_t unit = blockIdx.x / P;
    const int64_t VP = (V / P + 7) / 8 * 8;
    const int64_t v0 = rank * VP, v1 = v0 + VP < V ? v0 + VP : V;
    const int nch = (int)((v1 - v0 + CH - 1) / CH);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const __nv_bfloat16* base = z + unit * L * V;
    if (tid == 0) {
        for (int s = 0; s < S; ++s) mbar_init(&sm.full[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    auto issue = [&](int c, uint64_t pol) {          // chunk c (of 2 * nch: pass 1 then pass 2)
        const int cc = c % nch, st = c % S;
        const int64_t e0 = v0 + (int64_t)cc * CH;
        const uint32_t bytes = (uint32_t)(((v1 - e0) < CH ? (v1 - e0) : CH) * 2);
        mbar_expect(&sm.full[st], bytes * L);
        for (int l = 0; l < L; ++l) bulk_g2s(&sm.ring[st][l][0], base + l * V + e0, bytes, &sm.full[st], pol);
    };
    const int ntot = mode == 3 ? nch : 2 * nch;
    if (tid == 0)
        for (int c = 0; c < S && c < nch; ++c) issue(c, pol_last());
    // ---------------- pass 1
    float m[L], s[L], kl[L];
    for (int l = 0; l < L; ++l) { m[l] = -1e30f; s[l] = 0.f; kl[l] = 0.f; }
    for (int c = 0; c < nch; ++c) {
        const int st = c % S;
        mbar_wait(&sm.full[st], (uint32_t)((c / S) & 1));
        const int64_t e0 = v0 + (int64_t)(c % nch) * CH;
        const int n = (int)((v1 - e0) < CH ? (v1 - e0) : CH);
        for (int i = tid * 8; i < n && mode != 2; i += TH * 8) {
            float x[L][8];
            for (int l = 0; l < L; ++l) {
                const uint4 w = *reinterpret_cast<const uint4*>(&sm.ring[st][l][i]);
                const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
                float mx = m[l];
                for (int k = 0; k < 8; ++k) { x[l][k] = __uint_as_float((ws[k / 2] >> (16 * (k & 1))) << 16); mx = fmaxf(mx, x[l][k]); }
                if (mx > m[l]) { s[l] *= ex2f((m[l] - mx) * LOG2E); kl[l] *= ex2f((m[l] - mx) * LOG2E); m[l] = mx; }
                for (int k = 0; k < 8; ++k) {
                    const float e = ex2f((x[l][k] - m[l]) * LOG2E);
                    s[l] += e;
                    if (l) kl[l] = fmaf(e, x[l][k] - x[l - 1][k], kl[l]);
                }
            }
        }
        __syncthreads();
        if (tid == 0 && c + S < ntot) issue(c + S, c + S < nch ? pol_last() : pol_first());
    }
    // block combine -> this CTA's record, cluster exchange
    for (int l = 0; l < L; ++l) {
        float mw = m[l];
        for (int o = 16; o; o >>= 1) mw = fmaxf(mw, __shfl_xor_sync(~0u, mw, o));
        float sv = s[l] * ex2f((m[l] - mw) * LOG2E);
        for (int o = 16; o; o >>= 1) sv += __shfl_xor_sync(~0u, sv, o);
        if (lane == 0) { sm.red[warp][2 * l] = mw; sm.red[warp][2 * l + 1] = sv; }
    }
    __syncthreads();
    if (tid < L) {
        float M = -1e30f, Sx = 0.f;
        for (int w = 0; w < TH / 32; ++w) M = fmaxf(M, sm.red[w][2 * tid]);
        for (int w = 0; w < TH / 32; ++w) Sx += sm.red[w][2 * tid + 1] * ex2f((sm.red[w][2 * tid] - M) * LOG2E);
        sm.rec_m[tid] = M; sm.rec_s[tid] = Sx;
    }
    cluster_sync();
    float Mr[L], iS[L];
    for (int l = 0; l < L; ++l) {
        float M = -1e30f, Sx = 0.f;
        for (int q = 0; q < P; ++q) M = fmaxf(M, ld_peer(&sm.rec_m[l], q));
        for (int q = 0; q < P; ++q) Sx += ld_peer(&sm.rec_s[l], q) * ex2f((ld_peer(&sm.rec_m[l], q) - M) * LOG2E);
        Mr[l] = M; iS[l] = 1.f / Sx;
    }
    cluster_sync();
    // ---------------- pass 2 (re-streamed from L2)
    float r2[L];
    for (int l = 0; l < L; ++l) r2[l] = 0.f;
    for (int c = nch; c < ntot; ++c) {  // (mode 3: none)
        const int st = c % S;
        mbar_wait(&sm.full[st], (uint32_t)((c / S) & 1));
        const int64_t e0 = v0 + (int64_t)(c % nch) * CH;
        const int n = (int)((v1 - e0) < CH ? (v1 - e0) : CH);
        for (int i = tid * 8; i < n && mode == 0; i += TH * 8) {
            float pprev[8];
            for (int l = 0; l < L; ++l) {
                const uint4 w = *reinterpret_cast<const uint4*>(&sm.ring[st][l][i]);
                const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
                for (int k = 0; k < 8; ++k) {
                    const float x = __uint_as_float((ws[k / 2] >> (16 * (k & 1))) << 16);
                    const float p = ex2f((x - Mr[l]) * LOG2E) * iS[l];
                    if (l) r2[l] += fmaxf(p - pprev[k], 0.f);
                    pprev[k] = p;
                }
            }
        }
        __syncthreads();
        if (tid == 0 && c + S < ntot) issue(c + S, pol_first());
    }
    for (int l = 1; l < L; ++l) {
        float v = r2[l] + kl[l];
        for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(~0u, v, o);
        if (lane == 0) atomicAdd(&out[unit * L + l], v);
    }
}

int main() {
    const int64_t V = 128256;
    const int U = 4096;
    std::vector<int> Ps = {8, 4};
    size_t n = (size_t)U * L * V;
    __nv_bfloat16* z;
    float* out;
    cudaMalloc(&z, n * 2);
    cudaMalloc(&out, (size_t)U * L * 4);
    std::vector<__nv_bfloat16> h(1 << 20);
    for (size_t i = 0; i < h.size(); ++i) h[i] = __float2bfloat16((float)((i * 2654435761u) % 1000) / 100.f - 5.f);
    for (size_t o = 0; o < n; o += h.size()) cudaMemcpy(z + o, h.data(), std::min(h.size(), n - o) * 2, cudaMemcpyHostToDevice);
    const size_t smem = sizeof(Sm);
    cudaFuncSetAttribute(core2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (int mode = 0; mode < 4; ++mode)
    for (int P : Ps) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)(U * P));
        cfg.blockDim = dim3(TH);
        cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = P; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        int ncl = 0;
        cudaOccupancyMaxActiveClusters(&ncl, core2, &cfg);
        cudaEvent_t a, b;
        cudaEventCreate(&a); cudaEventCreate(&b);
        for (int it = 0; it < 3; ++it) cudaLaunchKernelEx(&cfg, core2, (const __nv_bfloat16*)z, V, P, out, mode);
        cudaEventRecord(a);
        const int R = 10;
        for (int it = 0; it < R; ++it) cudaLaunchKernelEx(&cfg, core2, (const __nv_bfloat16*)z, V, P, out, mode);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        ms /= R;
        printf("mode %d P=%d smem %zu B, active clusters %d: %.3f ms  %.0f GB/s  (%s)\n", mode, P, smem, ncl, ms, n * 2 / (ms * 1e-3) / 1e9,
               cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
