// msd_core.cu -- the streaming pass over every logit row at the draft positions.
//
// Rows a1 (Eq. 1 normaliser) and a5 (Eq. 5 DTV; KL) of the
// hot path, for all L chain levels at once so that every logit byte is read from
// HBM exactly once.
//
// Work decomposition.  A *unit* is one (request b, draft position i < K); it owns
// the L rows Z_l[b, i, :] (one per level).  A unit is cut into C slices of VS = 4096
// vocabulary entries; an *item* is (unit, slice).  The kernel is persistent and
// cooperative: CTA g processes items g, g+G, g+2G, ... in order, so the C items of
// a unit run concurrently on C different CTAs (G >= C => no deadlock).
//
// Per item:
//   1. TMA (cp.async.bulk) streams the L row slices into a S-stage shared-memory
//      ring; thread 0 keeps S items in flight per CTA.
//   2. pass 1 (registers): per warp, e_v = 2^((z_v - m_w) log2 e) relative to the
//      warp max m_w (one MUFU.EX2 per element), sum S_w and the KL numerator
//      K_w = sum e_v (z_v - z'_v) against the previous level's row.  The e_v stay in
//      registers for pass 2 (no second exp, no second read).
//   3. warp 0 folds the 8 warp records into the slice partial (m_s, S_s, K_s, argmax)
//      and publishes it; the CTA that publishes the unit's last slice combines the C
//      partials (fixed order, float64) into the unit's row stats and releases them.
//   4. pass 2 (registers): with M_l, S_l known, the residual mass of each adjacent
//      pair in this slice, R_s = sum_v max(p_v - q_v, 0) (= its DTV share, and the
//      per-slice CDF the tail's residual draw needs), evaluated as
//      max(e_a - rho e_b, 0) with rho = c_b S_a / (S_b c_a) split into hi+lo floats.
#include "msd_common.cuh"
#include "msd_internal.h"

namespace msd {

template <typename Tin, int L, bool GREEDY>
__global__ void __launch_bounds__(T, 2) core_kernel(CoreParams p) {
    constexpr int VEC = Elem<Tin>::VEC;
    constexpr int NV = ET / VEC;
    constexpr int ES = (int)sizeof(Tin);
    extern __shared__ __align__(128) unsigned char smem[];
    const int S = p.stages;
    Tin* ring = reinterpret_cast<Tin*>(smem);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)S * L * VS * ES);

    __shared__ float w_m[L][NWARP];
    __shared__ float w_S[L][NWARP];
    __shared__ float w_K[L][NWARP];
    __shared__ int w_am[L][NWARP];
    __shared__ double w_R[L][NWARP];
    __shared__ RowStat s_row[L];
    __shared__ double s_K[L];
    __shared__ int s_last;

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t G = gridDim.x;
    const int64_t n_my = p.n_items > (int64_t)blockIdx.x ? (p.n_items - blockIdx.x + G - 1) / G : 0;
    const uint64_t pol = policy_evict_first();

    if (tid == 0) {
        for (int st = 0; st < S; ++st) mbar_init(&full[st], 1);
        fence_mbar_init();
    }
    __syncthreads();

    auto issue = [&](int64_t j) {
        const int64_t w = blockIdx.x + j * G;
        const int64_t u = w / p.C;
        const int s = (int)(w % p.C);
        const int64_t b = u / p.K, i = u % p.K;
        const int st = (int)(j % S);
        const int64_t len = min((int64_t)VS, p.V - (int64_t)s * VS);
        const uint32_t bytes = (uint32_t)((len * ES) / 16 * 16);
        mbar_arrive_expect_tx(&full[st], bytes * L);
        if (bytes) {
#pragma unroll
            for (int l = 0; l < L; ++l) {
                const Tin* src = reinterpret_cast<const Tin*>(p.lv.ptr[l]) + b * p.lv.bs[l] +
                                 i * p.lv.ld[l] + (int64_t)s * VS;
                bulk_g2s(ring + ((size_t)st * L + l) * VS, src, bytes, &full[st], pol);
            }
        }
    };

    if (tid == 0)
        for (int64_t j = 0; j < S && j < n_my; ++j) issue(j);

    for (int64_t j = 0; j < n_my; ++j) {
        const int64_t w = blockIdx.x + j * G;
        const int64_t u = w / p.C;
        const int s = (int)(w % p.C);
        const int64_t b = u / p.K, i = u % p.K;
        const int st = (int)(j % S);
        const int64_t base = (int64_t)s * VS;
        const int len = (int)min((int64_t)VS, p.V - base);
        const int len_bulk = (len * ES) / 16 * 16 / ES;

        mbar_wait(&full[st], (uint32_t)((j / S) & 1));

        // ---------------- pass 1
        float e[L][ET];
        float xprev[ET];
        float wm_r[L];
#pragma unroll
        for (int l = 0; l < L; ++l) {
            float x[ET];
            const Tin* sl = ring + ((size_t)st * L + l) * VS;
#pragma unroll
            for (int jv = 0; jv < NV; ++jv) {
                const int e0 = (jv * T + tid) * VEC;
                if (e0 + VEC <= len_bulk) {
                    uint4 v = *reinterpret_cast<const uint4*>(sl + e0);
                    unpack_clamped<Tin>(v, &x[jv * VEC]);
                } else {
                    const Tin* g = reinterpret_cast<const Tin*>(p.lv.ptr[l]) + b * p.lv.bs[l] +
                                   i * p.lv.ld[l] + base;
#pragma unroll
                    for (int k = 0; k < VEC; ++k) {
                        const int ee = e0 + k;
                        float z = NEG_CLAMP;
                        if (ee < len_bulk) z = clamp1((float)sl[ee]);
                        else if (ee < len) z = clamp1(Elem<Tin>::load1(g + ee));
                        x[jv * VEC + k] = z;
                    }
                }
            }
            float tm = x[0];
#pragma unroll
            for (int k = 1; k < ET; ++k) tm = fmaxf(tm, x[k]);
            const float wm = warp_max(tm);
            wm_r[l] = wm;
            float sum = 0.f, ks = 0.f;
            // KL numerator relative to the shift s_w = m_w,l - m_w,l-1 (restored in float64
            // at the combine) so the dominant term does not sit in the fp32 accumulator.
            const float shift = l > 0 ? wm - wm_r[l > 0 ? l - 1 : 0] : 0.f;
#pragma unroll
            for (int k = 0; k < ET; ++k) {
                const float ev = ex2f((x[k] - wm) * LOG2E);
                e[l][k] = ev;
                sum += ev;
                if (l > 0) ks = fmaf(ev, (x[k] - xprev[k]) - shift, ks);
            }
            sum = warp_sum(sum);
            if (l > 0) ks = warp_sum(ks);
            int am = 0x7fffffff;
            if (GREEDY) {
#pragma unroll
                for (int k = ET - 1; k >= 0; --k)
                    if (x[k] == wm) am = (int)(base + ((k / VEC) * T + tid) * VEC + (k % VEC));
                am = warp_min_i(am);
            }
            if (lane == 0) {
                w_m[l][warp] = wm;
                w_S[l][warp] = sum;
                w_K[l][warp] = ks;
                w_am[l][warp] = am;
            }
#pragma unroll
            for (int k = 0; k < ET; ++k) xprev[k] = x[k];
        }
        __syncthreads();  // B1: stage `st` fully consumed, warp records visible
        if (tid == 0 && j + S < n_my) issue(j + S);

        // ---------------- slice partials -> publish -> unit combine
        if (warp == 0) {
            const int l = lane >> 3, wi = lane & 7;
            const bool act = l < L;
            const float mw = act ? w_m[l][wi] : -INFINITY;
            float ms = mw;
#pragma unroll
            for (int o = 4; o > 0; o >>= 1) ms = fmaxf(ms, __shfl_xor_sync(0xffffffffu, ms, o));
            double f = act ? exp((double)mw - (double)ms) : 0.0;
            if (!(mw > NEG_MASKED)) f = (ms > NEG_MASKED) ? 0.0 : 1.0;  // fully masked warp
            double Ss = act ? (double)w_S[l][wi] * f : 0.0;
            double Ks = 0.0;
            if (act && l > 0 && f != 0.0)
                Ks = ((double)w_K[l][wi] + ((double)mw - (double)w_m[l - 1][wi]) * (double)w_S[l][wi]) * f;
            int am = (act && mw == ms) ? w_am[l][wi] : 0x7fffffff;
#pragma unroll
            for (int o = 4; o > 0; o >>= 1) {
                Ss += __shfl_xor_sync(0xffffffffu, Ss, o);
                Ks += __shfl_xor_sync(0xffffffffu, Ks, o);
                am = min(am, __shfl_xor_sync(0xffffffffu, am, o));
            }
            if (act && wi == 0) {
                Partial pr;
                pr.m = ms;
                pr.amax = am;
                pr.S = Ss;
                pr.Kl = Ks;
                p.partials[((size_t)u * L + l) * p.C + s] = pr;
            }
            __threadfence();
            __syncwarp();
            if (lane == 0) s_last = (atomicAdd(&p.cnt[u], 1u) == (uint32_t)(p.C - 1));
        }
        __syncthreads();
        if (s_last) {
            __threadfence();
            if (warp < L) {
                double Kl;
                RowStat r = combine_row(p.partials + ((size_t)u * L + warp) * p.C, p.C, &Kl);
                if (lane == 0) {
                    s_row[warp] = r;
                    s_K[warp] = Kl;
                    p.rowstat[(size_t)u * L + warp] = r;
                }
            }
            __syncthreads();
            if (tid == 0) {
                bool bad = false;
#pragma unroll
                for (int l = 0; l < L; ++l) bad |= s_row[l].bad != 0;
#pragma unroll
                for (int l = 1; l < L; ++l) {
                    double kl = s_K[l] / s_row[l].S - (s_row[l].lse - s_row[l - 1].lse);
                    p.kl[(size_t)u * (L - 1) + (l - 1)] = kl;
                }
                if (bad) atomicOr(&p.flags[b], (uint32_t)MSD_F_NONFINITE);
                __threadfence();
                st_release_u32(&p.ready[u], 1u);
            }
        } else {
            if (tid == 0) {
                const uint64_t t0 = globaltimer();
                while (ld_acquire_u32(&p.ready[u]) == 0u) {
                    __nanosleep(64);
                    if (globaltimer() - t0 > 4000000000ull) {  // 4 s watchdog
                        atomicOr(p.err, 1u);
                        atomicOr(&p.flags[b], (uint32_t)MSD_F_TIMEOUT);
                        break;
                    }
                }
            }
            __syncthreads();
            if (tid < L) {
                const RowStat* g = p.rowstat + (size_t)u * L + tid;
                RowStat r;
                r.M = __ldcg(&g->M);
                r.S = __ldcg(&g->S);
                r.lse = __ldcg(&g->lse);
                r.amax = __ldcg(&g->amax);
                r.bad = __ldcg(&g->bad);
                s_row[tid] = r;
            }
        }
        __syncthreads();

        // ---------------- pass 2: residual mass of each adjacent pair in this slice
        double c_self = 0.0;   // lane l: exp(m_w,l - M_l)
        if (lane < L) {
            float wml = wm_r[0];
#pragma unroll
            for (int l = 1; l < L; ++l)
                if (lane == l) wml = wm_r[l];
            c_self = (wml > NEG_MASKED) ? exp((double)wml - s_row[lane].M) : 0.0;
        }
#pragma unroll
        for (int l = 1; l < L; ++l) {
            const double ca = __shfl_sync(0xffffffffu, c_self, l);
            const double cb = __shfl_sync(0xffffffffu, c_self, l - 1);
            float acc = 0.f;
            if (ca > 0.0) {
                const double rho = cb * s_row[l].S / (s_row[l - 1].S * ca);
                const float rh = (float)rho;
                const float rl = (float)(rho - (double)rh);
#pragma unroll
                for (int k = 0; k < ET; ++k) {
                    float t = fmaf(-e[l - 1][k], rh, e[l][k]);
                    t = fmaf(-e[l - 1][k], rl, t);
                    acc += fmaxf(t, 0.f);
                }
            }
            acc = warp_sum(acc);
            if (lane == 0) w_R[l][warp] = (double)acc * ca;
        }
        __syncthreads();
        if (warp == 0 && lane >= 1 && lane < L) {
            double R = 0.0;
#pragma unroll
            for (int wi = 0; wi < NWARP; ++wi) R += w_R[lane][wi];
            p.resid[((size_t)u * (L - 1) + (lane - 1)) * p.C + s] = R / s_row[lane].S;
        }
    }
}

template <typename Tin, int L, bool G>
static cudaError_t launch_one(const CoreParams& p0, cudaStream_t s) {
    CoreParams p = p0;
    const int ES = (int)sizeof(Tin);
    const size_t stage_bytes = (size_t)L * VS * ES;
    int S = (int)(98304 / stage_bytes);
    if (S < 2) S = 2;
    if (S > 4) S = 4;
    p.stages = S;
    const size_t smem = stage_bytes * S + 64;
    auto k = core_kernel<Tin, L, G>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int dev = 0, nsm = 0, occ = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, T, smem);
    if (e != cudaSuccess) return e;
    if (occ < 1) return cudaErrorInvalidConfiguration;
    int64_t grid = (int64_t)nsm * occ;
    if (grid > p.n_items) grid = p.n_items;
    if (grid < p.C) return cudaErrorInvalidConfiguration;  // never: C <= 128 < 148
    void* args[] = {&p};
    return cudaLaunchCooperativeKernel((const void*)k, dim3((unsigned)grid), dim3(T), args, smem, s);
}

cudaError_t launch_core(const CoreParams& p, int bf16, int greedy, cudaStream_t s) {
#define MSD_CASE(TY, LL)                                                         \
    if (p.L == LL) return greedy ? launch_one<TY, LL, true>(p, s) : launch_one<TY, LL, false>(p, s);
    if (bf16) {
        MSD_CASE(__nv_bfloat16, 2)
        MSD_CASE(__nv_bfloat16, 3)
        MSD_CASE(__nv_bfloat16, 4)
    } else {
        MSD_CASE(float, 2)
        MSD_CASE(float, 3)
        MSD_CASE(float, 4)
    }
#undef MSD_CASE
    return cudaErrorInvalidValue;
}

}  // namespace msd
