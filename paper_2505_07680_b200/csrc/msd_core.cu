// msd_core.cu -- the streaming pass over every logit row at the draft positions.
//
// Rows a1 (Eq. 1 normaliser) and a5 (Eq. 5 DTV; KL) of the
// hot path, for all L chain levels at once so every logit byte is read from HBM
// exactly once.
//
// Decomposition.  A *unit* is one (request b, draft position i < K) and owns the L
// rows Z_l[b, i, :].  A unit is cut into C slices of VS = 4096 vocabulary entries;
// an *item* is (unit, slice).  The kernel is persistent and cooperative (one CTA per
// SM): CTA g processes items g, g+G, g+2G, ...; the C items of a unit run
// concurrently on C CTAs, which exchange per-slice partials through global memory.
//
// Warp specialisation (15 warps):
//   warps 0-7  compute: pass 1 of item j  -- slice max (named barrier among compute
//                warps), e_v = 2^((z_v - m_s) log2 e) (one MUFU.EX2 per element), sums S
//                and the KL numerator, e_v parked in TMEM (tcgen05.st);
//              then pass 2 of item j-LAG -- e_v back from TMEM (tcgen05.ld), residual
//                mass of each adjacent pair  sum_v max(p_v - q_v, 0)  in this slice.
//   warp 8     producer: TMA bulk copies (cp.async.bulk) of the L row slices into an
//                S-stage shared-memory ring.
//   warp 9     publisher: folds the compute warps' records into the slice partial,
//                publishes it and bumps the unit counter (release); the CTA completing
//                a unit later combines its row statistics for the tail kernel (idle time).
//   warps 10-13 fetchers (items j = f mod 4): wait for the unit counter, combine the
//                unit's compact partials (float64, fixed order) and derive this slice's
//                pass-2 factors.
//   warp 14    reducer: sums the pass-2 warp records into the slice residual R_s.
// The exchange latency is hidden behind LAG items of pass 1 (TMEM holds LAG+1 items
// of exponentials per compute thread: 256 columns / (16 L)).
#include "msd_common.cuh"
#include "msd_internal.h"

namespace msd {

constexpr int NCW = 8;                 // compute warps
constexpr int CT = NCW * 32;           // compute threads (the slice mapping uses CT == T)
constexpr int NFETCH = 4;              // fetcher warps (items j = f mod NFETCH)
constexpr int CORE_THREADS = CT + (3 + NFETCH) * 32;
constexpr int W_PROD = 8, W_PUB = 9, W_FETCH0 = 10, W_RED = W_FETCH0 + NFETCH;
constexpr int NDEFER = 64;
constexpr int SMAX = 6;
constexpr int NRMAX = 8;
static_assert(CT == T, "slice mapping assumes 256 compute threads");

struct Rec1 {
    float S, K;
    int am;
    float pad;
};
struct RowF {               // pass-2 factors of one row of the current slice
    float rho_hi, rho_lo;   // rho = c_b S_a / (S_b c_a) for the pair ending at this row
    double scale;           // c_a / S_a
    int skip;               // c_a == 0: the slice carries no mass of this row
    int pad;
};
template <int L>
struct Ctl {
    uint64_t full[SMAX], empty[SMAX];
    uint64_t rec1_full[NRMAX], rowf_full[NRMAX], rowf_empty[NRMAX], rec2_full[NRMAX], rec2_empty[NRMAX];
    uint32_t taddr;
    float wmax[2][L][NWARP];
    float ms[NRMAX][L];
    Rec1 rec1[NRMAX][L][NWARP];
    RowF rowf[NRMAX][L];
    double rec2[NRMAX][L][NWARP];
    double rec2_scale[NRMAX][L];
    int rec2_skip[NRMAX][L];
    int64_t defer[NDEFER];       // units whose tail-side combine this CTA owes (publisher-private)
};

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void bar_compute() { asm volatile("bar.sync 1, 256;" ::: "memory"); }

__device__ __forceinline__ uint32_t atom_add_release(uint32_t* p, uint32_t v) {
    uint32_t r;
    asm volatile("atom.release.gpu.global.add.u32 %0, [%1], %2;" : "=r"(r) : "l"(p), "r"(v) : "memory");
    return r;
}
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
    uint32_t done;
    asm volatile(
        "{ .reg .pred p; mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return done != 0;
}
__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ uint32_t ld_relaxed_u32(const uint32_t* p) {
    uint32_t r;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(r) : "l"(p) : "memory");
    return r;
}

__device__ __forceinline__ void tm_st16(uint32_t ta, const float* v) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(ta),
        "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]), "f"(v[8]), "f"(v[9]),
        "f"(v[10]), "f"(v[11]), "f"(v[12]), "f"(v[13]), "f"(v[14]), "f"(v[15])
        : "memory");
}
__device__ __forceinline__ void tm_ld16(uint32_t ta, float* v) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7]), "=f"(v[8]),
          "=f"(v[9]), "=f"(v[10]), "=f"(v[11]), "=f"(v[12]), "=f"(v[13]), "=f"(v[14]), "=f"(v[15])
        : "r"(ta)
        : "memory");
}
__device__ __forceinline__ void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tm_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ uint32_t clamp_bf16x2(uint32_t w) { return max_nan_bf16x2(w, 0xF149F149u); }

template <typename Tin, int L, bool GREEDY>
__global__ void __launch_bounds__(CORE_THREADS, 1) core_kernel(CoreParams p) {
    constexpr int VEC = Elem<Tin>::VEC;
    constexpr int NV = ET / VEC;
    constexpr int ES = (int)sizeof(Tin);
    constexpr int NR = 256 / (16 * L);      // TMEM item slots per compute thread
    constexpr int LAG = NR - 1;
    static_assert(NR <= NRMAX && NR >= 2, "TMEM slots");
    extern __shared__ __align__(128) unsigned char smem[];
    const int S = p.stages;
    Tin* ring = reinterpret_cast<Tin*>(smem);
    Ctl<L>& c = *reinterpret_cast<Ctl<L>*>(smem + align_up((size_t)S * L * VS * ES, 128));

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t G = gridDim.x;
    const int64_t n_my = p.n_items > (int64_t)blockIdx.x ? (p.n_items - blockIdx.x + G - 1) / G : 0;
    const int C = p.C;

    if (warp == W_PROD) {
        if (lane == 0) {
            for (int s = 0; s < S; ++s) { mbar_init(&c.full[s], 1); mbar_init(&c.empty[s], NCW); }
            for (int q = 0; q < NR; ++q) {
                mbar_init(&c.rec1_full[q], NCW);
                mbar_init(&c.rowf_full[q], 1);
                mbar_init(&c.rowf_empty[q], NCW);
                mbar_init(&c.rec2_full[q], NCW);
                mbar_init(&c.rec2_empty[q], 1);
            }
            fence_mbar_init();
        }
        __syncwarp();
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&c.taddr)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");

    auto stamp = [&](int64_t j, int k) {
        if (p.trace) p.trace[(blockIdx.x + j * G) * 8 + k] = globaltimer();
    };
    auto item = [&](int64_t j, int64_t& u, int& s, int64_t& b, int64_t& i) {
        const int64_t w = blockIdx.x + j * G;
        u = w / C;
        s = (int)(w % C);
        b = u / p.K;
        i = u % p.K;
    };

    if (warp < NCW) {
        // ================================================================ compute warps
        const uint32_t tbase = c.taddr + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)((warp >> 2) * 256);
        for (int64_t j = 0; j < n_my + LAG; ++j) {
            if (j < n_my) {
                int64_t u, b, i;
                int s;
                item(j, u, s, b, i);
                const int st = (int)(j % S);
                const int q = (int)(j % NR);
                const int64_t base = (int64_t)s * VS;
                const int len = (int)min((int64_t)VS, p.V - base);
                const int len_bulk = (len * ES) / 16 * 16 / ES;
                mbar_wait(&c.full[st], (uint32_t)((j / S) & 1));
                if (tid == 0) stamp(j, 1);
                // ---- raw rows -> registers (clamped), warp max per row
                uint4 raw[L][NV];
#pragma unroll
                for (int l = 0; l < L; ++l) {
                    const Tin* sl = ring + ((size_t)st * L + l) * VS;
#pragma unroll
                    for (int jv = 0; jv < NV; ++jv) {
                        const int e0 = (jv * T + tid) * VEC;
                        if (e0 + VEC <= len_bulk) {
                            raw[l][jv] = *reinterpret_cast<const uint4*>(sl + e0);
                        } else {   // ragged end of the row: element-wise from smem / global
                            const Tin* g = reinterpret_cast<const Tin*>(p.lv.ptr[l]) + b * p.lv.bs[l] +
                                           i * p.lv.ld[l] + base;
                            Tin xs[VEC];
#pragma unroll
                            for (int k = 0; k < VEC; ++k) {
                                const int ee = e0 + k;
                                Tin z = (Tin)(-INFINITY);
                                if (ee < len_bulk) z = sl[ee];
                                else if (ee < len) z = g[ee];
                                xs[k] = z;
                            }
                            raw[l][jv] = *reinterpret_cast<const uint4*>(xs);
                        }
                    }
                }
                float msl[L];
#pragma unroll
                for (int l = 0; l < L; ++l) {
                    float tm = -INFINITY;
                    if (ES == 2) {
                        uint32_t mx = 0xFF80FF80u;  // (-inf, -inf)
#pragma unroll
                        for (int jv = 0; jv < NV; ++jv) {
                            raw[l][jv].x = clamp_bf16x2(raw[l][jv].x);
                            raw[l][jv].y = clamp_bf16x2(raw[l][jv].y);
                            raw[l][jv].z = clamp_bf16x2(raw[l][jv].z);
                            raw[l][jv].w = clamp_bf16x2(raw[l][jv].w);
                            mx = max_nan_bf16x2(mx, max_nan_bf16x2(max_nan_bf16x2(raw[l][jv].x, raw[l][jv].y),
                                                                   max_nan_bf16x2(raw[l][jv].z, raw[l][jv].w)));
                        }
                        tm = fmaxf(bf16lo(mx), bf16hi(mx));
                    } else {
#pragma unroll
                        for (int jv = 0; jv < NV; ++jv) {
                            float xs[4];
                            unpack_clamped<float>(raw[l][jv], xs);
                            raw[l][jv] = make_uint4(__float_as_uint(xs[0]), __float_as_uint(xs[1]),
                                                    __float_as_uint(xs[2]), __float_as_uint(xs[3]));
                            tm = fmaxf(tm, fmaxf(fmaxf(xs[0], xs[1]), fmaxf(xs[2], xs[3])));
                        }
                    }
                    tm = warp_max(tm);
                    if (lane == 0) c.wmax[j & 1][l][warp] = tm;
                }
                bar_compute();
#pragma unroll
                for (int l = 0; l < L; ++l) {
                    float m = lane < NWARP ? c.wmax[j & 1][l][lane] : -INFINITY;
#pragma unroll
                    for (int o = 4; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
                    msl[l] = __shfl_sync(0xffffffffu, m, 0);
                }
                if (warp == 0 && lane == 0) {
#pragma unroll
                    for (int l = 0; l < L; ++l) c.ms[q][l] = msl[l];
                }
                // ---- exponentials relative to the slice max, sums, TMEM park
                float xprev[ET];
#pragma unroll
                for (int l = 0; l < L; ++l) {
                    float x[ET];
#pragma unroll
                    for (int jv = 0; jv < NV; ++jv) {
                        const uint4 r = raw[l][jv];
                        if (ES == 2) {
                            x[jv * 8 + 0] = bf16lo(r.x); x[jv * 8 + 1] = bf16hi(r.x);
                            x[jv * 8 + 2] = bf16lo(r.y); x[jv * 8 + 3] = bf16hi(r.y);
                            x[jv * 8 + 4] = bf16lo(r.z); x[jv * 8 + 5] = bf16hi(r.z);
                            x[jv * 8 + 6] = bf16lo(r.w); x[jv * 8 + 7] = bf16hi(r.w);
                        } else {
                            x[(jv * 4 + 0) % ET] = __uint_as_float(r.x); x[(jv * 4 + 1) % ET] = __uint_as_float(r.y);
                            x[(jv * 4 + 2) % ET] = __uint_as_float(r.z); x[(jv * 4 + 3) % ET] = __uint_as_float(r.w);
                        }
                    }
                    const float m = msl[l];
                    const float shift = l > 0 ? m - msl[l > 0 ? l - 1 : 0] : 0.f;
                    float e[ET];
                    float sum = 0.f, ks = 0.f;
#pragma unroll
                    for (int k = 0; k < ET; ++k) {
                        e[k] = ex2f((x[k] - m) * LOG2E);
                        sum += e[k];
                        if (l > 0) ks = fmaf(e[k], (x[k] - xprev[k]) - shift, ks);
                    }
                    tm_st16(tbase + (uint32_t)(q * 16 * L + l * 16), e);
                    sum = warp_sum(sum);
                    if (l > 0) ks = warp_sum(ks);
                    int am = 0x7fffffff;
                    if (GREEDY) {
#pragma unroll
                        for (int k = ET - 1; k >= 0; --k)
                            if (x[k] == m) am = (int)(base + ((k / VEC) * T + tid) * VEC + (k % VEC));
                        am = warp_min_i(am);
                    }
                    if (lane == 0) {
                        Rec1 r;
                        r.S = sum; r.K = ks; r.am = am; r.pad = 0.f;
                        c.rec1[q][l][warp] = r;
                    }
#pragma unroll
                    for (int k = 0; k < ET; ++k) xprev[k] = x[k];
                }
                tm_wait_st();
                __syncwarp();
                if (tid == 0) stamp(j, 2);
                if (lane == 0) {
                    mbar_arrive(&c.empty[st]);
                    mbar_arrive(&c.rec1_full[q]);
                }
            }
            if (j >= LAG) {
                // ---- pass 2 of item j2 = j - LAG
                const int64_t j2 = j - LAG;
                const int q2 = (int)(j2 % NR);
                mbar_wait(&c.rowf_full[q2], (uint32_t)((j2 / NR) & 1));
                if (tid == 0) stamp(j2, 6);
                RowF f[L];
#pragma unroll
                for (int l = 0; l < L; ++l) f[l] = c.rowf[q2][l];
                __syncwarp();
                if (lane == 0) mbar_arrive(&c.rowf_empty[q2]);
                float ev[L][ET];
#pragma unroll
                for (int l = 0; l < L; ++l) tm_ld16(tbase + (uint32_t)(q2 * 16 * L + l * 16), ev[l]);
                tm_wait_ld();
                float acc[L];
#pragma unroll
                for (int l = 1; l < L; ++l) {
                    float a = 0.f;
                    if (!f[l].skip) {
                        const float rh = f[l].rho_hi, rl = f[l].rho_lo;
#pragma unroll
                        for (int k = 0; k < ET; ++k) {
                            float t = fmaf(-ev[l - 1][k], rh, ev[l][k]);
                            t = fmaf(-ev[l - 1][k], rl, t);
                            a += fmaxf(t, 0.f);
                        }
                    }
                    acc[l] = warp_sum(a);
                }
                if (j2 >= NR) mbar_wait(&c.rec2_empty[q2], (uint32_t)(((j2 / NR) - 1) & 1));
                if (lane == 0) {
#pragma unroll
                    for (int l = 1; l < L; ++l) c.rec2[q2][l][warp] = (double)acc[l];
                    if (warp == 0) {
#pragma unroll
                        for (int l = 1; l < L; ++l) {
                            c.rec2_scale[q2][l] = f[l].scale;
                            c.rec2_skip[q2][l] = f[l].skip;
                        }
                    }
                }
                __syncwarp();
                if (tid == 0) stamp(j2, 7);
                if (lane == 0) mbar_arrive(&c.rec2_full[q2]);
            }
        }
    } else if (warp == W_PROD) {
        // ================================================================ TMA producer
        if (lane == 0) {
            const uint64_t pol = policy_evict_first();
            for (int64_t j = 0; j < n_my; ++j) {
                const int st = (int)(j % S);
                if (j >= S) mbar_wait(&c.empty[st], (uint32_t)(((j / S) - 1) & 1));
                int64_t u, b, i;
                int s;
                item(j, u, s, b, i);
                const int64_t len = min((int64_t)VS, p.V - (int64_t)s * VS);
                const uint32_t bytes = (uint32_t)((len * ES) / 16 * 16);
                stamp(j, 0);
                mbar_arrive_expect_tx(&c.full[st], bytes * L);
                if (bytes) {
#pragma unroll
                    for (int l = 0; l < L; ++l) {
                        const Tin* src = reinterpret_cast<const Tin*>(p.lv.ptr[l]) + b * p.lv.bs[l] +
                                         i * p.lv.ld[l] + (int64_t)s * VS;
                        bulk_g2s(ring + ((size_t)st * L + l) * VS, src, bytes, &c.full[st], pol);
                    }
                }
            }
        }
    } else if (warp == W_PUB) {
        // ================================================================ publisher
        // Publishes each item's slice partial (compact (m, S) for the pass-2 exchange, full
        // record for the tail) and bumps the unit counter with release semantics.  The CTA
        // that completes a unit owes the unit's row statistics / KL to the tail kernel; that
        // combine is off the critical path and runs whenever the publisher is idle.
        int nd = 0, hd = 0;
        int64_t prev_u = -1;
        uint32_t prev_old = 0;
        auto combine_unit = [&](int64_t u) {
            fence_acq_rel_gpu();
            RowStat rs[L];
            double Kl[L];
#pragma unroll
            for (int l = 0; l < L; ++l) rs[l] = combine_row(p.partials + ((size_t)u * L + l) * C, C, &Kl[l]);
            if (lane == 0) {
                bool bad = false;
#pragma unroll
                for (int l = 0; l < L; ++l) {
                    p.rowstat[(size_t)u * L + l] = rs[l];
                    bad |= rs[l].bad != 0;
                }
#pragma unroll
                for (int l = 1; l < L; ++l)
                    p.kl[(size_t)u * (L - 1) + (l - 1)] = Kl[l] / rs[l].S - (rs[l].lse - rs[l - 1].lse);
                if (bad) atomicOr(&p.flags[u / p.K], (uint32_t)MSD_F_NONFINITE);
            }
            __syncwarp();
        };
        for (int64_t j = 0; j < n_my; ++j) {
            int64_t u, b, i;
            int s;
            item(j, u, s, b, i);
            const int q = (int)(j % NR);
            const uint32_t par = (uint32_t)((j / NR) & 1);
            while (!mbar_test(&c.rec1_full[q], par)) {
                if (hd < nd) combine_unit(c.defer[(hd++) % NDEFER]);
                else __nanosleep(20);
            }
            const int l = lane >> 3, wi = lane & 7;
            const bool act = l < L;
            double Ss = act ? (double)c.rec1[q][l][wi].S : 0.0;
            double Ks = act ? (double)c.rec1[q][l][wi].K : 0.0;
            int am = act ? c.rec1[q][l][wi].am : 0x7fffffff;
#pragma unroll
            for (int o = 4; o > 0; o >>= 1) {
                Ss += __shfl_xor_sync(0xffffffffu, Ss, o);
                Ks += __shfl_xor_sync(0xffffffffu, Ks, o);
                am = min(am, __shfl_xor_sync(0xffffffffu, am, o));
            }
            // lane 0 writes every row's records itself so its release covers them
            double Sr[L], Kr[L];
            int ar[L];
#pragma unroll
            for (int r = 0; r < L; ++r) {
                Sr[r] = __shfl_sync(0xffffffffu, Ss, r * 8);
                Kr[r] = __shfl_sync(0xffffffffu, Ks, r * 8);
                ar[r] = __shfl_sync(0xffffffffu, am, r * 8);
            }
            uint32_t old = 0;
            if (lane == 0) {
#pragma unroll
                for (int r = 0; r < L; ++r) {
                    const float m = c.ms[q][r];
                    const size_t idx = ((size_t)u * L + r) * C + s;
                    p.partms[idx] = make_float2(m, (float)Sr[r]);
                    Partial pr;
                    pr.m = m;
                    pr.amax = ar[r];
                    pr.S = Sr[r];
                    // restore the per-slice KL shift (m_l - m_{l-1}) in float64
                    pr.Kl = r > 0 ? Kr[r] + ((double)m - (double)c.ms[q][r > 0 ? r - 1 : 0]) * Sr[r] : 0.0;
                    p.partials[idx] = pr;
                }
                old = atom_add_release(&p.cnt[(size_t)u * CNT_STRIDE], 1u);
                stamp(j, 3);
            }
            // the counter result of the previous item is examined now (its latency was hidden)
            const uint32_t po = __shfl_sync(0xffffffffu, prev_old, 0);
            if (prev_u >= 0 && po == (uint32_t)(C - 1)) {
                if (nd - hd >= NDEFER) combine_unit(c.defer[(hd++) % NDEFER]);
                if (lane == 0) c.defer[nd % NDEFER] = prev_u;
                __syncwarp();
                ++nd;
            }
            prev_u = u;
            prev_old = old;
        }
        if (prev_u >= 0 && __shfl_sync(0xffffffffu, prev_old, 0) == (uint32_t)(C - 1)) {
            if (lane == 0) c.defer[nd % NDEFER] = prev_u;
            __syncwarp();
            ++nd;
        }
        while (hd < nd) combine_unit(c.defer[(hd++) % NDEFER]);
    } else if (warp >= W_FETCH0 && warp < W_FETCH0 + NFETCH) {
        // ================================================================ fetchers (pass-2 factors)
        // Fetcher f serves items j = f (mod NFETCH) in order: wait for the unit counter
        // (relaxed polling, one acquire fence), load the unit's L*C compact partials in one
        // round trip, combine them (float64, fixed order) and derive this slice's pass-2
        // factors.  A fetcher only ever blocks on the next item it owns.
        constexpr int MAXT = (MAXL * 128 + 31) / 32;
        const int f = warp - W_FETCH0;
        const int LC = L * C;
        for (int64_t j = f; j < n_my; j += NFETCH) {
            int64_t u, b, i;
            int s;
            item(j, u, s, b, i);
            const int q = (int)(j % NR);
            if (lane == 0) {
                const uint64_t t0 = globaltimer();
                while (ld_relaxed_u32(&p.cnt[(size_t)u * CNT_STRIDE]) < (uint32_t)C) {
                    __nanosleep(128);
                    if (globaltimer() - t0 > 4000000000ull) {
                        atomicOr(p.err, 1u);
                        atomicOr(&p.flags[b], (uint32_t)MSD_F_TIMEOUT);
                        break;
                    }
                }
                fence_acq_rel_gpu();
                stamp(j, 4);
            }
            __syncwarp();
            const float2* pm = p.partms + (size_t)u * LC;
            float2 v[MAXT];
#pragma unroll
            for (int t = 0; t < MAXT; ++t) {
                const int idx = t * 32 + lane;
                v[t] = idx < LC ? __ldcg(&pm[idx]) : make_float2(-INFINITY, 0.f);
            }
            double Ml[L], Sl[L];
#pragma unroll
            for (int l = 0; l < L; ++l) {
                float m = -INFINITY;
#pragma unroll
                for (int t = 0; t < MAXT; ++t) {
                    const int idx = t * 32 + lane;
                    if (idx >= l * C && idx < (l + 1) * C) m = fmaxf(m, v[t].x);
                }
                Ml[l] = (double)warp_max(m);
            }
#pragma unroll
            for (int l = 0; l < L; ++l) {
                double S = 0.0;
#pragma unroll
                for (int t = 0; t < MAXT; ++t) {
                    const int idx = t * 32 + lane;
                    if (idx >= l * C && idx < (l + 1) * C && v[t].x > NEG_MASKED)
                        S += (double)v[t].y * exp((double)v[t].x - Ml[l]);
                }
                Sl[l] = warp_sum_d(S);
            }
            if (lane == 0) {
                RowF fr[L];
                double cl[L];
#pragma unroll
                for (int l = 0; l < L; ++l) {
                    const float m = c.ms[q][l];
                    cl[l] = (m > NEG_MASKED && Ml[l] > NEG_MASKED) ? exp((double)m - Ml[l]) : 0.0;
                }
                fr[0].rho_hi = fr[0].rho_lo = 0.f;
                fr[0].scale = 0.0;
                fr[0].skip = 1;
                fr[0].pad = 0;
#pragma unroll
                for (int l = 1; l < L; ++l) {
                    const bool skip = !(cl[l] > 0.0) || !(Sl[l] > 0.0) || !(Sl[l - 1] > 0.0) || !isfinite(Sl[l]) ||
                                      !isfinite(Sl[l - 1]);
                    const double rho = skip ? 0.0 : cl[l - 1] * Sl[l] / (Sl[l - 1] * cl[l]);
                    fr[l].rho_hi = (float)rho;
                    fr[l].rho_lo = (float)(rho - (double)fr[l].rho_hi);
                    fr[l].scale = skip ? 0.0 : cl[l] / Sl[l];
                    fr[l].skip = skip ? 1 : 0;
                    fr[l].pad = 0;
                }
                if (j >= NR) mbar_wait(&c.rowf_empty[q], (uint32_t)(((j / NR) - 1) & 1));
#pragma unroll
                for (int l = 0; l < L; ++l) c.rowf[q][l] = fr[l];
                stamp(j, 5);
                mbar_arrive(&c.rowf_full[q]);
            }
            __syncwarp();
        }
    } else if (warp == W_RED) {
        // ================================================================ reducer (slice residual)
        for (int64_t j = 0; j < n_my; ++j) {
            int64_t u, b, i;
            int s;
            item(j, u, s, b, i);
            const int q = (int)(j % NR);
            mbar_wait(&c.rec2_full[q], (uint32_t)((j / NR) & 1));
            const int l = 1 + (lane >> 3), wi = lane & 7;
            const bool act = l < L;
            double R = act ? c.rec2[q][l][wi] : 0.0;
#pragma unroll
            for (int o = 4; o > 0; o >>= 1) R += __shfl_xor_sync(0xffffffffu, R, o);
            if (act && wi == 0) {
                const double v = c.rec2_skip[q][l] ? 0.0 : R * c.rec2_scale[q][l];
                p.resid[((size_t)u * (L - 1) + (l - 1)) * C + s] = v;
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&c.rec2_empty[q]);
        }
    }

    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (warp == W_PROD) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(c.taddr));
}

template <typename Tin, int L, bool G>
static cudaError_t launch_one(const CoreParams& p0, cudaStream_t s) {
    CoreParams p = p0;
    const int ES = (int)sizeof(Tin);
    const size_t stage_bytes = (size_t)L * VS * ES;
    int S = (int)(147456 / stage_bytes);
    if (S < 2) S = 2;
    if (S > SMAX) S = SMAX;
    p.stages = S;
    const size_t smem = align_up(stage_bytes * S, 128) + sizeof(Ctl<L>) + 128;
    auto k = core_kernel<Tin, L, G>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int dev = 0, nsm = 0, occ = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, CORE_THREADS, smem);
    if (e != cudaSuccess) return e;
    if (occ < 1) return cudaErrorInvalidConfiguration;
    int64_t grid = nsm;                    // one CTA per SM (it owns all 512 TMEM columns)
    if (grid > p.n_items) grid = p.n_items;
    if (grid < p.C && grid < p.n_items) return cudaErrorInvalidConfiguration;
    void* args[] = {&p};
    return cudaLaunchCooperativeKernel((const void*)k, dim3((unsigned)grid), dim3(CORE_THREADS), args, smem, s);
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
