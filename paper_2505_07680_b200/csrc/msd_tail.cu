// msd_tail.cu -- the per-request cascade after the streaming pass.
//
// Rows a2 (acceptance, P:64 / S:349-350), a3 (first rejection and cascade,
// P:64), a4 (residual / bonus draw), a5
// (per-position DTV / KL outputs and stats) and a6 (commit and per-model rollback
// lengths).  One CTA per request; levels run in order because level
// l+1's candidates are level l's emission.
//
// Draws.  The core published, for every draft-position row pair, the residual
// mass R_s of each 4096-entry vocabulary slice (and the slice partials from which
// the bonus mass P_s follows).  A draw picks the slice from these (float64
// prefix) and rescans only that slice in float64 (`draw_fast`).  When the
// residual mass is small (Z < z_safe, default 0.01) or the target is within the margin of a
// slice / token boundary, the fp32-derived slice masses are not
// accurate enough relative to Z, so the whole row pair is recomputed in float64
// (`draw_exact`, flagged MSD_F_EXACT_DRAW).  Rows at positions >= K (bonus rows,
// needed only when a level accepts everything) are computed on demand here.
#include "msd_common.cuh"
#include "msd_internal.h"

namespace msd {

constexpr int MAXSLICES = 128;   // V <= 524288

#ifdef MSD_PROF
__device__ unsigned long long g_tail_prof[16];
__device__ unsigned long long g_tail_cta[4096][2];   // per request: start / end globaltimer
__device__ unsigned long long g_tail_req[4096][16];  // per request: cycles per phase
#define TPROF_DECL long long _tp = clock64();
#define TPROF(k) if (threadIdx.x == 0) { const long long _t = clock64(); atomicAdd(&g_tail_prof[k], (unsigned long long)(_t - _tp)); if (blockIdx.x < 4096) g_tail_req[blockIdx.x][k] += (unsigned long long)(_t - _tp); _tp = _t; }
#else
#define TPROF_DECL
#define TPROF(k)
#endif
constexpr double TIE_EPS = 1e-6;
// Fast-path draws (Z >= z_safe) decide a crossing only when it is farther than DRAW_MARGIN * Z
// from the chosen slice's and token's boundaries; the fp32-derived masses drift by ~3e-8 / Z
// (R4), far inside the margin.  Otherwise the exact path decides.
constexpr double DRAW_MARGIN_REL = 2e-5, DRAW_MARGIN_ABS = 0.0;
// u Z this close (relative to Z) to a slice boundary of the fp32-derived slice prefix: the slice
// itself may be the wrong one, so the exact path re-selects it from float64 slice masses.  The
// prefix error relative to Z grows as the residual mass shrinks (~3e-8 / Z measured), so the
// margin is max(1e-6, 1.5e-7 / Z): 5x the drift down to z_safe = 0.01
constexpr double SLICE_MARGIN_REL = 1e-6, SLICE_MARGIN_Z = 1.5e-7;

struct TailShared {
    RowStat row[MAXC][MAXL];      // row statistics of draft positions i < K (from the core partials)
    double kl[MAXC][MAXL];        // KL(p_l || p_{l-1}) at draft position i, l >= 1
    int32_t c[MAXL + 1][MAXC];    // c_l: candidates fed to verifier l (l = 1..L-1); c_L = commit
    int32_t m[MAXL + 1];
    int32_t n[MAXL];
    RowStat extra[MAXL][MAXL];    // rows at positions K..K+L-2, per level
    int32_t extra_ok[MAXL][MAXL];
    double w[MAXSLICES];          // per-slice weights of the current draw
    Partial part[MAXSLICES];      // per-slice partials of an on-demand row
    double red_d[NWARP];
    float red_f[NWARP];
    int32_t red_i[NWARP];
    int32_t y;
    int32_t found;
    uint32_t flags;
    int32_t near;
    int32_t exact;
    double sel_before, sel_after;
    int32_t sel_slice;
    int32_t ex_job, ex_ok, ex_go, ex_pick, ex_phase, ex_chunk;   // exact-draw job board scratch
    float zpre[MAXL][MAXC];       // z_l[b, i, x_i]: the draft token's logit in every row i < K
    float ua[MAXL][MAXC], ue[MAXL][MAXC];   // the request's acceptance / emission uniforms
    int32_t ftok, fclear;         // fast-path draw: crossing token, decided outside the margins
    const double* exptab;         // exp of every bf16 value (float64), or NULL
};
constexpr size_t TAIL_DYN_MAX = 96 * 1024;   // prefetched partials + slice residuals

template <typename Tin>
__device__ __forceinline__ const Tin* row_ptr(const TailParams& p, int l, int64_t b, int64_t i) {
    return reinterpret_cast<const Tin*>(p.lv.ptr[l]) + b * p.lv.bs[l] + i * p.lv.ld[l];
}

__device__ __forceinline__ double block_sum_d(double v, TailShared& sh) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    v = warp_sum_d(v);
    __syncthreads();
    if (lane == 0) sh.red_d[warp] = v;
    __syncthreads();
    double t = 0.0;
#pragma unroll
    for (int w = 0; w < NWARP; ++w) t += sh.red_d[w];
    return t;
}
__device__ __forceinline__ int block_min_i(int v, TailShared& sh) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    v = warp_min_i(v);
    __syncthreads();
    if (lane == 0) sh.red_i[warp] = v;
    __syncthreads();
    int t = 0x7fffffff;
#pragma unroll
    for (int w = 0; w < NWARP; ++w) t = min(t, sh.red_i[w]);
    return t;
}
__device__ __forceinline__ float block_max_f(float v, TailShared& sh) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    v = warp_max(v);
    __syncthreads();
    if (lane == 0) sh.red_f[warp] = v;
    __syncthreads();
    float t = -INFINITY;
#pragma unroll
    for (int w = 0; w < NWARP; ++w) t = fmaxf(t, sh.red_f[w]);
    return t;
}

// Temperature (logits processor): the distributions are softmax(z / T).  The tail keeps
// logits and maxima in raw units and applies sc = 1 / T inside every exponent, (z - M) sc, in
// float64 where the decision depends on it; a normaliser `lse` is in scaled units (M sc + log S).
__shared__ float s_sc;               // 1 / T for this launch (set by thread 0 at kernel start)

// Load this thread's ET elements of slice s of a row (same mapping as the core),
// clamped; out-of-row entries are NEG_CLAMP.
template <typename Tin>
__device__ __forceinline__ void load_slice(const Tin* row, int64_t V, int s, int vse, float* x) {
    constexpr int VEC = Elem<Tin>::VEC;
    constexpr int NV = ET / VEC;
    const int64_t base = (int64_t)s * vse;
    V = min(V, base + vse);           // the slice ends at the next slice's start
#pragma unroll
    for (int jv = 0; jv < NV; ++jv) {
        const int64_t e0 = base + (jv * T + threadIdx.x) * VEC;
        if (e0 + VEC <= V) {
            uint4 v = __ldg(reinterpret_cast<const uint4*>(row + e0));
            unpack_clamped<Tin>(v, &x[jv * VEC]);
        } else {
#pragma unroll
            for (int k = 0; k < VEC; ++k)
                x[jv * VEC + k] = (e0 + k < V) ? clamp1(Elem<Tin>::load1(row + e0 + k)) : NEG_CLAMP;
        }
    }
}

// One vector (VEC entries) of a row at entry e (a multiple of VEC), clamped; entries >= Vend
// are NEG_CLAMP.
template <typename Tin>
__device__ __forceinline__ void load_vec(const Tin* row, int64_t e, int64_t Vend, float* x) {
    constexpr int VEC = Elem<Tin>::VEC;
    if (e + VEC <= Vend) {
        unpack_clamped<Tin>(__ldg(reinterpret_cast<const uint4*>(row + e)), x);
    } else {
#pragma unroll
        for (int k = 0; k < VEC; ++k) x[k] = (e + k < Vend) ? clamp1(Elem<Tin>::load1(row + e + k)) : NEG_CLAMP;
    }
}

// Row statistics of an arbitrary row (bonus rows at positions >= K): per-slice partials into
// sh.part[] (one warp per slice, online max / sum with float64 accumulation, no block
// barriers inside), combined RowStat returned to every thread.
// Fast per-slice partial of a bf16 row for one warp: pass 1 the slice maximum (bf16x2 max
// tree, redux), pass 2 (L1-resident re-read) sum 2^((z - m) log2 e) with the mixed-precision
// add.f32.bf16, packed fp32 per vector and float64 across vectors.  Returns false (the caller
// takes the generic path) when the maximum is not finite.  Argmax only when `want_am`.
__device__ bool slice_partial_bf16(const __nv_bfloat16* row, int64_t s0, int64_t s1, bool want_am, Partial* out) {
    const int lane = threadIdx.x & 31;
    constexpr int VEC = 8, U = 8;   // vectors in flight per lane
    uint32_t mx = 0xFF80FF80u;   // -inf pair
    for (int64_t e0 = s0 + (int64_t)lane * VEC; e0 < s1; e0 += U * 32 * VEC) {
        uint4 v[U];
#pragma unroll
        for (int uu = 0; uu < U; ++uu) {
            const int64_t e = e0 + (int64_t)uu * 32 * VEC;
            v[uu] = e + VEC <= s1 ? __ldg(reinterpret_cast<const uint4*>(row + e)) : make_uint4(0xFF80FF80u, 0xFF80FF80u, 0xFF80FF80u, 0xFF80FF80u);
            if (e < s1 && e + VEC > s1) {     // straddling vector: element-wise, -inf past the end
                __nv_bfloat16 xs[VEC];
#pragma unroll
                for (int k = 0; k < VEC; ++k) xs[k] = e + k < s1 ? row[e + k] : __float2bfloat16(-INFINITY);
                v[uu] = *reinterpret_cast<const uint4*>(xs);
            }
        }
#pragma unroll
        for (int uu = 0; uu < U; ++uu)
            mx = max_nan_bf16x2(mx, max_nan_bf16x2(max_nan_bf16x2(v[uu].x, v[uu].y), max_nan_bf16x2(v[uu].z, v[uu].w)));
    }
    float m = fmaxf(bf16lo(mx), bf16hi(mx));
    if (isnan(bf16lo(mx)) || isnan(bf16hi(mx))) m = NAN;
    m = warp_max(m);
    m = __shfl_sync(0xffffffffu, m, 0);
    if (!(m > NEG_MASKED) || !(m < INFINITY)) return false;
    const float nm = -m;
    const float2 l2e = make_float2(LOG2E * s_sc, LOG2E * s_sc);   // (z - m) / T
    double S = 0.0;
    int am = 0x7fffffff;
    for (int64_t e0 = s0 + (int64_t)lane * VEC; e0 < s1; e0 += U * 32 * VEC) {
        uint4 v[U];
#pragma unroll
        for (int uu = 0; uu < U; ++uu) {
            const int64_t e = e0 + (int64_t)uu * 32 * VEC;
            v[uu] = e + VEC <= s1 ? __ldg(reinterpret_cast<const uint4*>(row + e)) : make_uint4(0xFF80FF80u, 0xFF80FF80u, 0xFF80FF80u, 0xFF80FF80u);
            if (e < s1 && e + VEC > s1) {
                __nv_bfloat16 xs[VEC];
#pragma unroll
                for (int k = 0; k < VEC; ++k) xs[k] = e + k < s1 ? row[e + k] : __float2bfloat16(-INFINITY);
                v[uu] = *reinterpret_cast<const uint4*>(xs);
            }
        }
        float2 acc = make_float2(0.f, 0.f);
#pragma unroll
        for (int uu = 0; uu < U; ++uu) {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const uint32_t w = k == 0 ? v[uu].x : k == 1 ? v[uu].y : k == 2 ? v[uu].z : v[uu].w;
                float y0, y1;
                asm("{ .reg .b16 lo, hi; mov.b32 {lo, hi}, %2; add.rn.f32.bf16 %0, lo, %3; add.rn.f32.bf16 %1, hi, %3; }"
                    : "=f"(y0), "=f"(y1) : "r"(w), "f"(nm));
                const float2 t = __fmul2_rn(make_float2(y0, y1), l2e);
                acc = __fadd2_rn(acc, make_float2(ex2f(t.x), ex2f(t.y)));
                if (want_am) {
                    const int64_t e = e0 + (int64_t)uu * 32 * VEC + 2 * k;
                    if (y0 == 0.f && am == 0x7fffffff) am = (int)e;
                    if (y1 == 0.f && am == 0x7fffffff) am = (int)(e + 1);
                }
            }
        }
        S += (double)(acc.x + acc.y);
    }
    S = warp_sum_d(S);
    if (want_am) am = warp_min_i(am);
    out->m = m;
    out->amax = am;
    out->S = S;
    out->Kl = 0.0;
    return true;
}

// Every 128-byte line of a row requested into L2 by the whole CTA (no registers held).
template <typename Tin>
__device__ __forceinline__ void prefetch_row_l2(const Tin* row, int64_t V) {
    const char* b0 = reinterpret_cast<const char*>(row);
    const int64_t nb = V * (int64_t)sizeof(Tin);
    for (int64_t o = (int64_t)threadIdx.x * 128; o < nb; o += (int64_t)blockDim.x * 128)
        asm volatile("prefetch.global.L2 [%0];" ::"l"(b0 + o));
}

template <typename Tin>
__device__ RowStat row_stats(const Tin* row, int64_t V, int C, int vse, TailShared& sh, bool want_am = true) {
    constexpr int VEC = Elem<Tin>::VEC;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    prefetch_row_l2(row, V);    // the slices below then stream from L2, not one HBM trip per 4 vectors
    for (int s = warp; s < C; s += NWARP) {
        if (sizeof(Tin) == 2) {
            Partial pr;
            const int64_t s0 = (int64_t)s * vse, s1 = min(V, s0 + vse);
            if (slice_partial_bf16(reinterpret_cast<const __nv_bfloat16*>(row), s0, s1, want_am, &pr)) {
                if (lane == 0) sh.part[s] = pr;
                continue;
            }
        }
        const int64_t s0 = (int64_t)s * vse, s1 = min(V, s0 + vse);
        float m = -INFINITY;
        double S = 0.0;
        int am = 0x7fffffff;
        constexpr int U = 4;    // vectors in flight per lane
        for (int64_t e0 = s0 + (int64_t)lane * VEC; e0 < s1; e0 += U * 32 * VEC) {
            float x[U][VEC];
#pragma unroll
            for (int uu = 0; uu < U; ++uu) load_vec<Tin>(row, e0 + (int64_t)uu * 32 * VEC, s1, x[uu]);
#pragma unroll
            for (int uu = 0; uu < U; ++uu) {
                const int64_t e = e0 + (int64_t)uu * 32 * VEC;
                float mv = x[uu][0];
#pragma unroll
                for (int k = 1; k < VEC; ++k) mv = fmaxf(mv, x[uu][k]);
                if (mv > m) {      // new running maximum: rescale (first index of the maximum kept)
                    S *= dexp_neg(((double)m - (double)mv) * (double)s_sc);
                    m = mv;
                    am = 0x7fffffff;
                }
                float sv = 0.f;
#pragma unroll
                for (int k = 0; k < VEC; ++k) sv += ex2f((x[uu][k] - m) * (LOG2E * s_sc));
                S += (double)sv;
#pragma unroll
                for (int k = 0; k < VEC; ++k)
                    if (x[uu][k] == m && am == 0x7fffffff && e + k < s1) am = (int)(e + k);
            }
        }
        // combine the lanes (fixed order)
        const float ms = warp_max(m);
        double f = dexp_neg(((double)m - (double)ms) * (double)s_sc);
        if (!(m > NEG_MASKED)) f = (ms > NEG_MASKED) ? 0.0 : 1.0;
        double Ss = warp_sum_d(S * f);
        const int a = warp_min_i(m == ms ? am : 0x7fffffff);
        if (lane == 0) {
            Partial pr;
            pr.m = ms; pr.amax = a; pr.S = Ss; pr.Kl = 0.0;
            sh.part[s] = pr;
        }
    }
    __syncthreads();
    // combine (same arithmetic as combine_row, from shared memory)
    __shared__ RowStat res;
    if (warp == 0) {
        float m = -INFINITY;
        for (int s = lane; s < C; s += 32) m = fmaxf(m, sh.part[s].m);
        m = warp_max(m);
        double S = 0.0;
        int am = 0x7fffffff;
        bool bad = false;
        for (int s = lane; s < C; s += 32) {
            S += sh.part[s].S * dexp_neg(((double)sh.part[s].m - (double)m) * (double)s_sc);
            if (sh.part[s].m == m) am = min(am, sh.part[s].amax);
            if (isnan(sh.part[s].m) || isnan(sh.part[s].S)) bad = true;
        }
        S = warp_sum_d(S);
        am = warp_min_i(am);
        bad = __any_sync(0xffffffffu, bad);
        if (lane == 0) {
            RowStat r;
            r.M = m; r.S = S; r.lse = (double)m * (double)s_sc + log(S);
            r.amax = am == 0x7fffffff ? 0 : am;
            r.bad = (bad || !(m > NEG_MASKED) || !isfinite(S) || !(m < INFINITY)) ? 1 : 0;
            res = r;
        }
    }
    __syncthreads();
    RowStat r = res;
    __syncthreads();
    return r;
}

// Per-slice residual mass R_s = sum max(p - q, 0) of an arbitrary row pair into sh.w[]
// (one warp per slice; fp32 per vector, float64 across vectors and lanes).
template <typename Tin>
__device__ void pair_resid(const Tin* ra, const Tin* rb, const RowStat& A, const RowStat& Bq,
                           int64_t V, int C, int vse, TailShared& sh) {
    constexpr int VEC = Elem<Tin>::VEC;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const double rho = Bq.S > 0 ? A.S / Bq.S : 0.0;
    const float rh = (float)rho, rl = (float)(rho - (double)rh);
    const float Ma = (float)A.M, Mb = (float)Bq.M;
    for (int s = warp; s < C; s += NWARP) {
        const int64_t s0 = (int64_t)s * vse, s1 = min(V, s0 + vse);
        double acc = 0.0;
        constexpr int U = 4;    // vector pairs in flight per lane
        for (int64_t e0 = s0 + (int64_t)lane * VEC; e0 < s1; e0 += U * 32 * VEC) {
            float xa[U][VEC], xb[U][VEC];
#pragma unroll
            for (int uu = 0; uu < U; ++uu) {
                load_vec<Tin>(ra, e0 + (int64_t)uu * 32 * VEC, s1, xa[uu]);
                load_vec<Tin>(rb, e0 + (int64_t)uu * 32 * VEC, s1, xb[uu]);
            }
#pragma unroll
            for (int uu = 0; uu < U; ++uu) {
                float av = 0.f;
#pragma unroll
                for (int k = 0; k < VEC; ++k) {
                    const float ea = ex2f((xa[uu][k] - Ma) * (LOG2E * s_sc));
                    const float eb = ex2f((xb[uu][k] - Mb) * (LOG2E * s_sc));
                    float t = fmaf(-eb, rh, ea);
                    t = fmaf(-eb, rl, t);
                    av += fmaxf(t, 0.f);
                }
                acc += (double)av;
            }
        }
        acc = warp_sum_d(acc);
        if (lane == 0) sh.w[s] = acc / A.S;
    }
    __syncthreads();
}

// The 16 contiguous entries [e0, e0 + 16) of a row, clamped; entries >= Vend are NEG_CLAMP.
// e0 is a multiple of 16 entries, so whole vectors are 16-byte aligned (rows are, by the ABI).
template <typename Tin>
__device__ __forceinline__ void load16(const Tin* row, int64_t e0, int64_t Vend, float* x) {
    constexpr int VEC = Elem<Tin>::VEC;
    if (e0 + ET <= Vend) {
        uint4 v[ET / VEC];
#pragma unroll
        for (int jv = 0; jv < ET / VEC; ++jv) v[jv] = __ldg(reinterpret_cast<const uint4*>(row + e0) + jv);
#pragma unroll
        for (int jv = 0; jv < ET / VEC; ++jv) unpack_clamped<Tin>(v[jv], &x[jv * VEC]);
    } else {
#pragma unroll
        for (int k = 0; k < ET; ++k) x[k] = (e0 + k < Vend) ? clamp1(Elem<Tin>::load1(row + e0 + k)) : NEG_CLAMP;
    }
}

// Weight of vocabulary entry z (and z' for the residual) in float64.
// exp(z - S) in float64.  For bf16 logits (every z is a bf16 value) it is tab[bits(z)] * e^-S
// with tab[h] = exp(bf16 h) (msd_api: exp_table), one lookup and one multiply instead of a
// float64 exp; outside the table's range (|z| >= 700, |S| >= 700) the FMA-pipe dexp_neg.
#ifndef MSD_EXACT_U
#define MSD_EXACT_U 1
#endif
// out of line: the rare fallback must not be unrolled into the table loops (inlined, its copies
// made the exact draw instruction-cache bound: 'no_inst' stalls at the table gathers)
__device__ __noinline__ double dexp_neg_cold(double x) { return dexp_neg(x); }

// exp(z sc - S) for a raw logit z and a scaled offset S (sc = 1 / T; the bf16 table only when
// sc = 1: it holds exp of raw bf16 values)
struct ExpShift {
    const double* tab;   // NULL: no table (f32 logits, or a temperature)
    double S, eS, sc;
    __device__ void init(const double* t, double s_) {
        tab = (t && fabs(s_) < 700.0 && s_sc == 1.f) ? t : nullptr;
        S = s_;
        sc = (double)s_sc;
        eS = tab ? exp(-s_) : 0.0;
    }
    __device__ __forceinline__ double operator()(float z) const {
        if (tab) {
            const double t = __ldg(tab + (__float_as_uint(z) >> 16));
            if (t == t) return t * eS;      // NaN entry: outside the table's range
        }
        return dexp_neg_cold((double)z * sc - S);     // z sc <= max sc <= S: argument <= 0
    }
};

// Table path of ExpShift for a batch of N values: every gather issued before any is used (the
// exact draw is bound by table-gather latency otherwise); same value as ExpShift::operator().
template <int N>
__device__ __forceinline__ void exp_shift_batch(const ExpShift& es, const float* z, double* out) {
#pragma unroll
    for (int k = 0; k < N; ++k) out[k] = __ldg(es.tab + (__float_as_uint(z[k]) >> 16));
#pragma unroll
    for (int k = 0; k < N; ++k) out[k] = (out[k] == out[k]) ? out[k] * es.eS : dexp_neg_cold((double)z[k] * es.sc - es.S);
}

__device__ __forceinline__ double wt(bool resid, float za, float zb, double A, double B) {
    if (!(za > NEG_MASKED)) return 0.0;
    const double sc = (double)s_sc;
    const double pa = dexp_neg((double)za * sc - A);     // z sc <= max sc <= lse: argument <= 0
    if (!resid) return pa;
    const double qb = (zb > NEG_MASKED) ? dexp_neg((double)zb * sc - B) : 0.0;
    const double r = pa - qb;
    return r > 0.0 ? r : 0.0;
}
__device__ __forceinline__ double wt(bool resid, float za, float zb, const ExpShift& ea, const ExpShift& eb) {
    if (!(za > NEG_MASKED)) return 0.0;
    const double pa = ea(za);
    if (!resid) return pa;
    const double qb = (zb > NEG_MASKED) ? eb(zb) : 0.0;
    const double r = pa - qb;
    return r > 0.0 ? r : 0.0;
}

// Inverse-CDF search inside slice s with weights wt(), given the float64 mass of
// all earlier slices (`before`) and the target u*Z.  Thread t scans the 16
// contiguous entries [t*16, t*16+16) of the slice.  Returns the token or -1.
// Block-wide inverse-CDF step over the threads' 16 weights each (fixed order): the first entry
// whose float64 prefix exceeds `target`; the crossing thread gets its prefix bounds.
template <typename WF>
__device__ __forceinline__ int scan_find(WF w, int64_t e0, double before, double target, TailShared& sh,
                                         int* found, double* cprev_f, double* c_f) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double loc = 0.0;
#pragma unroll
    for (int k = 0; k < ET; ++k) loc += (double)w(k);
    double incl = loc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const double t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
    }
    __syncthreads();
    if (lane == 31) sh.red_d[warp] = incl;
    __syncthreads();
    double woff = 0.0;
    for (int wi = 0; wi < warp; ++wi) woff += sh.red_d[wi];
    double c = before + woff + (incl - loc);
    *found = 0x7fffffff;
#pragma unroll
    for (int k = 0; k < ET; ++k) {
        const double cp = c;
        const double wk = (double)w(k);
        c += wk;
        if (*found == 0x7fffffff && wk > 0.0 && c > target) {
            *found = (int)(e0 + k);
            *cprev_f = cp;
            *c_f = c;
        }
    }
    return block_min_i(*found, sh);
}

// Fast-pass inverse-CDF step in float32, relative to the slice: thread t holds the ET weights of
// entries [e0, e0 + ET); `t` is the slice-local target (target - before) and `margin` the
// decision margin.  Every thread's exclusive / inclusive prefix is formed with the same
// operations as its neighbours' (warp scan, then the preceding warps' totals summed in a fixed
// order), so exactly one thread holds a crossing; it scans its weights and records the token and
// whether the crossing lies farther than `margin` from both of its boundaries.  Two barriers.
// The float32 accumulation error (< 30 roundings of the slice mass, ~2e-6 Z) is far inside the
// margin (2e-5 Z).  Returns the token or 0x7fffffff (none: the caller takes the float64 pass).
__device__ __forceinline__ int scan_find_f32(const float* w, int64_t e0, float t, float margin, TailShared& sh,
                                             bool* clear) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    float q[ET / 2];
#pragma unroll
    for (int k = 0; k < ET / 2; ++k) q[k] = w[2 * k] + w[2 * k + 1];
#pragma unroll
    for (int h = ET / 4; h > 0; h >>= 1)
#pragma unroll
        for (int k = 0; k < h; ++k) q[k] = q[k] + q[k + h];
    const float loc = q[0];
    float incl = loc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const float x = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += x;
    }
    float excl = __shfl_up_sync(0xffffffffu, incl, 1);
    if (lane == 0) excl = 0.f;
    if (threadIdx.x == 0) { sh.ftok = 0x7fffffff; sh.fclear = 0; }
    if (lane == 31) sh.red_f[warp] = incl;
    __syncthreads();
    float woff = 0.f;
#pragma unroll
    for (int wi = 0; wi < NWARP - 1; ++wi)
        if (wi < warp) woff += sh.red_f[wi];
    const float lo = woff + excl, hi = woff + incl;
    if (loc > 0.f && lo <= t && t < hi) {
        float c = lo, cp = lo;
        int kk = -1;
#pragma unroll
        for (int k = 0; k < ET; ++k) {
            const float c0 = c;
            c += w[k];
            if (kk < 0 && w[k] > 0.f && c > t) { kk = k; cp = c0; }
        }
        if (kk >= 0) {
            sh.ftok = (int)(e0 + kk);
            sh.fclear = (t - cp > margin && (c - t) > margin) ? 1 : 0;
        }
    }
    __syncthreads();
    *clear = sh.fclear != 0;
    return sh.ftok;
}

// Inverse-CDF search inside slice s with weights wt(), given the float64 mass of all earlier
// slices (`before`) and the target u*Z.  Thread t scans the 16 contiguous entries
// [t*16, t*16+16) of the slice.  Returns the token or -1.
// Fast pass: fp32 weights (MUFU), float64 prefix; their total error is far below
// the draw margins (DRAW_MARGIN_REL * Z + DRAW_MARGIN_ABS), so the crossing token
// is the exact one unless the target lies within that margin of a boundary -- then the exact
// pass (float64 weights, the oracle's arithmetic, R5) decides.
template <typename Tin>
__device__ int32_t scan_slice(bool resid, const Tin* ra, const Tin* rb, double A, double B,
                              int64_t V, int s, int vse, double before, double target, double Z, double u,
                              TailShared& sh, bool* tie, bool exact_only = false) {
    const int64_t e0 = (int64_t)s * vse + threadIdx.x * ET;
    V = min(V, (int64_t)(s + 1) * vse);
    if (threadIdx.x == 0) { sh.near = 0; sh.found = 0; }
#ifdef MSD_PROF
    long long q0 = clock64();
#endif
    float xa[ET], xb[ET];
    load16<Tin>(ra, e0, V, xa);
    if (resid) load16<Tin>(rb, e0, V, xb);
    int found;
    double cprev_f = 0.0, c_f = 0.0;
    if (!exact_only) {
        const float Ah = (float)A, Al = (float)(A - (double)Ah);
        const float Bh = (float)B, Bl = (float)(B - (double)Bh);
        float wf[ET];
#pragma unroll
        for (int k = 0; k < ET; ++k) {
            float wk = 0.f;
            if (xa[k] > NEG_MASKED) {
                wk = ex2f(((xa[k] * s_sc - Ah) - Al) * LOG2E);     // fast path: fp32 z / T (margins)
                if (resid) {
                    const float qk = xb[k] > NEG_MASKED ? ex2f(((xb[k] * s_sc - Bh) - Bl) * LOG2E) : 0.f;
                    wk = fmaxf(wk - qk, 0.f);
                }
            }
            wf[k] = wk;
        }
#ifdef MSD_PROF
        if (threadIdx.x == 0) { const long long q = clock64(); atomicAdd(&g_tail_prof[9], (unsigned long long)(q - q0)); q0 = q; }
#endif
        // c - t and t - cp are slice-local float32 distances; the crossing token's own boundaries
        bool clear;
        const int best = scan_find_f32(wf, e0, (float)(target - before), (float)(DRAW_MARGIN_REL * Z + DRAW_MARGIN_ABS),
                                       sh, &clear);
#ifdef MSD_PROF
        if (threadIdx.x == 0) {
            const long long q = clock64();
            atomicAdd(&g_tail_prof[10], (unsigned long long)(q - q0));
            atomicAdd(&g_tail_prof[15], 1ull);
            if (!clear) atomicAdd(&g_tail_prof[14], 1ull);
        }
#endif
        if (best != 0x7fffffff && clear) {
            *tie = false;
            return best;
        }
        // within the margin of a token boundary: the float64 rescan below decides
    }
    ExpShift ea, eb;
    ea.init(sizeof(Tin) == 2 ? sh.exptab : nullptr, A);
    eb.init(sizeof(Tin) == 2 ? sh.exptab : nullptr, B);
    int best;
    if (ea.tab && (!resid || eb.tab)) {
        // table path: every gather of the thread's ET weights issued before any is used (one L2
        // round trip), the float64 weights formed once (the two scans below reuse them)
        double wd[ET];
        exp_shift_batch<ET>(ea, xa, wd);
        if (resid) {
            double tb[ET];
            exp_shift_batch<ET>(eb, xb, tb);
#pragma unroll
            for (int k = 0; k < ET; ++k) {
                const double r = (xa[k] > NEG_MASKED ? wd[k] : 0.0) - (xb[k] > NEG_MASKED ? tb[k] : 0.0);
                wd[k] = xa[k] > NEG_MASKED && r > 0.0 ? r : 0.0;
            }
        } else {
#pragma unroll
            for (int k = 0; k < ET; ++k) wd[k] = xa[k] > NEG_MASKED ? wd[k] : 0.0;
        }
        best = scan_find([&](int k) { return wd[k]; }, e0, before, target, sh, &found, &cprev_f, &c_f);
    } else {
        // (weights recomputed on demand: no table -- f32 logits or a temperature)
        best = scan_find([&](int k) { return wt(resid, xa[k], resid ? xb[k] : NEG_CLAMP, ea, eb); }, e0,
                         before, target, sh, &found, &cprev_f, &c_f);
    }
    if (best != 0x7fffffff && found == best) {
        *tie = fabs(u - cprev_f / Z) < TIE_EPS || fabs(u - c_f / Z) < TIE_EPS;
        sh.near = *tie ? 1 : 0;
    }
    __syncthreads();
    *tie = sh.near != 0;
    return best == 0x7fffffff ? -1 : best;
}

// Last entry with positive weight in slice s (clamp rule, reading R5).
template <typename Tin>
__device__ int32_t last_positive(bool resid, const Tin* ra, const Tin* rb, double A, double B,
                                 int64_t V, int s, int vse, TailShared& sh) {
    int best = -1;
    for (int64_t v = (int64_t)s * vse + threadIdx.x; v < min(V, (int64_t)(s + 1) * vse); v += T) {
        const float za = clamp1(Elem<Tin>::load1(ra + v));
        const float zb = resid ? clamp1(Elem<Tin>::load1(rb + v)) : NEG_CLAMP;
        if (wt(resid, za, zb, A, B) > 0.0) best = max(best, (int)v);
    }
    return -block_min_i(-best, sh);
}

// Draw with given per-slice weights sh.w[0..C): pick the slice by the float64
// prefix, rescan it.  Returns token or -1 (inconsistent -> caller goes exact).
template <typename Tin>
__device__ int32_t draw_slices(bool resid, const Tin* ra, const Tin* rb, double A, double B,
                               int64_t V, int C, int vse, double Z, double u, TailShared& sh, bool* tie,
                               bool exact = false) {
    if (threadIdx.x < 32) {
        // first slice whose inclusive float64 prefix exceeds u Z (warp scan, 32 slices a step)
        const int lane = threadIdx.x;
        const double target = u * Z;
        double base = 0.0;
        int sel = -1, lastpos = -1;
        double before = 0.0, after = 0.0;
        for (int s0 = 0; s0 < C; s0 += 32) {
            const double ws = (s0 + lane < C) ? sh.w[s0 + lane] : 0.0;
            double incl = ws;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const double t = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += t;
            }
            const unsigned hit = __ballot_sync(0xffffffffu, ws > 0.0 && base + incl > target);
            const unsigned pos = __ballot_sync(0xffffffffu, ws > 0.0);
            if (pos) lastpos = s0 + 31 - __clz((int)pos);
            if (sel < 0 && hit) {
                const int f = __ffs((int)hit) - 1;
                sel = s0 + f;
                before = base + __shfl_sync(0xffffffffu, incl - ws, f);
                after = base + __shfl_sync(0xffffffffu, incl, f);
            }
            base += __shfl_sync(0xffffffffu, incl, 31);
        }
        if (sel < 0) { sel = -1 - (lastpos < 0 ? 0 : lastpos); before = base; }
        if (lane == 0) {
            sh.sel_slice = sel;
            sh.sel_before = before;
            sh.sel_after = after;
        }
    }
    __syncthreads();
    const int sel = sh.sel_slice;
    const double before = sh.sel_before, after = sh.sel_after;
    __syncthreads();
    const double smarg = fmax(SLICE_MARGIN_REL * Z, SLICE_MARGIN_Z);
    if (!exact && sel >= 0 && (u * Z - before < smarg || after - u * Z < smarg))
        return -1;      // next to a slice boundary: the caller takes the exact path
    if (sel < 0) {  // u*Z beyond the total (rounding): clamp to the last positive entry
        *tie = true;
        return last_positive<Tin>(resid, ra, rb, A, B, V, -1 - sel, vse, sh);
    }
    return scan_slice<Tin>(resid, ra, rb, A, B, V, sel, vse, before, u * Z, Z, u, sh, tie, exact);
}

// ------------------------------------------------------------------ exact draws
// Exact float64 draw over the whole row (pair): exact normalisers, exact slice masses, exact
// scan.  Residual mass < 1e-12 -> draw from p.  The two full-row passes are cut into
// chunks (EXJ_NCH normaliser chunks, then one chunk per slice), each summed by one whole CTA
// in a fixed order and combined in chunk order, so the result does not depend on which CTA
// computed a chunk: the requesting CTA posts the job on the board and CTAs that finished
// their own request help (exact_help); with no helper (or a full board) it does all chunks.

// float64 sum of exp(z - M) over [e0, e1) of one row (and of the second row) -- whole CTA,
// result valid in every thread (fixed order: strided per thread, then block_sum_d)
template <typename Tin>
__device__ void exact_norm_chunk(const Tin* ra, const Tin* rb, bool resid, int64_t e0, int64_t e1, double Ma,
                                 double Mb, const double* tab, TailShared& sh, double* sa_out, double* sb_out) {
    constexpr int VEC = Elem<Tin>::VEC;
    ExpShift eMa, eMb;
    eMa.init(tab, Ma * (double)s_sc);     // raw maxima -> scaled offsets
    eMb.init(tab, Mb * (double)s_sc);
    double sa = 0.0, sb = 0.0;
#pragma unroll 1
    for (int64_t e = e0 + (int64_t)threadIdx.x * VEC; e < e1; e += (int64_t)T * VEC) {
        float xa[VEC], xb[VEC];
        load_vec<Tin>(ra, e, e1, xa);
        if (resid) load_vec<Tin>(rb, e, e1, xb);
        if (eMa.tab && (!resid || eMb.tab)) {
            double ga[VEC], gb[VEC];
            exp_shift_batch<VEC>(eMa, xa, ga);
            if (resid) exp_shift_batch<VEC>(eMb, xb, gb);
#pragma unroll
            for (int k = 0; k < VEC; ++k) {
                if (xa[k] > NEG_MASKED) sa += ga[k];
                if (resid && xb[k] > NEG_MASKED) sb += gb[k];
            }
        } else {
#pragma unroll
            for (int k = 0; k < VEC; ++k) {
                if (xa[k] > NEG_MASKED) sa += eMa(xa[k]);
                if (resid && xb[k] > NEG_MASKED) sb += eMb(xb[k]);
            }
        }
    }
    *sa_out = block_sum_d(sa, sh);
    *sb_out = resid ? block_sum_d(sb, sh) : 0.0;
}

// float64 mass of slice s of the (residual) weights with exact normalisers A, B -- whole CTA
template <typename Tin>
__device__ double exact_slice_mass(const Tin* ra, const Tin* rb, bool resid, int64_t V, int s, int vse, double A,
                                   double B, const double* tab, TailShared& sh) {
    constexpr int VEC = Elem<Tin>::VEC;
    ExpShift eA, eB;
    eA.init(tab, A);
    eB.init(tab, B);
    const int64_t s0 = (int64_t)s * vse, s1 = min(V, s0 + vse);
    double acc = 0.0;
#pragma unroll 1
    for (int64_t e = s0 + (int64_t)threadIdx.x * VEC; e < s1; e += (int64_t)T * VEC) {
        float xa[VEC], xb[VEC];
        load_vec<Tin>(ra, e, s1, xa);
        if (resid) load_vec<Tin>(rb, e, s1, xb);
        if (eA.tab && (!resid || eB.tab)) {
            double ga[VEC], gb[VEC];
            exp_shift_batch<VEC>(eA, xa, ga);
            if (resid) exp_shift_batch<VEC>(eB, xb, gb);
#pragma unroll
            for (int k = 0; k < VEC; ++k) {    // = wt(resid, za, zb, eA, eB)
                double w = 0.0;
                if (xa[k] > NEG_MASKED) {
                    w = ga[k];
                    if (resid) {
                        const double r = w - ((xb[k] > NEG_MASKED) ? gb[k] : 0.0);
                        w = r > 0.0 ? r : 0.0;
                    }
                }
                acc += w;
            }
        } else {
#pragma unroll
            for (int k = 0; k < VEC; ++k) acc += wt(resid, xa[k], resid ? xb[k] : NEG_CLAMP, eA, eB);
        }
    }
    return block_sum_d(acc, sh);
}

__device__ __forceinline__ uint32_t ld_acq(const uint32_t* p) { return ld_acquire_u32(p); }

// Process chunks of job j until none is left in its current phase (whole CTA).  Returns after
// the phase's chunks are all claimed.  Used by the requester and by helpers.
template <typename Tin>
__device__ __noinline__ void exact_work(JobBoard* bd, int j, uint32_t phase, TailShared& sh) {
    ExactJob& J = bd->job[j];
    // the job was written by another CTA during this kernel: L1-bypassing loads (ld.cg)
    const Tin* ra = reinterpret_cast<const Tin*>(__ldcg(reinterpret_cast<const unsigned long long*>(&J.ra)));
    const Tin* rb = reinterpret_cast<const Tin*>(__ldcg(reinterpret_cast<const unsigned long long*>(&J.rb)));
    const double* tab = sizeof(Tin) == 2 ? sh.exptab : nullptr;
    const bool resid = __ldcg(&J.resid) != 0;
    const int Cj = __ldcg(&J.C), vse = __ldcg(&J.vse), chunk = __ldcg(&J.chunk);
    const int64_t Vj = __ldcg(&J.V);
    const double Ma = __ldcg(&J.Ma), Mb = __ldcg(&J.Mb);
    const double Aj = phase == 2 ? __ldcg(&J.A) : 0.0, Bj = phase == 2 ? __ldcg(&J.B) : 0.0;
    const int nch = phase == 1 ? EXJ_NCH : (Cj + EXJ_SPC - 1) / EXJ_SPC;
    while (true) {
        if (threadIdx.x == 0) sh.ex_chunk = (int)atomicAdd(phase == 1 ? &J.next1 : &J.next2, 1u);
        __syncthreads();
        const int ch = sh.ex_chunk;
        __syncthreads();
        if (ch >= nch) return;
        if (phase == 1) {
            const int64_t e0 = min(Vj, (int64_t)ch * chunk), e1 = min(Vj, e0 + chunk);
            double sa, sb;
            exact_norm_chunk<Tin>(ra, rb, resid, e0, e1, Ma, Mb, tab, sh, &sa, &sb);
            if (threadIdx.x == 0) {
                bd->part1[j][ch][0] = sa;
                bd->part1[j][ch][1] = sb;
                __threadfence();
                atomicAdd(&J.done1, 1u);
            }
        } else {
            for (int s = ch * EXJ_SPC; s < min(Cj, (ch + 1) * EXJ_SPC); ++s) {
                const double m = exact_slice_mass<Tin>(ra, rb, resid, Vj, s, vse, Aj, Bj, tab, sh);
                if (threadIdx.x == 0) bd->part2[j][s] = m;
            }
            if (threadIdx.x == 0) {
                __threadfence();
                atomicAdd(&J.done2, 1u);
            }
        }
    }
}

// wait (thread 0 spins, the CTA then syncs) until *cnt == n; 2 s timeout -> false
__device__ bool exact_wait(const uint32_t* cnt, uint32_t n, TailShared& sh) {
    if (threadIdx.x == 0) {
        const uint64_t t0 = globaltimer();
        int ok = 1;
        while (ld_acq(cnt) < n) {
            if (globaltimer() - t0 > 2000000000ull) { ok = 0; break; }
            __nanosleep(100);
        }
        sh.ex_ok = ok;
    }
    __syncthreads();
    const bool ok = sh.ex_ok != 0;
    __syncthreads();
    return ok;
}

template <typename Tin>
__device__ __noinline__ int32_t draw_exact(bool resid, const Tin* ra, const Tin* rb, const RowStat& Ar,
                              const RowStat& Br, int64_t V, int C, int vse, double u, TailShared& sh,
                              bool* tie, bool* small, JobBoard* bd) {
  constexpr int VEC = Elem<Tin>::VEC;
#ifdef MSD_PROF
  if (threadIdx.x == 0) g_tail_req[blockIdx.x][11] += (unsigned long long)clock64();
#endif
  // both rows into L2 up front (helpers and the slice-mass pass re-read them from L2)
  prefetch_row_l2(ra, V);
  if (resid) prefetch_row_l2(rb, V);
  const double* tab = sizeof(Tin) == 2 ? sh.exptab : nullptr;
  const int64_t chunk = ((V + EXJ_NCH - 1) / EXJ_NCH + VEC - 1) / VEC * VEC;
  // post the job (or keep it local when the board is full: same chunks, computed here)
  if (threadIdx.x == 0) {
      int j = bd ? (int)atomicAdd(&bd->alloc, 1u) : EXJ_MAX;
      sh.ex_job = j < EXJ_MAX ? j : -1;
  }
  __syncthreads();
  const int jid = sh.ex_job;
  __syncthreads();
  double A, B0;
  if (jid >= 0) {
      ExactJob& J = bd->job[jid];
      if (threadIdx.x == 0) {
          J.ra = ra; J.rb = rb; J.Ma = Ar.M; J.Mb = Br.M; J.V = V;
          J.resid = resid ? 1 : 0; J.C = C; J.vse = vse; J.chunk = (int32_t)chunk;
          J.next1 = J.done1 = J.next2 = J.done2 = 0u;
          __threadfence();
          st_release_u32(&J.phase, 1u);
      }
      __syncthreads();
      exact_work<Tin>(bd, jid, 1, sh);
      if (!exact_wait(&J.done1, EXJ_NCH, sh)) return 0;
      double sa = 0.0, sb = 0.0;
      for (int c = 0; c < EXJ_NCH; ++c) { sa += __ldcg(&bd->part1[jid][c][0]); sb += __ldcg(&bd->part1[jid][c][1]); }
      A = Ar.M * (double)s_sc + log(sa);
      B0 = resid ? Br.M * (double)s_sc + log(sb) : 0.0;
      if (threadIdx.x == 0) {
          J.A = A; J.B = B0;
          __threadfence();
          st_release_u32(&J.phase, 2u);
      }
      __syncthreads();
      exact_work<Tin>(bd, jid, 2, sh);
      if (!exact_wait(&J.done2, (uint32_t)((C + EXJ_SPC - 1) / EXJ_SPC), sh)) return 0;
      for (int s = threadIdx.x; s < C; s += T) sh.w[s] = __ldcg(&bd->part2[jid][s]);
      if (threadIdx.x == 0) st_release_u32(&J.phase, 3u);
      __syncthreads();
  } else {
      double sa = 0.0, sb = 0.0;
      for (int c = 0; c < EXJ_NCH; ++c) {
          const int64_t e0 = min(V, (int64_t)c * chunk), e1 = min(V, e0 + chunk);
          double ca, cb;
          exact_norm_chunk<Tin>(ra, rb, resid, e0, e1, Ar.M, Br.M, tab, sh, &ca, &cb);
          sa += ca;
          sb += cb;
      }
      A = Ar.M * (double)s_sc + log(sa);
      B0 = resid ? Br.M * (double)s_sc + log(sb) : 0.0;
      for (int s = 0; s < C; ++s) {
          const double m = exact_slice_mass<Tin>(ra, rb, resid, V, s, vse, A, B0, tab, sh);
          if (threadIdx.x == 0) sh.w[s] = m;
      }
      __syncthreads();
  }
#ifdef MSD_PROF
  if (threadIdx.x == 0) g_tail_req[blockIdx.x][9] += (unsigned long long)clock64();
#endif
  for (int attempt = 0; attempt < 2; ++attempt) {
    const double B = resid ? B0 : 0.0;
    if (attempt == 1) {     // residual vanished: the slice masses of p, computed here
        for (int s = 0; s < C; ++s) {
            const double m = exact_slice_mass<Tin>(ra, rb, false, V, s, vse, A, 0.0, tab, sh);
            if (threadIdx.x == 0) sh.w[s] = m;
        }
        __syncthreads();
    }
#ifdef MSD_PROF
    if (threadIdx.x == 0) g_tail_req[blockIdx.x][10] += (unsigned long long)clock64();
#endif
    const int lane = threadIdx.x & 31;
    double Z = 0.0;
    for (int s = lane; s < C; s += 32) Z += sh.w[s];
    Z = warp_sum_d(Z);
    if (threadIdx.x < 32 && lane == 0) sh.red_d[0] = Z;
    __syncthreads();
    Z = sh.red_d[0];
    __syncthreads();
    if (resid && Z < 1e-12) {   // residual vanished -> draw from p
        *small = true;
        resid = false;
        continue;
    }
    int32_t y = draw_slices<Tin>(resid, ra, rb, A, B, V, C, vse, Z, u, sh, tie, /*exact=*/true);
    return y < 0 ? 0 : y;
  }
  return 0;
}

// Help with posted exact-draw jobs after this CTA's own request is done: claim chunks of any
// job in its normaliser or slice-mass phase; linger only while every request has started
// (so no waiting request is denied this slot) and some request is unfinished.
template <typename Tin>
__device__ __noinline__ void exact_help(JobBoard* bd, int64_t B, TailShared& sh) {
    if (!bd) return;
    const uint64_t t0 = globaltimer();
    while (true) {
        if (threadIdx.x == 0) {
            int pick = -1, ph = 0;
            const uint32_t n = min(ld_acq(&bd->alloc), (uint32_t)EXJ_MAX);
            for (uint32_t j = 0; j < n && pick < 0; ++j) {
                const uint32_t phs = ld_acq(&bd->job[j].phase);
                if (phs == 1u && ld_acq(&bd->job[j].next1) < (uint32_t)EXJ_NCH) { pick = (int)j; ph = 1; }
                else if (phs == 2u && ld_acq(&bd->job[j].next2) < (uint32_t)((__ldcg(&bd->job[j].C) + EXJ_SPC - 1) / EXJ_SPC)) { pick = (int)j; ph = 2; }
            }
            int go = 0;
            if (pick < 0) {
                const bool all_started = ld_acq(&bd->started) >= (uint32_t)B;
                const bool all_done = ld_acq(&bd->finished) >= (uint32_t)B;
                go = (!all_started || all_done || globaltimer() - t0 > 2000000000ull) ? -1 : 0;
                if (go == 0) __nanosleep(1000);   // idle poll: keep the co-resident request's SM quiet
            } else {
                go = 1;
            }
            sh.ex_go = go;
            sh.ex_pick = pick;
            sh.ex_phase = ph;
        }
        __syncthreads();
        const int go = sh.ex_go, pick = sh.ex_pick, ph = sh.ex_phase;
        __syncthreads();
        if (go < 0) return;
        if (go > 0) exact_work<Tin>(bd, pick, (uint32_t)ph, sh);
    }
}

// Block-wide copy of `bytes` (a multiple of 8) from global to shared memory with every load of
// a thread issued before its stores (one memory round trip instead of one per word): 16-byte
// words when both sides allow it, else 8-byte words.
__device__ __forceinline__ void copy_to_smem(void* dst, const void* src, size_t bytes) {
    constexpr int U = 8;
    if ((((uintptr_t)dst | (uintptr_t)src | bytes) & 15) == 0) {
        const uint4* s4 = reinterpret_cast<const uint4*>(src);
        uint4* d4 = reinterpret_cast<uint4*>(dst);
        const size_t n = bytes / 16;
        for (size_t t0 = threadIdx.x; t0 < n; t0 += (size_t)U * T) {
            uint4 v[U];
#pragma unroll
            for (int k = 0; k < U; ++k)
                if (t0 + (size_t)k * T < n) v[k] = s4[t0 + (size_t)k * T];
#pragma unroll
            for (int k = 0; k < U; ++k)
                if (t0 + (size_t)k * T < n) d4[t0 + (size_t)k * T] = v[k];
        }
    } else {
        const unsigned long long* s8 = reinterpret_cast<const unsigned long long*>(src);
        unsigned long long* d8 = reinterpret_cast<unsigned long long*>(dst);
        const size_t n = bytes / 8;
        for (size_t t0 = threadIdx.x; t0 < n; t0 += (size_t)U * T) {
            unsigned long long v[U];
#pragma unroll
            for (int k = 0; k < U; ++k)
                if (t0 + (size_t)k * T < n) v[k] = s8[t0 + (size_t)k * T];
#pragma unroll
            for (int k = 0; k < U; ++k)
                if (t0 + (size_t)k * T < n) d8[t0 + (size_t)k * T] = v[k];
        }
    }
}

template <typename Tin>
#ifndef MSD_TAIL_MINB
#define MSD_TAIL_MINB 2
#endif
__global__ void __launch_bounds__(T, MSD_TAIL_MINB) tail_kernel(TailParams p) {
    __shared__ TailShared sh;
    const int64_t b = blockIdx.x;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int L = p.L, K = p.K, C = p.C;
    const int64_t V = p.V;

    TPROF_DECL
#ifdef MSD_PROF
    if (tid == 0 && b < 4096) g_tail_cta[b][0] = globaltimer();
#endif
    if (tid == 0) {
        if (p.board) atomicAdd(&p.board->started, 1u);
        s_sc = p.inv_temp;
        sh.flags = 0;
        sh.exptab = p.exptab;
        int m1 = p.m0 ? p.m0[b] : K;
        m1 = max(0, min(m1, K));
        sh.m[1] = m1;
    }
    for (int q = tid; q < MAXL * MAXL; q += T) (&sh.extra_ok[0][0])[q] = 0;
    // one round trip for everything the request needs from the core and the draft: its slice
    // partials and residuals into shared memory (when they fit), the draft tokens' logits
    extern __shared__ __align__(16) unsigned char tdyn[];
    const size_t npart = (size_t)K * L * C, nres = (size_t)K * (L - 1) * C;
    const bool pre = p.prefetch != 0;
    const Partial* part_b = p.partials + (size_t)b * npart;
    const double* res_b = p.resid + (size_t)b * nres;
    if (pre) {
        double* rd = reinterpret_cast<double*>(tdyn + npart * sizeof(Partial));
        copy_to_smem(tdyn, part_b, npart * sizeof(Partial));
        copy_to_smem(rd, res_b, nres * sizeof(double));
        part_b = reinterpret_cast<const Partial*>(tdyn);
        res_b = rd;
    }
    for (int t = tid; t < L * K; t += T) {
        const int l = t / K, i = t % K;
        const int32_t x = p.cand0[b * K + i];
        sh.zpre[l][i] = (x >= 0 && x < V) ? clamp1(Elem<Tin>::load1(row_ptr<Tin>(p, l, b, i) + x)) : NEG_CLAMP;
    }
    // the request's uniforms, in the same round trip (acceptance and emission read them later)
    if (!p.greedy) {
        const int W = K + L - 1;
        for (int t = tid; t < (L - 1) * W; t += T) {
            const int l = t / W, i = t % W;
            sh.ua[l][i] = p.u_acc[l * p.ua_l + b * p.ua_b + i];
            sh.ue[l][i] = p.u_emit[l * p.ue_l + b * p.ue_b + i];
        }
    }
    __syncthreads();
    TPROF(12)
    // row normalisers (Eq. 1) and KL numerators of every draft-position row, combined from
    // the core's slice partials in a fixed order (one warp per row)
    for (int r = warp; r < K * L; r += NWARP) {
        const int i = r / L, l = r % L;
        double Kl;
        const Partial* pp = part_b + ((size_t)i * L + l) * C;
        RowStat rs = combine_row(pp, C, &Kl, (double)s_sc);   // KL numerators: sum e (z_l - z_{l-1}) / T
        if (lane == 0) { sh.row[i][l] = rs; sh.kl[i][l] = Kl; }
    }
    __syncthreads();
    TPROF(13)
    if (tid < K) {
        const int i = tid;
        bool bad = false;
        for (int l = 0; l < L; ++l) bad |= sh.row[i][l].bad != 0;
        for (int l = L - 1; l >= 1; --l)
            sh.kl[i][l] = sh.kl[i][l] / sh.row[i][l].S - (sh.row[i][l].lse - sh.row[i][l - 1].lse);
        if (bad) atomicOr(&sh.flags, (uint32_t)MSD_F_NONFINITE);
    }
    __syncthreads();
    for (int i = tid; i < K; i += T) sh.c[1][i] = p.cand0[b * K + i];
    __syncthreads();

    int64_t st_near[MAXL] = {0, 0, 0, 0}, st_exact[MAXL] = {0, 0, 0, 0};

    TPROF(0)
    for (int l = 1; l < L; ++l) {
        const int m = sh.m[l];
        // rows at positions >= K needed by this level's tests (level l and l-1)
        for (int i = K; i < m; ++i) {
            for (int lv = l - 1; lv <= l; ++lv) {
                if (!sh.extra_ok[lv][i - K]) {
                    RowStat r = row_stats<Tin>(row_ptr<Tin>(p, lv, b, i), V, C, p.VSe, sh, p.greedy != 0);
                    if (tid == 0) { sh.extra[lv][i - K] = r; sh.extra_ok[lv][i - K] = 1; }
                    __syncthreads();
                }
            }
        }
        __syncthreads();
        TPROF(1)

        // ---- acceptance tests (warp 0, lane i = position i), first rejection
        if (warp == 0) {
            bool acc = true, tie = false;
            const int i = lane;
            if (i < m) {
                const RowStat A = i < K ? sh.row[i][l] : sh.extra[l][i - K];
                const RowStat Bq = i < K ? sh.row[i][l - 1] : sh.extra[l - 1][i - K];
                const int32_t t = sh.c[l][i];
                if (A.bad || Bq.bad) atomicOr(&sh.flags, (uint32_t)MSD_F_NONFINITE);
                if (t < 0 || t >= V) {
                    acc = false;
                    atomicOr(&sh.flags, (uint32_t)MSD_F_TOKEN_OOB);
                } else if (p.greedy) {
                    acc = (t == A.amax);
                } else {
                    const bool draft = i < K && t == p.cand0[b * K + i];
                    const float za = draft ? sh.zpre[l][i] : clamp1(Elem<Tin>::load1(row_ptr<Tin>(p, l, b, i) + t));
                    const float zb = draft ? sh.zpre[l - 1][i] : clamp1(Elem<Tin>::load1(row_ptr<Tin>(p, l - 1, b, i) + t));
                    const double u = (double)sh.ua[l - 1][i];
                    if (!(za > NEG_MASKED)) {
                        acc = false;
                        tie = u < TIE_EPS;
                    } else if (!(zb > NEG_MASKED)) {
                        acc = true;
                    } else {
                        const double lr = ((double)za - (double)zb) * (double)s_sc - (A.lse - Bq.lse);
                        const double r = lr >= 0.0 ? 1.0 : exp(lr);
                        acc = u < r;
                        tie = fabs(u - r) < TIE_EPS;
                    }
                }
            }
            const unsigned rej = __ballot_sync(0xffffffffu, !acc);
            const int n = rej ? (__ffs(rej) - 1) : m;
            const unsigned ties = __ballot_sync(0xffffffffu, tie && i <= n && i < m);
            if (lane == 0) {
                sh.n[l] = min(n, m);
                if (ties) { st_near[l] += __popc(ties); atomicOr(&sh.flags, (uint32_t)MSD_F_NEAR_TIE); }
            }
        }
        __syncthreads();
        const int n = sh.n[l];

        TPROF(2)
        // ---- per-position divergence of pair (l-1, l), i < K
        for (int i = warp; i < K; i += NWARP) {   // one warp per position: lanes over slices
            double d = 0.0;
            const double* R = res_b + ((size_t)i * (L - 1) + (l - 1)) * C;
            for (int s = lane; s < C; s += 32) d += R[s];
            d = warp_sum_d(d);
            if (lane != 0) continue;
            double kl = sh.kl[i][l];
            const bool kinf = !(kl < KL_INF_THRESH);
            if (kinf) kl = INFINITY;
            if (p.pos_dtv) p.pos_dtv[((size_t)(l - 1) * p.B + b) * K + i] = (float)d;
            if (p.pos_kl) p.pos_kl[((size_t)(l - 1) * p.B + b) * K + i] = (float)kl;
            if (p.stats) {
                msd_pair_stats* st = p.stats + (l - 1);
                const double dc = d < 0 ? 0 : (d > 1 ? 1 : d);
                atomicAdd((unsigned long long*)&st->dtv_fx, (unsigned long long)llrint(dc * MSD_DTV_SCALE));
                if (kinf) atomicAdd((unsigned long long*)&st->kl_inf, 1ull);
                else {
                    const double kc = kl < 0 ? 0 : (kl > 1048576.0 ? 1048576.0 : kl);
                    atomicAdd((unsigned long long*)&st->kl_fx, (unsigned long long)llrint(kc * MSD_KL_SCALE));
                }
            }
            if (kinf) atomicOr(&sh.flags, (uint32_t)MSD_F_KL_INF);
        }

        TPROF(3)
        // ---- emission
        const bool is_final = (l == L - 1);
        const bool resid = n < m;
        const bool bonus = !resid && (is_final ? p.fbonus : p.ibonus);
        if (resid || bonus) {
            const int pos = resid ? n : m;
            const Tin* ra = row_ptr<Tin>(p, l, b, pos);
            const Tin* rb = row_ptr<Tin>(p, l - 1, b, pos);
            // stats of the rows at `pos`
            RowStat A, Bq;
            if (pos < K) {
                A = sh.row[pos][l];
                Bq = sh.row[pos][l - 1];
            } else {
                if (!resid) {  // bonus row: (re)compute so sh.part holds its slice partials
                    RowStat r = row_stats<Tin>(ra, V, C, p.VSe, sh, p.greedy != 0);
                    if (tid == 0) { sh.extra[l][pos - K] = r; sh.extra_ok[l][pos - K] = 1; }
                    __syncthreads();
                }
                A = sh.extra[l][pos - K];
                Bq = resid ? sh.extra[l - 1][pos - K] : A;
            }
            int32_t y;
            bool tie = false, small = false, exact = false;
            if (p.greedy) {
                y = A.amax;
            } else {
                const double u = (double)sh.ue[l - 1][pos];
                // per-slice weights
                if (resid) {
                    if (pos < K) {
                        const double* R = res_b + ((size_t)pos * (L - 1) + (l - 1)) * C;
                        for (int s = tid; s < C; s += T) sh.w[s] = R[s];
                        __syncthreads();
                    } else {
                        pair_resid<Tin>(ra, rb, A, Bq, V, C, p.VSe, sh);
                    }
                } else {
                    const Partial* P = part_b + ((size_t)pos * L + l) * C;
                    for (int s = tid; s < C; s += T) {
                        const Partial pr = pos < K ? P[s] : sh.part[s];
                        sh.w[s] = pr.S * dexp_neg(((double)pr.m - A.M) * (double)s_sc) / A.S;
                    }
                    __syncthreads();
                }
                double Z = 0.0;
                for (int s = lane; s < C; s += 32) Z += sh.w[s];
                Z = warp_sum_d(Z);
                TPROF(7)
                y = -1;
                if (!p.exact_all && (!resid || Z >= p.z_safe))
                    y = draw_slices<Tin>(resid, ra, rb, A.lse, Bq.lse, V, C, p.VSe, Z, u, sh, &tie);
                TPROF(8)
                if (y < 0) {
                    exact = true;
                    tie = false;
                    y = draw_exact<Tin>(resid, ra, rb, A, Bq, V, C, p.VSe, u, sh, &tie, &small, p.board);
                }
            }
            if (tid == 0) {
                sh.y = y;
                if (tie) { st_near[l] += 1; sh.flags |= MSD_F_NEAR_TIE; }
                if (small) sh.flags |= MSD_F_RESID_SMALL;
                if (exact) { st_exact[l] += 1; sh.flags |= MSD_F_EXACT_DRAW; }
            }
            __syncthreads();
        }
        TPROF(4)
        // ---- next candidate list
        if (tid == 0) {
            for (int i = 0; i < n; ++i) sh.c[l + 1][i] = sh.c[l][i];
            if (resid || bonus) { sh.c[l + 1][n] = sh.y; sh.m[l + 1] = n + 1; }
            else { for (int i = n; i < m; ++i) sh.c[l + 1][i] = sh.c[l][i]; sh.m[l + 1] = m; }
        }
        __syncthreads();
    }

    TPROF(5)
    // ---- outputs, rollback lengths, stats, counter reset
    const int clen = sh.m[L];
    for (int j = tid; j < p.out_ld; j += T) p.out_tok[b * p.out_ld + j] = j < clen ? sh.c[L][j] : -1;
    if (tid == 0) {
        p.out_len[b] = clen;
        for (int l = 1; l < L; ++l) {
            if (p.n_acc) p.n_acc[(size_t)(l - 1) * p.B + b] = sh.n[l];
            if (p.m_cand) p.m_cand[(size_t)(l - 1) * p.B + b] = sh.m[l];
            if (p.stats) {
                msd_pair_stats* st = p.stats + (l - 1);
                atomicAdd((unsigned long long*)&st->positions, (unsigned long long)K);
                atomicAdd((unsigned long long*)&st->proposed, (unsigned long long)sh.m[l]);
                atomicAdd((unsigned long long*)&st->accepted, (unsigned long long)sh.n[l]);
                if (st_near[l]) atomicAdd((unsigned long long*)&st->near_ties, (unsigned long long)st_near[l]);
                if (st_exact[l]) atomicAdd((unsigned long long*)&st->exact_draws, (unsigned long long)st_exact[l]);
            }
        }
        if (p.rollback) {
            // drafter: its first draft_fed draft tokens; verifier l: its candidates c_l
            int d = p.draft_fed, keep = 0;
            while (keep < d && keep < clen && p.cand0[b * K + keep] == sh.c[L][keep]) ++keep;
            p.rollback[b] = d - keep;
            for (int l = 1; l < L; ++l) {
                int kk = 0;
                while (kk < sh.m[l] && kk < clen && sh.c[l][kk] == sh.c[L][kk]) ++kk;
                p.rollback[(size_t)l * p.B + b] = sh.m[l] - kk;
            }
        }
        if (sh.flags) atomicOr(&p.flags[b], sh.flags);
    }
    // reset the core's exchange state of this request's units for the next call
    for (int i = tid; i < K; i += T) p.cnt[((size_t)b * K + i) * CNT_STRIDE] = 0u;
    unsigned long long* pm = reinterpret_cast<unsigned long long*>(p.partms) + (size_t)b * K * L * C;
    for (int t = tid; t < K * L * C; t += T) pm[t] = 0ull;
    TPROF(6)
    // this request is done: help with other requests' exact draws while any is unfinished
    if (tid == 0 && p.board) {
        __threadfence();
        atomicAdd(&p.board->finished, 1u);
    }
    exact_help<Tin>(p.board, p.B, sh);
#ifdef MSD_PROF
    if (tid == 0 && b < 4096) g_tail_cta[b][1] = globaltimer();
#endif
}

// tab[h] = exp(bf16 with bits h) in float64; NaN where |z| >= 700 or z is not finite
__global__ void exp_table_kernel(double* tab) {
    const uint32_t h = blockIdx.x * blockDim.x + threadIdx.x;
    if (h >= 65536u) return;
    const float z = __uint_as_float(h << 16);
    tab[h] = (isfinite(z) && fabsf(z) < 700.f) ? exp((double)z) : __longlong_as_double(0x7FF8000000000000LL);
}
__device__ double g_exptab[65536];

cudaError_t exp_table(const double** out, int init) {
    void* ptr = nullptr;
    cudaError_t e = cudaGetSymbolAddress(&ptr, g_exptab);
    if (e != cudaSuccess) return e;
    if (init) {
        cudaStream_t st;
        e = cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
        if (e != cudaSuccess) return e;
        exp_table_kernel<<<256, 256, 0, st>>>(reinterpret_cast<double*>(ptr));
        e = cudaGetLastError();
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);
        cudaStreamDestroy(st);
        if (e != cudaSuccess) return e;
    }
    *out = reinterpret_cast<const double*>(ptr);
    return cudaSuccess;
}

cudaError_t launch_tail(const TailParams& p0, int bf16, cudaStream_t s) {
    if (p0.B <= 0) return cudaSuccess;
    TailParams p = p0;
    const size_t dyn = (size_t)p.K * p.L * p.C * sizeof(Partial) + (size_t)p.K * (p.L - 1) * p.C * sizeof(double);
    p.prefetch = dyn <= TAIL_DYN_MAX ? 1 : 0;
    const size_t smem = p.prefetch ? dyn : 0;
    auto k = bf16 ? tail_kernel<__nv_bfloat16> : tail_kernel<float>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)TAIL_DYN_MAX);
    if (e != cudaSuccess) return e;
    k<<<p.B, T, smem, s>>>(p);
    return cudaGetLastError();
}

}  // namespace msd

#ifdef MSD_PROF
extern "C" int msd_debug_tail_req(unsigned long long* out) {
    return cudaMemcpyFromSymbol(out, msd::g_tail_req, sizeof(unsigned long long) * 4096 * 16) != cudaSuccess;
}
extern "C" int msd_debug_tail_cta(unsigned long long* out) {
    return cudaMemcpyFromSymbol(out, msd::g_tail_cta, sizeof(unsigned long long) * 4096 * 2) != cudaSuccess;
}
extern "C" int msd_debug_tail_prof(unsigned long long* out16, int reset) {
    if (cudaMemcpyFromSymbol(out16, msd::g_tail_prof, sizeof(unsigned long long) * 16) != cudaSuccess) return 1;
    if (reset) {
        unsigned long long z[16] = {};
        if (cudaMemcpyToSymbol(msd::g_tail_prof, z, sizeof(z)) != cudaSuccess) return 1;
    }
    return 0;
}
#endif
