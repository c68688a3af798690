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
// residual mass is small (Z < z_safe) the fp32-derived slice masses are not
// accurate enough relative to Z, so the whole row pair is recomputed in float64
// (`draw_exact`, flagged MSD_F_EXACT_DRAW).  Rows at positions >= K (bonus rows,
// needed only when a level accepts everything) are computed on demand here.
#include "msd_common.cuh"
#include "msd_internal.h"

namespace msd {

constexpr int MAXSLICES = 128;   // V <= 524288
constexpr double TIE_EPS = 1e-6;

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
    double sel_before;
    int32_t sel_slice;
};

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

// Row statistics of an arbitrary row (bonus rows at positions >= K): per-slice
// partials into sh.part[], combined RowStat returned to every thread.
template <typename Tin>
__device__ RowStat row_stats(const Tin* row, int64_t V, int C, int vse, TailShared& sh) {
    constexpr int VEC = Elem<Tin>::VEC;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __shared__ float wmx[NWARP], wsm[NWARP];
    __shared__ int wam[NWARP];
    for (int s = 0; s < C; ++s) {
        float x[ET];
        load_slice<Tin>(row, V, s, vse, x);
        float tm = x[0];
#pragma unroll
        for (int k = 1; k < ET; ++k) tm = fmaxf(tm, x[k]);
        const float wm = warp_max(tm);
        float sum = 0.f;
#pragma unroll
        for (int k = 0; k < ET; ++k) sum += ex2f((x[k] - wm) * LOG2E);
        sum = warp_sum(sum);
        int am = 0x7fffffff;
#pragma unroll
        for (int k = ET - 1; k >= 0; --k)
            if (x[k] == wm) am = (int)((int64_t)s * vse + ((k / VEC) * T + threadIdx.x) * VEC + (k % VEC));
        am = warp_min_i(am);
        __syncthreads();
        if (lane == 0) { wmx[warp] = wm; wsm[warp] = sum; wam[warp] = am; }
        __syncthreads();
        if (warp == 0) {
            const bool act = lane < NWARP;
            const float mw = act ? wmx[lane] : -INFINITY;
            const float ms = warp_max(mw);
            double f = act ? exp((double)mw - (double)ms) : 0.0;
            if (act && !(mw > NEG_MASKED)) f = (ms > NEG_MASKED) ? 0.0 : 1.0;
            double Ss = act ? (double)wsm[lane] * f : 0.0;
            int a = (act && mw == ms) ? wam[lane] : 0x7fffffff;
            Ss = warp_sum_d(Ss);
            a = warp_min_i(a);
            if (lane == 0) {
                Partial pr;
                pr.m = ms; pr.amax = a; pr.S = Ss; pr.Kl = 0.0;
                sh.part[s] = pr;
            }
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
            S += sh.part[s].S * exp((double)sh.part[s].m - (double)m);
            if (sh.part[s].m == m) am = min(am, sh.part[s].amax);
            if (isnan(sh.part[s].m) || isnan(sh.part[s].S)) bad = true;
        }
        S = warp_sum_d(S);
        am = warp_min_i(am);
        bad = __any_sync(0xffffffffu, bad);
        if (lane == 0) {
            RowStat r;
            r.M = m; r.S = S; r.lse = (double)m + log(S);
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

// Per-slice residual mass R_s = sum max(p - q, 0) of an arbitrary row pair into
// sh.w[] (fp32 per element, float64 across warps; the core's pass-2 arithmetic).
template <typename Tin>
__device__ void pair_resid(const Tin* ra, const Tin* rb, const RowStat& A, const RowStat& Bq,
                           int64_t V, int C, int vse, TailShared& sh) {
    const double rho = Bq.S > 0 ? A.S / Bq.S : 0.0;
    const float rh = (float)rho, rl = (float)(rho - (double)rh);
    const float Ma = (float)A.M, Mb = (float)Bq.M;
    for (int s = 0; s < C; ++s) {
        float xa[ET], xb[ET];
        load_slice<Tin>(ra, V, s, vse, xa);
        load_slice<Tin>(rb, V, s, vse, xb);
        float acc = 0.f;
#pragma unroll
        for (int k = 0; k < ET; ++k) {
            const float ea = ex2f((xa[k] - Ma) * LOG2E);
            const float eb = ex2f((xb[k] - Mb) * LOG2E);
            float t = fmaf(-eb, rh, ea);
            t = fmaf(-eb, rl, t);
            acc += fmaxf(t, 0.f);
        }
        const double tot = block_sum_d((double)acc, sh);
        if (threadIdx.x == 0) sh.w[s] = tot / A.S;
    }
    __syncthreads();
}

// Weight of vocabulary entry z (and z' for the residual) in float64.
__device__ __forceinline__ double wt(bool resid, float za, float zb, double A, double B) {
    if (!(za > NEG_MASKED)) return 0.0;
    const double pa = exp((double)za - A);
    if (!resid) return pa;
    const double qb = (zb > NEG_MASKED) ? exp((double)zb - B) : 0.0;
    const double r = pa - qb;
    return r > 0.0 ? r : 0.0;
}

// Inverse-CDF search inside slice s with weights wt(), given the float64 mass of
// all earlier slices (`before`) and the target u*Z.  Thread t scans the 16
// contiguous entries [t*16, t*16+16) of the slice.  Returns the token or -1.
template <typename Tin>
__device__ int32_t scan_slice(bool resid, const Tin* ra, const Tin* rb, double A, double B,
                              int64_t V, int s, int vse, double before, double target, double Z, double u,
                              TailShared& sh, bool* tie) {
    const int64_t e0 = (int64_t)s * vse + threadIdx.x * ET;
    V = min(V, (int64_t)(s + 1) * vse);
    if (threadIdx.x == 0) sh.near = 0;
    double w[ET];
    double loc = 0.0;
#pragma unroll
    for (int k = 0; k < ET; ++k) {
        const int64_t v = e0 + k;
        float za = NEG_CLAMP, zb = NEG_CLAMP;
        if (v < V) {
            za = clamp1(Elem<Tin>::load1(ra + v));
            if (resid) zb = clamp1(Elem<Tin>::load1(rb + v));
        }
        w[k] = wt(resid, za, zb, A, B);
        loc += w[k];
    }
    // exclusive scan of per-thread totals (fixed order: serial over warps)
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
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
    int found = 0x7fffffff;
    double cprev_f = 0.0, c_f = 0.0;
#pragma unroll
    for (int k = 0; k < ET; ++k) {
        const double cp = c;
        c += w[k];
        if (found == 0x7fffffff && w[k] > 0.0 && c > target) {
            found = (int)(e0 + k);
            cprev_f = cp;
            c_f = c;
        }
    }
    const int best = block_min_i(found, sh);
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
                               int64_t V, int C, int vse, double Z, double u, TailShared& sh, bool* tie) {
    if (threadIdx.x == 0) {
        const double target = u * Z;
        double c = 0.0;
        int sel = -1;
        int lastpos = -1;
        double before = 0.0;
        for (int s = 0; s < C; ++s) {
            if (sh.w[s] > 0.0) lastpos = s;
            if (sel < 0 && sh.w[s] > 0.0 && c + sh.w[s] > target) { sel = s; before = c; }
            c += sh.w[s];
        }
        if (sel < 0) { sel = -1 - (lastpos < 0 ? 0 : lastpos); before = c; }
        sh.sel_slice = sel;
        sh.sel_before = before;
    }
    __syncthreads();
    const int sel = sh.sel_slice;
    const double before = sh.sel_before;
    __syncthreads();
    if (sel < 0) {  // u*Z beyond the total (rounding): clamp to the last positive entry
        *tie = true;
        return last_positive<Tin>(resid, ra, rb, A, B, V, -1 - sel, vse, sh);
    }
    return scan_slice<Tin>(resid, ra, rb, A, B, V, sel, vse, before, u * Z, Z, u, sh, tie);
}

// Exact float64 draw over the whole row (pair): exact normalisers, exact slice
// masses, exact scan.  Residual mass < 1e-12 -> draw from p.
template <typename Tin>
__device__ int32_t draw_exact(bool resid, const Tin* ra, const Tin* rb, const RowStat& Ar,
                              const RowStat& Br, int64_t V, int C, int vse, double u, TailShared& sh,
                              bool* tie, bool* small) {
  for (int attempt = 0; attempt < 2; ++attempt) {
    // exact normalisers
    double sa = 0.0, sb = 0.0;
    for (int64_t v = threadIdx.x; v < V; v += T) {
        const float za = clamp1(Elem<Tin>::load1(ra + v));
        if (za > NEG_MASKED) sa += exp((double)za - Ar.M);
        if (resid) {
            const float zb = clamp1(Elem<Tin>::load1(rb + v));
            if (zb > NEG_MASKED) sb += exp((double)zb - Br.M);
        }
    }
    sa = block_sum_d(sa, sh);
    if (resid) sb = block_sum_d(sb, sh);
    const double A = Ar.M + log(sa);
    const double B = resid ? Br.M + log(sb) : 0.0;
    for (int s = 0; s < C; ++s) {
        double acc = 0.0;
        for (int64_t v = (int64_t)s * vse + threadIdx.x; v < min(V, (int64_t)(s + 1) * vse); v += T) {
            const float za = clamp1(Elem<Tin>::load1(ra + v));
            const float zb = resid ? clamp1(Elem<Tin>::load1(rb + v)) : NEG_CLAMP;
            acc += wt(resid, za, zb, A, B);
        }
        acc = block_sum_d(acc, sh);
        if (threadIdx.x == 0) sh.w[s] = acc;
    }
    __syncthreads();
    double Z = 0.0;
    for (int s = 0; s < C; ++s) Z += sh.w[s];
    if (resid && Z < 1e-12) {   // residual vanished -> draw from p
        *small = true;
        resid = false;
        continue;
    }
    int32_t y = draw_slices<Tin>(resid, ra, rb, A, B, V, C, vse, Z, u, sh, tie);
    return y < 0 ? 0 : y;
  }
  return 0;
}

template <typename Tin>
__global__ void __launch_bounds__(T) tail_kernel(TailParams p) {
    __shared__ TailShared sh;
    const int64_t b = blockIdx.x;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int L = p.L, K = p.K, C = p.C;
    const int64_t V = p.V;

    if (tid == 0) {
        sh.flags = 0;
        int m1 = p.m0 ? p.m0[b] : K;
        m1 = max(0, min(m1, K));
        sh.m[1] = m1;
    }
    for (int q = tid; q < MAXL * MAXL; q += T) (&sh.extra_ok[0][0])[q] = 0;
    // row normalisers (Eq. 1) and KL numerators of every draft-position row, combined from
    // the core's slice partials in a fixed order (one warp per row)
    for (int r = warp; r < K * L; r += NWARP) {
        const int i = r / L, l = r % L;
        double Kl;
        const Partial* pp = p.partials + (((size_t)b * K + i) * L + l) * C;
        RowStat rs = combine_row(pp, C, &Kl, l > 0 ? pp - C : nullptr);
        if (lane == 0) { sh.row[i][l] = rs; sh.kl[i][l] = Kl; }
    }
    __syncthreads();
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

    for (int l = 1; l < L; ++l) {
        const int m = sh.m[l];
        // rows at positions >= K needed by this level's tests (level l and l-1)
        for (int i = K; i < m; ++i) {
            for (int lv = l - 1; lv <= l; ++lv) {
                if (!sh.extra_ok[lv][i - K]) {
                    RowStat r = row_stats<Tin>(row_ptr<Tin>(p, lv, b, i), V, C, p.VSe, sh);
                    if (tid == 0) { sh.extra[lv][i - K] = r; sh.extra_ok[lv][i - K] = 1; }
                    __syncthreads();
                }
            }
        }
        __syncthreads();

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
                    const float za = clamp1(Elem<Tin>::load1(row_ptr<Tin>(p, l, b, i) + t));
                    const float zb = clamp1(Elem<Tin>::load1(row_ptr<Tin>(p, l - 1, b, i) + t));
                    const double u = (double)p.u_acc[(l - 1) * p.ua_l + b * p.ua_b + i];
                    if (!(za > NEG_MASKED)) {
                        acc = false;
                        tie = u < TIE_EPS;
                    } else if (!(zb > NEG_MASKED)) {
                        acc = true;
                    } else {
                        const double lr = ((double)za - (double)zb) - (A.lse - Bq.lse);
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

        // ---- per-position divergence of pair (l-1, l), i < K
        for (int i = tid; i < K; i += T) {
            const size_t u = (size_t)b * K + i;
            double d = 0.0;
            const double* R = p.resid + (u * (L - 1) + (l - 1)) * C;
            for (int s = 0; s < C; ++s) d += R[s];
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
                    RowStat r = row_stats<Tin>(ra, V, C, p.VSe, sh);
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
                const double u = (double)p.u_emit[(l - 1) * p.ue_l + b * p.ue_b + pos];
                // per-slice weights
                if (resid) {
                    if (pos < K) {
                        const double* R = p.resid + (((size_t)b * K + pos) * (L - 1) + (l - 1)) * C;
                        for (int s = tid; s < C; s += T) sh.w[s] = R[s];
                        __syncthreads();
                    } else {
                        pair_resid<Tin>(ra, rb, A, Bq, V, C, p.VSe, sh);
                    }
                } else {
                    const Partial* P = p.partials + (((size_t)b * K + pos) * L + l) * C;
                    for (int s = tid; s < C; s += T) {
                        const Partial pr = pos < K ? P[s] : sh.part[s];
                        sh.w[s] = pr.S * exp((double)pr.m - A.M) / A.S;
                    }
                    __syncthreads();
                }
                double Z = 0.0;
                for (int s = 0; s < C; ++s) Z += sh.w[s];
                y = -1;
                if (!p.exact_all && (!resid || Z >= p.z_safe))
                    y = draw_slices<Tin>(resid, ra, rb, A.lse, Bq.lse, V, C, p.VSe, Z, u, sh, &tie);
                if (y < 0) {
                    exact = true;
                    tie = false;
                    y = draw_exact<Tin>(resid, ra, rb, A, Bq, V, C, p.VSe, u, sh, &tie, &small);
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
        // ---- next candidate list
        if (tid == 0) {
            for (int i = 0; i < n; ++i) sh.c[l + 1][i] = sh.c[l][i];
            if (resid || bonus) { sh.c[l + 1][n] = sh.y; sh.m[l + 1] = n + 1; }
            else { for (int i = n; i < m; ++i) sh.c[l + 1][i] = sh.c[l][i]; sh.m[l + 1] = m; }
        }
        __syncthreads();
    }

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
}

cudaError_t launch_tail(const TailParams& p, int bf16, cudaStream_t s) {
    if (p.B <= 0) return cudaSuccess;
    if (bf16)
        tail_kernel<__nv_bfloat16><<<p.B, T, 0, s>>>(p);
    else
        tail_kernel<float><<<p.B, T, 0, s>>>(p);
    return cudaGetLastError();
}

}  // namespace msd
