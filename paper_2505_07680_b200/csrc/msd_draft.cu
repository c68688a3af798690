// msd_draft.cu -- draft-side sampling step ("the draft model ...
// autoregressively generates a sequence of gamma candidate tokens", P:245 DraftProcessor;
// S:337-345 "W sequential next_dist+sample (or argmax in greedy mode)").
//
// One draft step for B sequences: row b of the drafter's logits -> token[b] = min{t : C_t >
// u_b Z} with C_t = sum_{v<=t} exp(z_v - M), Z = C_{V-1} (inverse CDF of softmax, reading
// R5), or the first argmax in greedy mode; lse[b] = M + log Z (Eq. 1) and q_tok[b] =
// softmax(z_b)[token] (the q(x) of the verifier's ratio).
//
// One CTA per row, ONE streaming read of the row: every warp-iteration covers a chunk of
// 32 * VEC consecutive entries and leaves its (chunk max, fp64 chunk sum) in shared memory;
// the CTA then combines the chunks in float64, finds the chunk holding the crossing by a
// block-wide fp64 prefix, and one warp rescans that chunk (from L1/L2, 512 B) with float64
// weights exp(z - M) to place the token.  bf16 rows are reduced straight from the loaded
// words with packed f32x2 arithmetic; 2 of every 8 exponentials run as an FMA-pipe
// polynomial (MUFU alone would bound the kernel above HBM time).
#include "msd_common.cuh"
#include "msd_internal.h"

namespace msd {

constexpr int DT = 256;                 // threads per CTA
constexpr int DNW = DT / 32;

template <typename Tin>
__device__ __forceinline__ void draft_vec(const Tin* row, int64_t e, int64_t V, float* x) {
    constexpr int VEC = Elem<Tin>::VEC;
    if (e + VEC <= V) {
        unpack_clamped<Tin>(__ldg(reinterpret_cast<const uint4*>(row + e)), x);
    } else {
#pragma unroll
        for (int k = 0; k < VEC; ++k) x[k] = (e + k < V) ? clamp1(Elem<Tin>::load1(row + e + k)) : NEG_CLAMP;
    }
}

// exp(x - m) summed over one vector, 1 of every 8 entries on the FMA pipe
template <int VEC>
__device__ __forceinline__ float vec_expsum(const float* x, float m) {
    float s = 0.f;
#pragma unroll
    for (int q = 0; q < VEC; ++q) {
        const float a = (x[q] - m) * LOG2E;
        s += (q % 8 == 7) ? exp2f_fma(a) : ex2f(a);
    }
    return s;
}

__device__ __forceinline__ float warp_max_nan(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = max_nan_f32(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

__device__ __forceinline__ float redux_max_nan_f32(float v) {
    float r;
    asm("redux.sync.max.NaN.f32 %0, %1, 0xffffffff;" : "=f"(r) : "f"(v));
    return r;
}

// one chunk held in registers: CV vectors per lane -> warp max (one redux) and this lane's
// fp32 partial sum of exp(x - warp max); the float64 warp sums are formed after the stream
template <typename Tin, int CV, bool GREEDY>
__device__ __forceinline__ void chunk_stats(const float (&x)[CV][Elem<Tin>::VEC], int64_t e0,
                                            float& bestv, int& besti, float& wm, float& ls) {
    constexpr int VEC = Elem<Tin>::VEC;
    float mv = x[0][0];
#pragma unroll
    for (int v = 0; v < CV; ++v)
#pragma unroll
        for (int q = 0; q < VEC; ++q) mv = max_nan_f32(mv, x[v][q]);
    if (GREEDY) {
#pragma unroll
        for (int v = 0; v < CV; ++v)
#pragma unroll
            for (int q = 0; q < VEC; ++q)
                if (x[v][q] > bestv) { bestv = x[v][q]; besti = (int)(e0 + v * 32 * VEC) + q; }
    }
    wm = redux_max_nan_f32(mv);
    float s = 0.f;
    if (wm > NEG_MASKED) {
#pragma unroll
        for (int v = 0; v < CV; ++v) s += vec_expsum<VEC>(x[v], wm);
    }
    ls = s;
}

// bf16 chunk straight from the loaded words: max.NaN.bf16x2 for the lane maximum, then per
// pair FHADD.BF16 (x - wm without unpacking), one FMUL2 by log2 e, ex2 (every 8th element on
// the FMA pipe) and FADD2 partial sums -- about 3.5 issue slots per element.  Same values
// as chunk_stats on unpacked floats: x - wm and (x - wm) log2 e round identically.
template <int CV, int NPOLY>
__device__ __forceinline__ void chunk_stats_bf16(const uint4 (&raw)[CV], float& wm, float& ls) {
    uint32_t mw = raw[0].x;
#pragma unroll
    for (int v = 0; v < CV; ++v) {
        mw = max_nan_bf16x2(mw, raw[v].x);
        mw = max_nan_bf16x2(mw, raw[v].y);
        mw = max_nan_bf16x2(mw, raw[v].z);
        mw = max_nan_bf16x2(mw, raw[v].w);
    }
    wm = redux_max_nan_f32(max_nan_f32(bf16lo(mw), bf16hi(mw)));
    float2 acc = make_float2(0.f, 0.f);
    if (wm > NEG_MASKED) {
        const float nm = -wm;
        const float2 l2e = make_float2(LOG2E, LOG2E);
#pragma unroll
        for (int v = 0; v < CV; ++v) {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const uint32_t w = k == 0 ? raw[v].x : k == 1 ? raw[v].y : k == 2 ? raw[v].z : raw[v].w;
                float2 y;
                asm("{ .reg .b16 lo, hi; mov.b32 {lo, hi}, %2; add.rn.f32.bf16 %0, lo, %3; add.rn.f32.bf16 %1, hi, %3; }"
                    : "=f"(y.x), "=f"(y.y) : "r"(w), "f"(nm));
                const float2 t = __fmul2_rn(y, l2e);
                float2 e;
                if (2 * k >= 8 - NPOLY) e = exp2_pair_fma(t);      // NPOLY even: whole pairs
                else { e.x = ex2f(t.x); e.y = ex2f(t.y); }
                acc = __fadd2_rn(acc, e);
            }
        }
    }
    ls = acc.x + acc.y;
}

template <typename Tin, bool GREEDY, int DCV, int MINB, int DNPOLY>
__global__ void __launch_bounds__(DT, MINB) draft_kernel(DraftParams p) {
    // DCV vectors per lane per chunk (chunk = 32 * DCV * VEC entries)
    constexpr int VEC = Elem<Tin>::VEC;
    constexpr int SB = 32 * VEC;                          // entries per warp-vector (sub-block)
    constexpr int CH = DCV * SB;                          // entries per chunk
    extern __shared__ __align__(16) unsigned char dsm[];
    const int nch = (int)ceil_div(p.V, CH);
    float* cmax = reinterpret_cast<float*>(dsm);                       // [nch]
    double* csum = reinterpret_cast<double*>(dsm + align_up((size_t)nch * 4, 16));   // [nch]
    float* lsum = reinterpret_cast<float*>(csum + nch);                 // [nch][32] lane partials
    __shared__ double wred[DNW];
    __shared__ float fred[DNW];
    __shared__ int ired[DNW];
    __shared__ float s_M;
    __shared__ int s_ch;
    __shared__ double s_start;

    const int b = blockIdx.x;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t V = p.V;
    const Tin* row = reinterpret_cast<const Tin*>(p.z) + (int64_t)b * p.bs + (int64_t)p.row * p.ld;

    // ---- streaming pass: warp w takes chunks w, w + 8, ...; the next chunk's loads are in
    // flight while the current one is reduced.  Chunk c, vector v, lane l covers entries
    // c*CH + (v*32 + l)*VEC + [0, VEC).
    float bestv = -INFINITY;
    int besti = INT_MAX;
    const int nfull = (int)(V / CH);                       // chunks entirely inside the row
    int c = warp;
    if (sizeof(Tin) == 2 && !GREEDY) {
        // bf16: two register buffers, chunk c + 8 loads while chunk c is reduced
        uint4 ra[DCV], rb[DCV];
        auto ld = [&](uint4 (&r)[DCV], int cc) {
#pragma unroll
            for (int v = 0; v < DCV; ++v)
                r[v] = __ldg(reinterpret_cast<const uint4*>(row + (int64_t)cc * CH + (v * 32 + lane) * VEC));
        };
        auto put = [&](int cc, float wm, float ls) {
            lsum[cc * 32 + lane] = ls;
            if (lane == 0) cmax[cc] = wm;
        };
        if (c < nfull) ld(ra, c);
        for (; c < nfull; c += 2 * DNW) {
            float wm, ls;
            if (c + DNW < nfull) ld(rb, c + DNW);
            chunk_stats_bf16<DCV, DNPOLY>(ra, wm, ls);
            put(c, wm, ls);
            if (c + DNW >= nfull) break;
            if (c + 2 * DNW < nfull) ld(ra, c + 2 * DNW);
            chunk_stats_bf16<DCV, DNPOLY>(rb, wm, ls);
            put(c + DNW, wm, ls);
        }
    } else {
        uint4 raw[DCV];
        if (c < nfull) {
#pragma unroll
            for (int v = 0; v < DCV; ++v)
                raw[v] = __ldg(reinterpret_cast<const uint4*>(row + (int64_t)c * CH + (v * 32 + lane) * VEC));
        }
        for (; c < nfull; c += DNW) {
            float wm, ls;
            float x[DCV][VEC];
#pragma unroll
            for (int v = 0; v < DCV; ++v) unpack_clamped<Tin>(raw[v], x[v]);
            if (c + DNW < nfull) {
#pragma unroll
                for (int v = 0; v < DCV; ++v)
                    raw[v] = __ldg(reinterpret_cast<const uint4*>(row + (int64_t)(c + DNW) * CH + (v * 32 + lane) * VEC));
            }
            chunk_stats<Tin, DCV, GREEDY>(x, (int64_t)c * CH + lane * VEC, bestv, besti, wm, ls);
            lsum[c * 32 + lane] = ls;
            if (lane == 0) cmax[c] = wm;
        }
    }
    if (nfull < nch && warp == (nfull % DNW)) {            // the ragged last chunk
        const int cl = nfull;
        float x[DCV][VEC];
#pragma unroll
        for (int v = 0; v < DCV; ++v) {
            const int64_t e = (int64_t)cl * CH + (v * 32 + lane) * VEC;
            if (e < V) draft_vec<Tin>(row, e, V, x[v]);
            else {
#pragma unroll
                for (int q = 0; q < VEC; ++q) x[v][q] = NEG_CLAMP;
            }
        }
        float wm, ls;
        chunk_stats<Tin, DCV, GREEDY>(x, (int64_t)cl * CH + lane * VEC, bestv, besti, wm, ls);
        lsum[cl * 32 + lane] = ls;
        if (lane == 0) cmax[cl] = wm;
    }
    __syncthreads();

    // ---- row combine (float64, fixed order): M, Z; non-finite rows -> token -1
    for (int c = warp; c < nch; c += DNW) {              // chunk sums: fixed-order fp64 warp sums
        const double ws = warp_sum_d((double)lsum[c * 32 + lane]);
        if (lane == 0) csum[c] = ws;
    }
    float m = -INFINITY;
    for (int c = tid; c < nch; c += DT) m = max_nan_f32(m, cmax[c]);
    m = warp_max_nan(m);
    if (lane == 0) fred[warp] = m;
    __syncthreads();
    if (tid == 0) {
        float M = fred[0];
        for (int w = 1; w < DNW; ++w) M = max_nan_f32(M, fred[w]);
        s_M = M;
    }
    __syncthreads();                                     // (also orders the csum writes)
    const float M = s_M;
    // chunk weights relative to M, in place (csum[c] <- csum[c] exp(cmax[c] - M))
    double zt = 0.0;
    for (int c = tid; c < nch; c += DT) {
        const double w = (cmax[c] > NEG_MASKED) ? csum[c] * dexp_neg((double)cmax[c] - (double)M) : 0.0;
        csum[c] = w;
    }
    __syncthreads();
    // Z in a fixed order: thread t sums chunks [t*per, (t+1)*per), then warps, then the CTA
    const int per = (nch + DT - 1) / DT;
    const int c0 = min(nch, tid * per), c1 = min(nch, c0 + per);
    for (int c = c0; c < c1; ++c) zt += csum[c];
    // exclusive prefix of the per-thread sums (block scan in float64)
    double incl = zt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const double v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
    }
    if (lane == 31) wred[warp] = incl;
    __syncthreads();
    double wpre = 0.0, Z = 0.0;
    for (int w = 0; w < DNW; ++w) {
        if (w < warp) wpre += wred[w];
        Z += wred[w];
    }
    const double excl = wpre + incl - zt;
    const bool bad = !(M > NEG_MASKED) || !(M < INFINITY) || !(Z > 0.0) || !isfinite(Z);
    if (tid == 0) s_ch = INT_MAX;
    __syncthreads();
    if (bad) {
        if (tid == 0) {
            p.token[b] = -1;
            if (p.lse) p.lse[b] = NAN;
            if (p.q_tok) p.q_tok[b] = NAN;
            if (p.flags) atomicOr(&p.flags[b], (uint32_t)MSD_F_NONFINITE);
        }
        return;
    }
    const double lse = (double)M + log(Z);

    int tok = -1;
    uint32_t fl = 0;
    if (GREEDY) {
        // first argmax: max value, then smallest index
        float v = bestv;
        int i = besti;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const float v2 = __shfl_xor_sync(0xffffffffu, v, o);
            const int i2 = __shfl_xor_sync(0xffffffffu, i, o);
            if (v2 > v || (v2 == v && i2 < i)) { v = v2; i = i2; }
        }
        if (lane == 0) { fred[warp] = v; ired[warp] = i; }
        __syncthreads();
        if (tid == 0) {
            float bv = fred[0];
            int bi = ired[0];
            for (int w = 1; w < DNW; ++w)
                if (fred[w] > bv || (fred[w] == bv && ired[w] < bi)) { bv = fred[w]; bi = ired[w]; }
            s_ch = bi;
        }
        __syncthreads();
        tok = s_ch;
    } else {
        // ---- chunk holding the crossing: first c with prefix_c > u Z and weight > 0
        const double target = (double)p.u[b] * Z;
        if (zt > 0.0 && excl + zt > target) {
            double run = excl;
            for (int c = c0; c < c1; ++c) {
                run += csum[c];
                if (run > target && csum[c] > 0.0) {
                    atomicMin(&s_ch, c);
                    break;
                }
            }
        }
        __syncthreads();
        int c = s_ch;
        if (c == INT_MAX) {                   // fell off the end (rounding): last chunk with mass
            if (tid == 0) {
                int cl = nch - 1;
                while (cl > 0 && !(csum[cl] > 0.0)) --cl;
                s_ch = cl;
                fl |= MSD_F_NEAR_TIE;
            }
            __syncthreads();
            c = s_ch;
        }
        // exclusive prefix of chunk c (the same fixed-order sums as Z)
        if (tid == 0) {
            const int owner = c / per;
            double st = 0.0;
            for (int w = 0; w < owner / 32; ++w) st += wred[w];
            double s2 = 0.0;
            for (int cc = (owner / 32) * 32 * per; cc < c; ++cc) s2 += csum[cc];
            s_start = st + s2;
        }
        __syncthreads();
        if (warp == 0) {
            // rescan chunk c (and, if the float64 weights fall short, the chunks after it)
            double start = s_start;
            int found = -1, lastpos = -1;
            const int nsb = (int)ceil_div(V, SB);
            for (int sb = c * DCV; sb < nsb && found < 0; ++sb) {
                const int64_t e = (int64_t)sb * SB + (int64_t)lane * VEC;
                float x[VEC];
                if (e < V) draft_vec<Tin>(row, e, V, x);
                else {
#pragma unroll
                    for (int q = 0; q < VEC; ++q) x[q] = NEG_CLAMP;
                }
                double w[VEC], ls = 0.0;
#pragma unroll
                for (int q = 0; q < VEC; ++q) {
                    w[q] = (x[q] > NEG_MASKED) ? dexp_neg((double)x[q] - (double)M) : 0.0;
                    ls += w[q];
                }
                double li = ls;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const double v = __shfl_up_sync(0xffffffffu, li, o);
                    if (lane >= o) li += v;
                }
                double run = start + li - ls;
                int mine = -1;
                double cb_lo = 0.0, cb_hi = 0.0;
#pragma unroll
                for (int q = 0; q < VEC; ++q) {
                    const double nr = run + w[q];
                    if (mine < 0 && w[q] > 0.0 && nr > target) { mine = (int)e + q; cb_lo = run; cb_hi = nr; }
                    run = nr;
                }
                const unsigned hit = __ballot_sync(0xffffffffu, mine >= 0);
                int lp = -1;
#pragma unroll
                for (int q = 0; q < VEC; ++q)
                    if (w[q] > 0.0) lp = (int)e + q;
                lp = __reduce_max_sync(0xffffffffu, lp < 0 ? -1 : lp);
                if (lp >= 0) lastpos = lp;
                if (hit) {
                    const int src = __ffs(hit) - 1;
                    found = __shfl_sync(0xffffffffu, mine, src);
                    const double lo = __shfl_sync(0xffffffffu, cb_lo, src);
                    const double hi = __shfl_sync(0xffffffffu, cb_hi, src);
                    if (fabs(target - lo) < 1e-6 * Z || fabs(hi - target) < 1e-6 * Z) fl |= MSD_F_NEAR_TIE;
                }
                start = __shfl_sync(0xffffffffu, li, 31) + start;
            }
            if (found < 0) { found = lastpos; fl |= MSD_F_NEAR_TIE; }
            tok = found;
        }
    }
    if (tid == 0) {
        p.token[b] = tok;
        if (p.lse) p.lse[b] = (float)lse;
        if (p.q_tok) {
            const float zt_ = clamp1(Elem<Tin>::load1(row + tok));
            p.q_tok[b] = (float)dexp_neg((double)zt_ - lse);
        }
        if (fl && p.flags) atomicOr(&p.flags[b], fl);
    }
}

size_t draft_smem(int64_t V, int bf16, int cv) {
    const int VEC = bf16 ? 8 : 4;
    const int64_t nch = ceil_div(V, 32 * cv * VEC);
    return align_up((size_t)nch * 4, 16) + (size_t)nch * 8 + (size_t)nch * 32 * 4;
}

// chunks of 4 vectors per lane, 4 CTAs per SM (all rows of a 512-request batch resident),
// 2 of every 8 exponentials on the FMA pipe -- the best of the measured variants
template <typename Tin, bool G>
static cudaError_t launch_draft_t(const DraftParams& p, cudaStream_t s) {
    constexpr int CV = 4, MINB = 4, NPOLY = 2;
    const size_t smem = draft_smem(p.V, sizeof(Tin) == 2, CV);
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(draft_kernel<Tin, G, CV, MINB, NPOLY>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    draft_kernel<Tin, G, CV, MINB, NPOLY><<<p.B, DT, smem, s>>>(p);
    return cudaGetLastError();
}

cudaError_t launch_draft(const DraftParams& p, int bf16, cudaStream_t s) {
    if (p.B == 0) return cudaSuccess;
    if (bf16) return p.greedy ? launch_draft_t<__nv_bfloat16, true>(p, s) : launch_draft_t<__nv_bfloat16, false>(p, s);
    return p.greedy ? launch_draft_t<float, true>(p, s) : launch_draft_t<float, false>(p, s);
}

}  // namespace msd
