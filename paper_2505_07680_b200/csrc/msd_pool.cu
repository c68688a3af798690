// msd_pool.cu -- SimScore bootstrap: all-pairs divergence of an N-model pool (SURVEY 8(f)
// NEXT-1; "bootstrap(prefill dists per model) -> initialized pairwise SimScores";
// P:152 "initial logits used by the scheduler for baseline similarity calculations").
//
// For every position (b, k) and every pair (i < j) of the N models, in lexicographic pair
// order: DTV(p_i, p_j) = 1/2 sum_v |p_j(v) - p_i(v)| (Eq. 5) and KL(p_j || p_i)
// (reading R9: the later / larger model against the earlier one).  One CTA per position:
// pass 1 streams the N rows once with an online (max, sum) per thread (fp32 per vector,
// float64 across vectors) and reduces the row normalisers in float64; pass 2 streams them
// again and accumulates every pair at once.  Not on the per-step hot path (run at prefill or
// when the pool changes), so the second read is accepted: 2 N V elem bytes per position.
#include "msd_common.cuh"
#include "msd_internal.h"

namespace msd {

constexpr int PT = 256;           // threads per CTA
constexpr int PNW = PT / 32;
constexpr int UNR = 2;            // vectors per row in flight per thread

template <typename Tin>
__device__ __forceinline__ void pool_vec(const Tin* row, int64_t e, int64_t V, float* x) {
    constexpr int VEC = Elem<Tin>::VEC;
    if (e + VEC <= V) {
        unpack_clamped<Tin>(__ldg(reinterpret_cast<const uint4*>(row + e)), x);
    } else {
#pragma unroll
        for (int k = 0; k < VEC; ++k) x[k] = (e + k < V) ? clamp1(Elem<Tin>::load1(row + e + k)) : NEG_CLAMP;
    }
}


template <int N, int VEC>
__device__ __forceinline__ void p1_accum(const float (&x)[N][VEC], float (&m)[N], double (&S)[N]) {
#pragma unroll
    for (int l = 0; l < N; ++l) {
        float mv = x[l][0];
#pragma unroll
        for (int q = 1; q < VEC; ++q) mv = max_nan_f32(mv, x[l][q]);
        if (!(mv <= m[l])) {                         // larger (or NaN): rescale the running sum
            S[l] = (m[l] == -INFINITY) ? 0.0 : S[l] * dexp_neg((double)m[l] - (double)mv);
            m[l] = mv;
        }
        float sv = 0.f;
#pragma unroll
        for (int q = 0; q < VEC; ++q) sv += ex2f((x[l][q] - m[l]) * LOG2E);
        S[l] += (double)sv;
    }
}

// y_l = z_l - LSE_l, p_l = 2^(y_l log2 e); per pair (i < j): sum |p_j - p_i| and
// sum_{p_j > 0} p_j (y_j - y_i)  (fp32 per vector, float64 sums)
template <int N, int VEC, int NP>
__device__ __forceinline__ void p2_accum(const float (&x)[N][VEC], const float (&Lh)[N],
                                         const float (&Ll)[N], double (&dacc)[NP],
                                         double (&kacc)[NP], int& kinf) {
    float y[N][VEC], pr[N][VEC];
#pragma unroll
    for (int l = 0; l < N; ++l)
#pragma unroll
        for (int q = 0; q < VEC; ++q) {
            y[l][q] = (x[l][q] > NEG_MASKED) ? (x[l][q] - Lh[l]) - Ll[l] : -INFINITY;
            pr[l][q] = ex2f(y[l][q] * LOG2E);
        }
    int pi = 0;
#pragma unroll
    for (int i = 0; i < N; ++i) {
#pragma unroll
        for (int j = i + 1; j < N; ++j, ++pi) {
            float dv = 0.f, kv = 0.f;
#pragma unroll
            for (int q = 0; q < VEC; ++q) {
                dv += fabsf(pr[j][q] - pr[i][q]);
                if (y[j][q] > -INFINITY) {              // p_j > 0 (a finite logit; 0 log 0 = 0)
                    if (y[i][q] == -INFINITY) kinf |= 1 << pi;
                    else kv = fmaf(pr[j][q], y[j][q] - y[i][q], kv);
                }
            }
            dacc[pi] += (double)dv;
            kacc[pi] += (double)kv;
        }
    }
}

template <typename Tin, int N, typename F>
__device__ __forceinline__ void pool_stream(const Tin* const (&rows)[N], int64_t V, int tid, F&& f) {
    // UNR full vectors per row per iteration, every load issued before any arithmetic (bytes in
    // flight); then the ragged remainder one vector at a time
    constexpr int VEC = Elem<Tin>::VEC;
    constexpr int64_t STEP = (int64_t)PT * VEC;
    int64_t e0 = (int64_t)tid * VEC;
    for (; e0 + (UNR - 1) * STEP + VEC <= V; e0 += UNR * STEP) {
        uint4 raw[UNR][N];
#pragma unroll
        for (int u = 0; u < UNR; ++u)
#pragma unroll
            for (int l = 0; l < N; ++l)
                raw[u][l] = __ldg(reinterpret_cast<const uint4*>(rows[l] + e0 + u * STEP));
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
            float x[N][VEC];
#pragma unroll
            for (int l = 0; l < N; ++l) unpack_clamped<Tin>(raw[u][l], x[l]);
            f(x);
        }
    }
    for (; e0 < V; e0 += STEP) {
        float x[N][VEC];
#pragma unroll
        for (int l = 0; l < N; ++l) pool_vec<Tin>(rows[l], e0, V, x[l]);
        f(x);
    }
}

template <typename Tin, int N>
__global__ void __launch_bounds__(PT, 2) pool_kernel(PoolParams p) {
    constexpr int VEC = Elem<Tin>::VEC;
    constexpr int NP = N * (N - 1) / 2;
    const int64_t pos = blockIdx.x;                 // b * K + k
    const int64_t b = pos / p.K, k = pos % p.K;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t V = p.V;
    __shared__ double red[NP * 2 + N][PNW];
    __shared__ float redm[N][PNW];
    __shared__ double lse_s[N];
    __shared__ int bad_s[N];
    const Tin* rows[N];  // row (b, k) of every model
#pragma unroll
    for (int l = 0; l < N; ++l)
        rows[l] = reinterpret_cast<const Tin*>(p.lv.ptr[l]) + b * p.lv.bs[l] + k * p.lv.ld[l];

    // ---- pass 1: row normalisers (Eq. 1): online max / sum per thread, float64 combine
    float m[N];
    double S[N];
#pragma unroll
    for (int l = 0; l < N; ++l) { m[l] = -INFINITY; S[l] = 0.0; }
    pool_stream<Tin, N>(rows, V, tid, [&](const float (&x)[N][VEC]) { p1_accum<N, VEC>(x, m, S); });
#pragma unroll
    for (int l = 0; l < N; ++l) {
        const float wm = warp_max(m[l]);
        double f = (m[l] == -INFINITY) ? 0.0 : dexp_neg((double)m[l] - (double)wm);
        double ws = warp_sum_d(S[l] * f);
        if (lane == 0) { redm[l][warp] = wm; red[l][warp] = ws; }
    }
    __syncthreads();
    if (tid < N) {
        const int l = tid;
        float M = -INFINITY;
        for (int w = 0; w < PNW; ++w) M = max_nan_f32(M, redm[l][w]);
        double St = 0.0;
        for (int w = 0; w < PNW; ++w)
            if (redm[l][w] > -INFINITY) St += red[l][w] * dexp_neg((double)redm[l][w] - (double)M);
        lse_s[l] = (double)M + log(St);
        bad_s[l] = (!(M > NEG_MASKED) || !(M < INFINITY) || !isfinite(St)) ? 1 : 0;
    }
    __syncthreads();
    float Lh[N], Ll[N];
#pragma unroll
    for (int l = 0; l < N; ++l) {
        Lh[l] = (float)lse_s[l];
        Ll[l] = (float)(lse_s[l] - (double)Lh[l]);
    }

    // ---- pass 2: every pair at once (p2_accum)
    double dacc[NP], kacc[NP];
    int kinf = 0;
#pragma unroll
    for (int q = 0; q < NP; ++q) { dacc[q] = 0.0; kacc[q] = 0.0; }
    pool_stream<Tin, N>(rows, V, tid, [&](const float (&x)[N][VEC]) {
        p2_accum<N, VEC, NP>(x, Lh, Ll, dacc, kacc, kinf);
    });
#pragma unroll
    for (int q = 0; q < NP; ++q) {
        const double d = warp_sum_d(dacc[q]), kk = warp_sum_d(kacc[q]);
        if (lane == 0) { red[N + 2 * q][warp] = d; red[N + 2 * q + 1][warp] = kk; }
    }
    int kinf_all = __reduce_or_sync(0xffffffffu, kinf);
    __shared__ int kinf_s[PNW];
    if (lane == 0) kinf_s[warp] = kinf_all;
    __syncthreads();
    if (tid < NP) {
        const int q = tid;
        int i = 0, j = 1, c = 0;
        for (int a = 0; a < N; ++a)
            for (int bb = a + 1; bb < N; ++bb, ++c)
                if (c == q) { i = a; j = bb; }
        double D = 0.0, Kn = 0.0;
        int inf = 0;
        for (int w = 0; w < PNW; ++w) {
            D += red[N + 2 * q][w];
            Kn += red[N + 2 * q + 1][w];
            inf |= (kinf_s[w] >> q) & 1;
        }
        const bool bad = bad_s[i] || bad_s[j];
        double dtv = 0.5 * D;
        double kl = inf ? INFINITY : Kn;
        if (bad) { dtv = NAN; kl = NAN; }
        const size_t o = ((size_t)q * p.B + b) * p.K + k;
        if (p.pos_dtv) p.pos_dtv[o] = (float)dtv;
        if (p.pos_kl) p.pos_kl[o] = (float)kl;
        if (p.stats && !bad) {
            msd_pair_stats* st = p.stats + q;
            const double dc = dtv < 0 ? 0 : (dtv > 1 ? 1 : dtv);
            atomicAdd((unsigned long long*)&st->dtv_fx, (unsigned long long)llrint(dc * MSD_DTV_SCALE));
            if (inf) atomicAdd((unsigned long long*)&st->kl_inf, 1ull);
            else {
                const double kc = kl < 0 ? 0 : (kl > 1048576.0 ? 1048576.0 : kl);
                atomicAdd((unsigned long long*)&st->kl_fx, (unsigned long long)llrint(kc * MSD_KL_SCALE));
            }
            atomicAdd((unsigned long long*)&st->positions, 1ull);
        }
        if (bad && p.flags) atomicOr(&p.flags[b], (uint32_t)MSD_F_NONFINITE);
        if (inf && p.flags) atomicOr(&p.flags[b], (uint32_t)MSD_F_KL_INF);
    }
}

cudaError_t launch_pool(const PoolParams& p, int bf16, cudaStream_t s) {
    const int64_t grid = (int64_t)p.B * p.K;
    if (grid == 0) return cudaSuccess;
#define MSD_POOL(TY, NN) \
    if (p.N == NN) { pool_kernel<TY, NN><<<(unsigned)grid, PT, 0, s>>>(p); return cudaGetLastError(); }
    if (bf16) {
        MSD_POOL(__nv_bfloat16, 2) MSD_POOL(__nv_bfloat16, 3) MSD_POOL(__nv_bfloat16, 4)
    } else {
        MSD_POOL(float, 2) MSD_POOL(float, 3) MSD_POOL(float, 4)
    }
#undef MSD_POOL
    return cudaErrorInvalidValue;
}

}  // namespace msd
