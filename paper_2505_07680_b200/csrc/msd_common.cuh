// msd_common.cuh -- shared device helpers of libmsd (sm_100a only).
//
// Tiling used by every kernel: a "slice" is VS = T * ET consecutive vocabulary
// entries of one logit row; thread t of a T-thread CTA owns the elements
// (j * T + t) * VEC + k (j < ET/VEC, k < VEC) of the slice, i.e. 16-byte vectors
// with the warp covering 512 contiguous bytes per access (conflict-free LDS.128,
// fully coalesced LDG.128).
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/msd.h"

namespace msd {

constexpr int T = 256;             // threads per CTA (core and tail)
constexpr int NWARP = T / 32;
constexpr int ET = 16;             // elements per thread per row per slice
constexpr int VS = T * ET;         // slice length (4096 vocabulary entries)
constexpr int MAXL = 4;            // chain levels supported
constexpr int MAXC = 32;           // candidate slots (K + L - 1 <= 31)
constexpr float NEG_CLAMP = -1e30f;  // logits are clamped to >= this (NaN kept)
constexpr float NEG_MASKED = -1e29f; // clamped logits <= this mean "-inf" (p = 0)
constexpr float LOG2E = 1.4426950408889634f;
constexpr double KL_INF_THRESH = 1e20;
constexpr int CNT_STRIDE = 64;      // uint32 elements between unit counters (256 B)

// Per (unit, level, slice) pass-1 record, published for the cross-CTA exchange.
struct Partial {
    float m;        // slice max (after the -1e30 clamp)
    int32_t amax;   // first index (global vocab id) attaining m in the slice
    double S;       // sum_v exp(z_v - m) over the slice
    double Kl;      // sum_v exp(z_v - m) * (z_v - z'_v), z' = previous level's row
};

// Per (unit, level) result written by the combining CTA.
struct RowStat {
    double M;       // row max
    double S;       // sum_v exp(z_v - M)
    double lse;     // M + log S   (Eq. 1 normaliser)
    int32_t amax;   // argmax, lowest id on ties
    int32_t bad;    // NaN / +inf present or row all -inf
};

// Slice geometry of a vocabulary of V entries: C slices of VSe (<= VS) entries.  The core
// kernel gives each CTA two adjacent slices (bf16) per item, so a unit occupies ceil(C / 2)
// CTAs; C is the value in [ceil(V/VS), 5/4 ceil(V/VS)] for which k = floor(148 / ceil(C/2))
// groups keep the most SMs busy (an even C on ties: no half-empty CTA).  A group owns whole
// units, so units never straddle rounds and the groups never wait on each other (msd_core.cu).
struct SliceGeom {
    int32_t C;
    int32_t VSe;
};
constexpr int REF_SMS = 148;   // B200
__host__ __device__ inline int32_t geom_used_sms(int32_t c) {
    const int32_t cc = (c + 1) / 2;
    return (REF_SMS / cc) * cc;
}
__host__ __device__ inline SliceGeom slice_geometry(int64_t V) {
    const int32_t cmin = (int32_t)((V + VS - 1) / VS);
    int32_t best = cmin, used = geom_used_sms(cmin);
    for (int32_t c = cmin + 1; c <= cmin + cmin / 4 && c <= 2 * REF_SMS; ++c) {
        const int32_t u = geom_used_sms(c);
        if (u > used || (u == used && (best & 1) && !(c & 1))) { used = u; best = c; }
    }
    SliceGeom g;
    g.C = best;
    g.VSe = (int32_t)(((V + best - 1) / best + 7) / 8 * 8);
    return g;
}

// Exact-draw work sharing inside the tail kernel (msd_tail.cu): a request that needs an exact
// float64 draw posts a job; CTAs that finished their own request claim its chunks (normaliser
// chunks of the row pair, then slice masses).  Reset by the core kernel before every tail.
constexpr int EXJ_MAX = 32;        // concurrent jobs (more: the requester works alone)
constexpr int EXJ_NCH = 16;        // normaliser chunks per job
constexpr int EXJ_SPC = 4;         // slices per slice-mass chunk
constexpr int EXJ_MAXS = 128;      // slices per job (= the tail's MAXSLICES)
struct ExactJob {
    const void* ra;
    const void* rb;
    double Ma, Mb, A, B;
    int64_t V;
    int32_t resid, C, vse, chunk;
    uint32_t phase;                // 0 free / being filled, 1 normalisers, 2 slice masses, 3 done
    uint32_t next1, done1, next2, done2;
    uint32_t pad[5];
};
struct JobBoard {
    uint32_t alloc, started, finished, next;   // next: the tail's request counter (persistent grid)
    ExactJob job[EXJ_MAX];
    double part1[EXJ_MAX][EXJ_NCH][2];
    double part2[EXJ_MAX][EXJ_MAXS];
};

// Workspace layout (bytes), shared by host and device code.
struct WsLayout {
    size_t hdr, cnt, ready, partials, partms, rowstat, kl, resid, board, total;
    int32_t U, C, L;
};

__host__ __device__ inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
__host__ __device__ inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

__host__ __device__ inline WsLayout ws_layout(int32_t L, int32_t B, int32_t K, int64_t V) {
    WsLayout w;
    w.L = L;
    w.U = B * K;
    w.C = slice_geometry(V).C;
    size_t off = 0;
    w.hdr = off;      off += 256;
    // one counter per 256-byte block: concurrent units' counters must not share an L2 line
    w.cnt = off;      off = align_up(off + CNT_STRIDE * sizeof(uint32_t) * (size_t)w.U, 256);
    w.ready = off;    off = align_up(off + sizeof(uint32_t) * (size_t)w.U, 256);
    w.partials = off; off = align_up(off + sizeof(Partial) * (size_t)w.U * L * w.C, 256);
    w.partms = off;   off = align_up(off + sizeof(float2) * (size_t)w.U * L * w.C, 256);
    w.rowstat = off;  off = align_up(off + sizeof(RowStat) * (size_t)w.U * L, 256);
    w.kl = off;       off = align_up(off + sizeof(double) * (size_t)w.U * (L - 1), 256);
    w.resid = off;    off = align_up(off + sizeof(double) * (size_t)w.U * (L - 1) * w.C, 256);
    w.board = off;    off = align_up(off + sizeof(JobBoard), 256);
    w.total = off;
    return w;
}

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ float ex2f(float x) {
    float r;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ uint32_t max_nan_bf16x2(uint32_t a, uint32_t b) {
    uint32_t r;
    asm("max.NaN.bf16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
    return r;
}
__device__ __forceinline__ float max_nan_f32(float a, float b) {
    float r;
    asm("max.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t* p) {
    uint32_t r;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(r) : "l"(p) : "memory");
    return r;
}
__device__ __forceinline__ void st_release_u32(uint32_t* p, uint32_t v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint64_t globaltimer() {
    uint64_t r;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(r));
    return r;
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
    uint32_t done;
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return done != 0;
}
// try_wait with a suspend-time hint: the warp sleeps in hardware until the phase completes
// (or ~1 ms passes) instead of re-issuing the probe -- spinning warps steal issue slots
__device__ __forceinline__ bool mbar_try_wait_sleep(uint64_t* bar, uint32_t parity) {
    uint32_t done;
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3; selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity), "r"(1000000u)
        : "memory");
    return done != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    while (!mbar_try_wait_sleep(bar, parity)) {
    }
}
// 1-D bulk copy global -> shared (TMA engine, SASS UBLKCP), completes on `bar`.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                         uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], "
        "%2, [%3], %4;" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}
// fire-and-forget request of [src, src + bytes) into L2 (no shared memory, no barrier)
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_normal() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
    return p;
}

// ------------------------------------------------------------------ element access
template <typename Tin>
struct Elem;
template <>
struct Elem<float> {
    static constexpr int VEC = 4;
    __device__ static inline float load1(const float* p) { return __ldg(p); }
};
template <>
struct Elem<__nv_bfloat16> {
    static constexpr int VEC = 8;
    __device__ static inline float load1(const __nv_bfloat16* p) {
        return __bfloat162float(__ldg(p));
    }
};

__device__ __forceinline__ float bf16lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf16hi(uint32_t w) { return __uint_as_float(w & 0xffff0000u); }

// Unpack one 16-byte vector into VEC floats with the NaN-propagating -1e30 clamp.
template <typename Tin>
__device__ __forceinline__ void unpack_clamped(const uint4& v, float* x);
template <>
__device__ __forceinline__ void unpack_clamped<__nv_bfloat16>(const uint4& v, float* x) {
    // -1e30 as bf16x2 pair: 0xF149 (bf16 of -1e30 rounds to -9.98e29)
    const uint32_t c = 0xF149F149u;
    uint32_t a = max_nan_bf16x2(v.x, c), b = max_nan_bf16x2(v.y, c);
    uint32_t d = max_nan_bf16x2(v.z, c), e = max_nan_bf16x2(v.w, c);
    x[0] = bf16lo(a); x[1] = bf16hi(a); x[2] = bf16lo(b); x[3] = bf16hi(b);
    x[4] = bf16lo(d); x[5] = bf16hi(d); x[6] = bf16lo(e); x[7] = bf16hi(e);
}
template <>
__device__ __forceinline__ void unpack_clamped<float>(const uint4& v, float* x) {
    x[0] = max_nan_f32(__uint_as_float(v.x), NEG_CLAMP);
    x[1] = max_nan_f32(__uint_as_float(v.y), NEG_CLAMP);
    x[2] = max_nan_f32(__uint_as_float(v.z), NEG_CLAMP);
    x[3] = max_nan_f32(__uint_as_float(v.w), NEG_CLAMP);
}

__device__ __forceinline__ float clamp1(float z) { return max_nan_f32(z, NEG_CLAMP); }

// ------------------------------------------------------------------ warp reductions
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ int warp_min_i(int v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// exp(x) in float64 for x <= 0 on the FMA/ALU pipes only (no MUFU, no F2I/FRND: the
// MUFU pipe is saturated by the streaming ex2 of the pass-1 warps).  Relative error ~2e-16.
// 2^(x log2 e) = 2^n * e^(f ln 2), n = rint via the 1.5*2^52 magic, |f| <= 1/2.
__device__ __forceinline__ double dexp_neg(double x) {
    if (!(x > -700.0)) return 0.0;
    const double magic = 6755399441055744.0;
    const double y = x * 1.4426950408889634074;
    const double ym = y + magic;
    const double n = ym - magic;
    const double t = (y - n) * 0.69314718055994530942;     // |t| <= 0.347
    double r = 2.0876756987868098979e-09;                   // 1/12!
    r = fma(r, t, 2.5052108385441718775e-08);
    r = fma(r, t, 2.7557319223985890653e-07);
    r = fma(r, t, 2.7557319223985890653e-06);
    r = fma(r, t, 2.4801587301587301587e-05);
    r = fma(r, t, 1.9841269841269841270e-04);
    r = fma(r, t, 1.3888888888888888889e-03);
    r = fma(r, t, 8.3333333333333333333e-03);
    r = fma(r, t, 4.1666666666666666667e-02);
    r = fma(r, t, 1.6666666666666666667e-01);
    r = fma(r, t, 0.5);
    r = fma(r, t, 1.0);
    r = fma(r, t, 1.0);
    const int ni = __double2loint(ym);                      // n as a two's-complement int
    return r * __hiloint2double((ni + 1023) << 20, 0);
}

// float -> double on the integer pipe (no F2F: conversions share the XU pipe with MUFU).
// Exact for normal floats, zero and +-inf/NaN; float denormals flush to zero.
__device__ __forceinline__ double f2d_alu(float f) {
    const uint32_t b = __float_as_uint(f);
    const uint32_t e = (b >> 23) & 0xffu;
    const uint32_t sign = b & 0x80000000u;
    if (e == 0u) return __hiloint2double((int)sign, 0);
    const uint32_t m = b & 0x7fffffu;
    const uint32_t e64 = (e == 0xffu) ? 0x7ffu : (e + 896u);
    return __hiloint2double((int)(sign | (e64 << 20) | (m >> 3)), (int)(m << 29));
}
// double -> float by mantissa truncation on the integer pipe (normal range only); used to
// split a double into hi + lo floats where hi + lo reproduces it to ~2^-48.
__device__ __forceinline__ float d2f_trunc_alu(double d) {
    const uint32_t hi = (uint32_t)__double2hiint(d), lo = (uint32_t)__double2loint(d);
    const int e = (int)((hi >> 20) & 0x7ffu) - 1023 + 127;
    if (e <= 0) return 0.f;
    if (e >= 255) return __uint_as_float((hi & 0x80000000u) | 0x7f800000u);
    return __uint_as_float((hi & 0x80000000u) | ((uint32_t)e << 23) | ((hi & 0xfffffu) << 3) | (lo >> 29));
}

// 1/x in float64 for x > 0 with FMA-pipe Newton iterations only (no MUFU.RCP64H).
__device__ __forceinline__ double drcp_fma(double x) {
    double y = __longlong_as_double(0x7FDE623822FC16E6LL - __double_as_longlong(x));   // ~10% guess
#pragma unroll
    for (int it = 0; it < 5; ++it) y = y * fma(-x, y, 2.0);
    return y;
}

// 1/x in float32 (x > 0, normal) with FMA-pipe Newton iterations only (no MUFU.RCP).
__device__ __forceinline__ float frcp_fma(float x) {
    float y = __int_as_float(0x7EF311C3 - __float_as_int(x));   // ~12% initial guess
#pragma unroll
    for (int it = 0; it < 4; ++it) y = y * fmaf(-x, y, 2.0f);
    return y;
}

// 2^x in float32 for x <= 0 on the FMA/ALU pipes only (relative error ~1e-7).
__device__ __forceinline__ float exp2f_fma(float x) {
    if (!(x > -126.f)) return 0.f;
    const float magic = 12582912.f;                         // 1.5 * 2^23
    const float xm = x + magic;
    const float n = xm - magic;
    const float t = (x - n) * 0.69314718056f;              // |t| <= 0.347
    float r = 1.98412698e-4f;                               // 1/7!
    r = fmaf(r, t, 1.38888889e-3f);
    r = fmaf(r, t, 8.33333333e-3f);
    r = fmaf(r, t, 4.16666667e-2f);
    r = fmaf(r, t, 1.66666667e-1f);
    r = fmaf(r, t, 0.5f);
    r = fmaf(r, t, 1.0f);
    r = fmaf(r, t, 1.0f);
    const int ni = __float_as_int(xm) - 0x4B400000;         // n
    return r * __int_as_float((ni + 127) << 23);
}

// 2^x for a pair of x <= 0 on the FMA pipe with packed f32x2 ops, branch-free: x clamped at
// -127 (-> exactly 0, like ex2.approx.ftz; a NaN x gives 0, so callers detect NaN elsewhere), n = rint(x) by the 1.5*2^23 magic, degree-6
// Taylor polynomial of e^(t), t = (x - n) ln 2, |t| <= 0.347 (truncation 1.2e-7 relative).
__device__ __forceinline__ float2 exp2_pair_fma(float2 x) {
    x.x = fmaxf(x.x, -127.f);
    x.y = fmaxf(x.y, -127.f);
    const float2 magic = make_float2(12582912.f, 12582912.f);
    const float2 xm = __fadd2_rn(x, magic);
    const float2 n = __fadd2_rn(xm, make_float2(-12582912.f, -12582912.f));
    const float2 ln2 = make_float2(0.69314718056f, 0.69314718056f);
    const float2 t = __fmul2_rn(__fadd2_rn(x, make_float2(-n.x, -n.y)), ln2);
    float2 r = make_float2(1.38888889e-3f, 1.38888889e-3f);                  // 1/6!
    r = __ffma2_rn(r, t, make_float2(8.33333333e-3f, 8.33333333e-3f));
    r = __ffma2_rn(r, t, make_float2(4.16666667e-2f, 4.16666667e-2f));
    r = __ffma2_rn(r, t, make_float2(1.66666667e-1f, 1.66666667e-1f));
    r = __ffma2_rn(r, t, make_float2(0.5f, 0.5f));
    r = __ffma2_rn(r, t, make_float2(1.0f, 1.0f));
    r = __ffma2_rn(r, t, make_float2(1.0f, 1.0f));
    const int nx = __float_as_int(xm.x) - 0x4B400000, ny = __float_as_int(xm.y) - 0x4B400000;
    return __fmul2_rn(r, make_float2(__int_as_float((nx + 127) << 23), __int_as_float((ny + 127) << 23)));
}

// Combine C slice partials of one row into its RowStat (fixed order -> every CTA
// that does it gets bit-identical results).  Executed by one full warp.  The slice KL
// numerators K_s = sum_{v in s} e^{z_v - m_s} (z_v - z'_v) (raw logit differences) are
// rescaled to the row maximum in float64: K = sum_s K_s e^{m_s - M}.
__device__ inline RowStat combine_row(const Partial* parts, int C, double* K_out, double sc = 1.0) {
    const int lane = threadIdx.x & 31;
    float m = -INFINITY;
    for (int s = lane; s < C; s += 32) m = fmaxf(m, parts[s].m);
    m = warp_max(m);
    double S = 0.0, Kl = 0.0;
    int am = 0x7fffffff;
    bool bad = false;
    for (int s = lane; s < C; s += 32) {
        float ms = parts[s].m;
        double Ss = parts[s].S;
        double f = dexp_neg(((double)ms - (double)m) * sc);   // sc = 1 / temperature
        S += Ss * f;
        Kl += parts[s].Kl * f;
        if (ms == m) am = min(am, parts[s].amax);
        if (isnan(ms) || isnan(Ss)) bad = true;
    }
    S = warp_sum_d(S);
    Kl = warp_sum_d(Kl);
    am = warp_min_i(am);
    bad = __any_sync(0xffffffffu, bad);
    RowStat r;
    r.M = (double)m;
    r.S = S;
    r.lse = (double)m * sc + log(S);        // scaled units
    r.amax = am == 0x7fffffff ? 0 : am;
    r.bad = (bad || !(m > NEG_MASKED) || !isfinite(S) || !(m < INFINITY)) ? 1 : 0;
    if (K_out) *K_out = Kl;
    return r;
}

}  // namespace msd
