// msd_core.cu -- the streaming pass over every logit row at the draft positions.
//
// Rows a1 (Eq. 1 normaliser) and a5 (Eq. 5 DTV; KL) of the
// hot path, for all L chain levels at once so every logit byte is read from HBM
// exactly once.
//
// Decomposition.  A *unit* is one (request b, draft position i < K) and owns the L rows
// Z_l[b, i, :].  The vocabulary is cut into C tail slices of VSe <= VS = 4096 entries (the
// granularity of the records the tail kernel combines and rescans); an *item* is one unit's
// NH = 2 adjacent tail slices (bf16; 1 for f32): a ring row holds them in two halves of VS
// entries, copied by two 1-D bulk copies (TMA).  The kernel is persistent and cooperative (one
// CTA per SM) and runs k = floor(148 / Cc) groups of Cc = ceil(C / NH) CTAs: CTA (g, s) takes
// core slice s of units g, g + k, ..., so a unit's items run concurrently on Cc SMs, which
// exchange per-slice (max, sum) records through global memory (L2).
//
// Two passes per item; pass 2 needs the row normalisers, i.e. the records of all C slices,
// so an item stays on chip from its arrival until the exchange completes (several
// microseconds under full HBM load).  Two kinds of item keep it on chip:
//   T items  pass 1 parks the exponentials e in TMEM (fp32) and releases the ring stage at
//            once; pass 2 reads e back (tcgen05.ld) -- no recomputation.
//   R items  pass 1 keeps the ring stage (bf16, half the bytes of e); pass 2 recomputes e
//            from it (one more MUFU.EX2 per element) and releases the stage.
// Of every pat_p items the first pat_t are T items (host-chosen).
//
// Exponent reference: the warp maximum of each row over the warp's region (the dominant
// entries then have |z - m| small, so the fp32 exponent argument keeps full relative accuracy;
// a fixed reference such as the first logit was measured to break the KL tolerance).
//
// Warp roles (low warp ids first: the latency-critical ones; 28 warps, 72 registers):
//   producer  (warp 0)  TMA bulk copies of the L row halves into the S-stage ring.
//   publisher (warp 1)  folds the pass-1 warp records into one record per (row, tail slice)
//                       and publishes it (exchange record first, then the tail's Partial).
//   fetcher   (warp 2)  polls the unit's L x C records, combines them into the row
//                       normalisers relative to this CTA's first slice, and derives the pass-2
//                       factors of every (row, region).
//   reducer   (warp 3)  folds the pass-2 records into the per-slice residuals R_s.
//   pass 2    (8 warps) per-region residual sum max(e_l - rho e_{l-1}, 0) of every adjacent
//                       pair -- this slice's share of DTV (Eq. 5) and of the residual CDF.
//   pass 1    (2 x 8)   two groups take alternate items; warp r of a group owns the contiguous
//                       1024-entry region r of the item (regions past a slice's end idle):
//                       y = z - m with the mixed-precision add.f32.bf16 (no unpacking),
//                       e = 2^(y log2 e) on the MUFU, the sum of e and the KL numerator
//                       sum e_l (z_l - z_{l-1}) of the raw logit differences in packed fp32.
#include "msd_common.cuh"
#include "msd_internal.h"

#include <algorithm>
#include <cstdlib>

namespace msd {

constexpr int NCW = 8;                 // pass-1 warps = element regions of an item
#ifndef MSD_P2W
#define MSD_P2W 8
#endif
constexpr int NCW2 = MSD_P2W;          // pass-2 warps: warp v handles regions v, v + NCW2, ...
constexpr int NPR = NCW / NCW2;        // regions per pass-2 warp
constexpr int CET = 32;                // elements per pass-1 thread per row
constexpr int WCH = CET * 32;          // contiguous entries per region (1024)
constexpr int HREG = VS / WCH;         // regions per half (4): half h = tail slice 2 s + h
constexpr int TCOLS = 256;             // TMEM columns per region (2 regions per lane quadrant)
#ifndef MSD_NFETCH
#define MSD_NFETCH 1
#endif
#ifndef MSD_POLL_NS
#define MSD_POLL_NS 64                 // fetcher back-off between polls of the exchange records
#endif
constexpr int NFETCH = MSD_NFETCH;
// Warp numbering: latency-critical service warps first, then pass 2, then the throughput
// warps (pass 1).  Pass-1 warp W_P1 + r owns region r in TMEM lane quadrant r % 4; pass-2
// warp W_P2 + v serves regions v and v + 4 (quadrant v): both bases are multiples of 4.
constexpr int W_PROD = 0, W_PUB = 1, W_FETCH0 = 2, W_RED = W_FETCH0 + NFETCH;
constexpr int W_P2 = (W_RED + 1 + 3) / 4 * 4, W_P1 = W_P2 + NCW2;   // (4 with one fetcher: 28 warps, 72 registers)
#ifndef MSD_SPLIT
#define MSD_SPLIT 1                    // 2: all 16 pass-1 warps on every item, two per region
#endif
constexpr int NSPLIT = MSD_SPLIT;      // pass-1 warps per region of an item
constexpr int NG1 = 2 / NSPLIT;        // pass-1 warp groups: group g processes items j = g mod NG1
constexpr int NW1 = NCW * NSPLIT;      // pass-1 warps per item
constexpr int CORE_THREADS = (W_P1 + NG1 * NW1) * 32;
static_assert(W_RED < W_P2 && W_P2 % 4 == 0 && W_P1 % 4 == 0 && NCW % NCW2 == 0 && NCW2 % 4 == 0, "warp roles");
constexpr int SMAX = 14;               // ring stages (upper bound)
constexpr int NQ = 16;                 // per-item record slots (references, pass-2 factors)
constexpr int NTMAX = 8;               // TMEM item slots (upper bound)
constexpr int FBUF = 192;              // records per fetcher staging buffer (L * C <= 192)
constexpr int SMEM_BUDGET = 227 * 1024;
constexpr int R1 = 4, R2 = 4;          // pass-1 / pass-2 record rings (powers of two)
constexpr int NSUB = 4;                // per-warp pass-2 records after a 3-step shuffle fold (lanes 0..3)
constexpr int NSUB1 = 4;               // per-warp pass-1 records after a 3-step shuffle fold (lanes
                                       // 0..3): the publisher sums them in float64 (KL / LSE precision)
static_assert(NCW == 2 * HREG, "two halves of HREG regions");

struct WF {                // pass-2 factors of one (row, warp) of the current slice
    float rho;             // rho = c_b S_a / (S_b c_a)  (pair ending at this row)
    float scale;           // c_a / S_a
};
template <int L>
struct Ctl {
    uint64_t full[SMAX], empty[SMAX];
    uint64_t r1_full[R1], r1_empty[R1], r2_full[R2], r2_empty[R2];
    uint64_t rowf_full[NQ], rowf_empty[NQ];
    uint64_t tm_full[NTMAX], tm_empty[NTMAX];  // TMEM item slots: pass-1 warps -> pass-2 warps
    uint64_t pub[NQ];                       // this CTA's slice record of item j is published
    uint32_t p1cnt[R1];                     // pass-1 warps done with the item of a record slot
    uint32_t taddr;
    float wmx[NQ][L][NW1];                  // per-warp max of each row, per item
    uint32_t clampw[NQ];                    // bit w: pass-1 warp w took the clamped path
    alignas(16) float r1S[R1][L][NW1][NSUB1];  // pass-1 partial sums
    alignas(16) float r1K[R1][L][NW1][NSUB1];  // pass-1 KL numerators sum e (z_l - z_{l-1})
    int r1A[R1][L][NW1];                    // greedy: first argmax index per warp
    WF rowf[NQ][L][NW1];
    float r2R[R2][L][NCW][NSUB];            // pass-2 residual partials per region (probability units)
    unsigned long long fbuf_pad;
    unsigned long long fbuf[NFETCH][FBUF];  // fetcher staging of a unit's records
};

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// relaxed load without a compiler memory clobber: independent loads stay in flight together
__device__ __forceinline__ unsigned long long ld_relaxed_u64_nc(const unsigned long long* p) {
    unsigned long long r;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(r) : "l"(p));
    return r;
}
__device__ __forceinline__ void st_relaxed_u64(unsigned long long* p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
// TMEM stores / loads of 8 consecutive columns (no "memory" clobber: TMEM is ordered by the
// tcgen05.wait / fence instructions, and arithmetic may be scheduled across these)
__device__ __forceinline__ void tm_st16(uint32_t ta, const float* v) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(ta),
        "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]), "f"(v[8]), "f"(v[9]),
        "f"(v[10]), "f"(v[11]), "f"(v[12]), "f"(v[13]), "f"(v[14]), "f"(v[15]));
}
__device__ __forceinline__ void tm_ld16(uint32_t ta, float* v) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7]), "=f"(v[8]),
          "=f"(v[9]), "=f"(v[10]), "=f"(v[11]), "=f"(v[12]), "=f"(v[13]), "=f"(v[14]), "=f"(v[15])
        : "r"(ta));
}
#ifndef MSD_PUB_LATE
#define MSD_PUB_LATE 1                 // this CTA's fetcher starts polling after the Partials too (0: earlier polling, measured 3 % slower)
#endif
#ifndef MSD_INLINE_PUB
#define MSD_INLINE_PUB 0               // 1: the last pass-1 warp of an item publishes its records (measured slower: 1.06 vs 1.00 ms)
#endif
#ifndef MSD_SPIN_SERVICE
#define MSD_SPIN_SERVICE 1
#endif
// latency-critical waits (publisher, fetchers, reducer, pass 2): a spinning probe, so the warp
// resumes as soon as the phase completes instead of after a suspended try_wait wakes it
__device__ __forceinline__ void mbar_wait_lat(uint64_t* bar, uint32_t parity) {
#if MSD_SPIN_SERVICE
    while (!mbar_try_wait(bar, parity)) {
    }
#else
    mbar_wait(bar, parity);
#endif
}

// non-blocking probe of a phase (no suspend)
__device__ __forceinline__ bool mbar_test_wait(uint64_t* bar, uint32_t parity) {
    uint32_t done;
    asm volatile(
        "{ .reg .pred p; mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return done != 0;
}
__device__ __forceinline__ void mbar_arrive_cnt(uint64_t* bar, uint32_t n) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(n) : "memory");
}
__device__ __forceinline__ void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tm_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ uint32_t clamp_bf16x2(uint32_t w) { return max_nan_bf16x2(w, 0xF149F149u); }

// warp max (NaN-propagating) in one instruction (CREDUX)
__device__ __forceinline__ float redux_max_nan(float v) {
    float r;
    asm("redux.sync.max.NaN.f32 %0, %1, 0xffffffff;" : "=f"(r) : "f"(v));
    return r;
}
__device__ __forceinline__ int redux_min_s32(int v) {
    int r;
    asm("redux.sync.min.s32 %0, %1, 0xffffffff;" : "=r"(r) : "r"(v));
    return r;
}
// bf16 half of a packed word plus an fp32 value, in fp32 (FHADD.BF16: no unpacking)
__device__ __forceinline__ float bf16lo_add(uint32_t w, float c) {
    float r;
    asm("{ .reg .b16 lo, hi; mov.b32 {lo, hi}, %1; add.rn.f32.bf16 %0, lo, %2; }" : "=f"(r) : "r"(w), "f"(c));
    return r;
}
__device__ __forceinline__ float bf16hi_add(uint32_t w, float c) {
    float r;
    asm("{ .reg .b16 lo, hi; mov.b32 {lo, hi}, %1; add.rn.f32.bf16 %0, hi, %2; }" : "=f"(r) : "r"(w), "f"(c));
    return r;
}
__device__ __forceinline__ uint32_t word_of(const uint4& r, int k) {
    return k == 0 ? r.x : k == 1 ? r.y : k == 2 ? r.z : r.w;
}

// fold a per-lane value into lanes 0..3 (lane k holds the sum over lanes == k mod 4)
__device__ __forceinline__ float fold4(float v) {
    v += __shfl_xor_sync(0xffffffffu, v, 16);
    v += __shfl_xor_sync(0xffffffffu, v, 8);
    v += __shfl_xor_sync(0xffffffffu, v, 4);
    return v;
}

// 2^x in float32 on the FMA/ALU pipes (no MUFU: its queue is full of pass-1 ex2); +inf
// above 2^127, 0 below 2^-126.
__device__ __forceinline__ float exp2f_fma_any(float x) {
    if (x > 127.f) return INFINITY;
    return exp2f_fma(x);
}

#ifndef MSD_CORE_NPOLY
#define MSD_CORE_NPOLY 0
#endif
constexpr int CORE_NPOLY = MSD_CORE_NPOLY;   // of every 4 exponential pairs, this many on the FMA pipe

__host__ __device__ constexpr int core_tslots(int L) { return TCOLS / (CET * L); }

// element index (within the slice) of vector jv of pass-1 thread (warp w, lane)
template <typename Tin>
__device__ __forceinline__ int vec_index(int w, int lane, int jv) {
    constexpr int VEC = Elem<Tin>::VEC;
    constexpr int NV = CET / VEC;
    return (w * NV + jv) * 32 * VEC + lane * VEC;
}

// The VEC-element vector that straddles the end of a row: the bulk-copied part from shared
// memory, the tail (< 16 bytes) from global memory, the pad value (~ -2.4e30) past the row.
template <typename Tin>
__device__ __noinline__ uint4 load_straddle(const Tin* sl, const Tin* g, int e0, int len_bulk, int len) {
    constexpr int VEC = Elem<Tin>::VEC;
    uint4 pv = make_uint4(0xF1F1F1F1u, 0xF1F1F1F1u, 0xF1F1F1F1u, 0xF1F1F1F1u);
    Tin xs[VEC];
    const Tin* pz = reinterpret_cast<const Tin*>(&pv);
#pragma unroll
    for (int k = 0; k < VEC; ++k) {
        const int ee = e0 + k;
        Tin z = pz[k];
        if (ee < len_bulk) z = sl[ee];
        else if (ee < len) z = g[ee];
        xs[k] = z;
    }
    return *reinterpret_cast<const uint4*>(xs);
}

// An item whose row length is not a whole number of 16-byte vectors: each pass-1 thread
// rewrites its own straddling vector of the ring stage from the ring and global memory, so
// the pass-1 loads stay unconditional.  Out of line.
template <typename Tin, int L, int NV>
__device__ __noinline__ void repair_stage(Tin* stage, int rs, const LevelDesc& lv, int64_t b, int64_t i,
                                          int64_t base, int w, int lane, int len_bulk, int len, int jv0, int jv1) {
    constexpr int VEC = Elem<Tin>::VEC;
    const int hoff = (w / HREG) * VS;            // this region's half of the ring row
    for (int l = 0; l < L; ++l) {
        Tin* sl = stage + (size_t)l * rs + hoff;
        for (int jv = jv0; jv < jv1; ++jv) {
            const int e0 = vec_index<Tin>(w, lane, jv) - hoff;
            if (e0 + VEC <= len_bulk || e0 >= len) continue;
            const uint4 v = load_straddle<Tin>(
                sl, reinterpret_cast<const Tin*>(lv.ptr[l]) + b * lv.bs[l] + i * lv.ld[l] + base, e0, len_bulk, len);
            *reinterpret_cast<uint4*>(sl + e0) = v;
        }
    }
    // these generic-proxy writes precede the next bulk copy (async proxy) into the stage
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// e = 2^((z - m) log2 e) of a 16-element chunk of one thread's elements of one row (y = z - m
// returned too); `clamp`: the -1e30 clamp first (-inf -> p = 0 without 0 * inf), NaN kept.
constexpr int CH = 16;
template <typename Tin>
__device__ __forceinline__ void row_exp(const uint4* raw, float m, bool clamp, float* e, float2* y, float l2s) {
    const float nm = -m;
    const float2 nm2 = make_float2(nm, nm);
    const float2 l2e = make_float2(l2s, l2s);     // log2(e) / temperature
#pragma unroll
    for (int pp = 0; pp < CH / 2; ++pp) {
        float2 yy;
        if (sizeof(Tin) == 2) {
            uint32_t w = word_of(raw[pp >> 2], pp & 3);
            if (clamp) w = clamp_bf16x2(w);
            yy = make_float2(bf16lo_add(w, nm), bf16hi_add(w, nm));
        } else {
            const uint4& r = raw[pp >> 1];
            float2 xv = (pp & 1) ? make_float2(__uint_as_float(r.z), __uint_as_float(r.w))
                                 : make_float2(__uint_as_float(r.x), __uint_as_float(r.y));
            xv.x = clamp1(xv.x);
            xv.y = clamp1(xv.y);
            yy = __fadd2_rn(xv, nm2);
        }
        const float2 t = __fmul2_rn(yy, l2e);
        if ((pp & 3) >= 4 - CORE_NPOLY) {              // this pair on the FMA pipe (MUFU relief)
            const float2 ee = exp2_pair_fma(t);
            e[2 * pp] = ee.x;
            e[2 * pp + 1] = ee.y;
        } else {
            e[2 * pp] = ex2f(t.x);
            e[2 * pp + 1] = ex2f(t.y);
        }
        y[pp] = yy;
    }
}

// e and y = z - m of quarter h (8 of the thread's 32 elements) of one row of a ring stage
template <typename Tin>
__device__ __forceinline__ void half_exp(const Tin* row, int rg, int lane, int h, float m, bool clamp, float* e,
                                         float2* y, float l2s) {
    constexpr int VEC = Elem<Tin>::VEC;
    constexpr int NVH = 8 / VEC;        // vectors per half: 1 (bf16) or 2 (f32)
    uint4 raw[NVH];
#pragma unroll
    for (int jv = 0; jv < NVH; ++jv)
        raw[jv] = *reinterpret_cast<const uint4*>(row + vec_index<Tin>(rg, lane, h * NVH + jv));
    const float nm = -m;
    const float2 nm2 = make_float2(nm, nm);
    const float2 l2e = make_float2(l2s, l2s);     // log2(e) / temperature
#pragma unroll
    for (int pp = 0; pp < 4; ++pp) {
        float2 yy;
        if (sizeof(Tin) == 2) {
            uint32_t w = word_of(raw[0], pp);
            if (clamp) w = clamp_bf16x2(w);
            yy = make_float2(bf16lo_add(w, nm), bf16hi_add(w, nm));
        } else {
            const uint4& r = raw[pp >> 1];
            float2 xv = (pp & 1) ? make_float2(__uint_as_float(r.z), __uint_as_float(r.w))
                                 : make_float2(__uint_as_float(r.x), __uint_as_float(r.y));
            xv.x = clamp1(xv.x);
            xv.y = clamp1(xv.y);
            yy = __fadd2_rn(xv, nm2);
        }
        const float2 t = __fmul2_rn(yy, l2e);
        if ((pp & 3) >= 4 - CORE_NPOLY) {              // this pair on the FMA pipe (MUFU relief)
            const float2 ee = exp2_pair_fma(t);
            e[2 * pp] = ee.x;
            e[2 * pp + 1] = ee.y;
        } else {
            e[2 * pp] = ex2f(t.x);
            e[2 * pp + 1] = ex2f(t.y);
        }
        y[pp] = yy;
    }
}
// ring-row index of element 2 pp (+1) of quarter h of pass-1 thread (rg, lane)
template <typename Tin>
__device__ __forceinline__ int half_index(int rg, int lane, int h, int pp) {
    constexpr int VEC = Elem<Tin>::VEC;
    constexpr int NVH = 8 / VEC;
    return vec_index<Tin>(rg, lane, h * NVH + (2 * pp) / VEC) + (2 * pp) % VEC;
}
__device__ __forceinline__ void tm_st8(uint32_t ta, const float* v) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(ta), "f"(v[0]),
                 "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]));
}

#ifdef MSD_PROF
#define PROF_DECL long long _pa[8] = {0, 0, 0, 0, 0, 0, 0, 0}; long long _pt = clock64(); long long _pn = 0;
#define PROF(k) { const long long _t = clock64(); _pa[k] += _t - _pt; _pt = _t; }
#define PROF_ITEM ++_pn;
#define PROF_FLUSH(role) if (p.trace && lane == 0) { for (int _k = 0; _k < 8; ++_k) { atomicAdd(p.trace + (role) * 16 + _k, (unsigned long long)_pa[_k]); atomicAdd(p.trace + 128 + ((size_t)blockIdx.x * 8 + (role)) * 16 + _k, (unsigned long long)_pa[_k]); } atomicAdd(p.trace + (role) * 16 + 15, (unsigned long long)_pn); atomicAdd(p.trace + 128 + ((size_t)blockIdx.x * 8 + (role)) * 16 + 15, (unsigned long long)_pn); }
#else
#define PROF_DECL
#define PROF(k)
#define PROF_ITEM
#define PROF_FLUSH(role)
#endif

// Incremental ring / pattern position of item j (no runtime integer division in the loops:
// it would issue on the busy MUFU pipe).
struct Cursor {
    int j = 0;
    int st = 0, sph = 0;           // ring stage, its phase parity
    int pr = 0;                    // position within the item pattern period
    int q = 0, tph = 0, tj = 0;    // TMEM slot of the next T item, its phase parity, T-item count
    __device__ __forceinline__ bool isT(int PT) const { return pr < PT; }
    __device__ __forceinline__ void next(int S, int PP, int PT, int NT) {
        if (pr < PT) {
            ++tj;
            if (++q == NT) { q = 0; tph ^= 1; }
        }
        if (++pr == PP) pr = 0;
        if (++st == S) { st = 0; sph ^= 1; }
        ++j;
    }
};

// LSE: producer-supplied row normalisers (msd_chain_verify_lse), a separate instantiation so the
// exchange path's register allocation is untouched
template <typename Tin, int L, bool GREEDY, bool LSE>
__global__ void __launch_bounds__(CORE_THREADS, 1) core_kernel(CoreParams p) {
    constexpr int VEC = Elem<Tin>::VEC;
    constexpr int NV = CET / VEC;           // 2 (bf16) or 4 (f32) vectors per thread and row
    constexpr int ES = (int)sizeof(Tin);
    constexpr int NT = core_tslots(L);      // TMEM item slots
    static_assert(NT <= NTMAX && NT >= 2, "item slots");
    extern __shared__ __align__(128) unsigned char smem[];
    Ctl<L>& c = *reinterpret_cast<Ctl<L>*>(smem);
    Tin* ring = reinterpret_cast<Tin*>(smem + align_up(sizeof(Ctl<L>), 128));

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int C = p.C;
    const int VSe = p.VSe;
    // temperature T (logits processor): every exponent is (z - m) / T, sc = 1 / T.  Records
    // and Partials keep raw maxima (the tail scales its exponents the same way); the Partials' KL
    // numerator is sum e (z_l - z_{l-1}) / T.
    const float sc = p.inv_temp, l2s = LOG2E * p.inv_temp;
    const int RS = p.rs;                    // ring row stride (entries)
    const int S = p.stages;
    const int PP = p.pat_p, PT = p.pat_t;
    // An item is NH (2 for bf16, 1 for f32) consecutive tail slices t = NH s + h of one unit:
    // the ring row holds them in halves of VS entries, region w (1024 entries) lies in half
    // w / HREG.  Group scheduling: the grid is k groups of Cc = ceil(C / NH) CTAs; CTA (group, s)
    // handles core slice s of units group, group + k, ... -- a unit's slices always run
    // together on one group.
    constexpr int NH = ES == 2 ? 2 : 1;
    const int Cc = (C + NH - 1) / NH;
    const int kgrp = gridDim.x / Cc;
    // With one CTA on every SM (1024 threads x 64 registers: never two per SM) the SM id is a
    // permutation of the CTA ids; grouping by SM id keeps a group's exchange among neighbouring
    // SMs (measured: core 1.1455 -> 1.1412 ms on Llama-3; interleaved groups 1.1444 ms)
    int vcta = blockIdx.x;
    {
        uint32_t smid, nsmid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        asm volatile("mov.u32 %0, %%nsmid;" : "=r"(nsmid));
        if (nsmid == gridDim.x) vcta = (int)smid;
    }
    const int grp = vcta / Cc, sfix = vcta % Cc;
    const int n_my = grp < kgrp && grp < p.U ? (p.U - grp + kgrp - 1) / kgrp : 0;

    // this CTA's tail slices t_h = NH s + h are the same for all its items, so are their
    // lengths: the tail [len_bulk_h, VS) of every half row is never written by the bulk copies
    // -- the pad value (~ -2.4e30) once, so every active warp loads whole vectors
    // unconditionally (and the last slice of a row needs no second copy)
    const int s = sfix;
    int64_t hbase[NH];
    int hlen[NH], hbulk[NH];
    uint32_t amask = 0;                     // bit w: region w holds data
#pragma unroll
    for (int h = 0; h < NH; ++h) {
        const int t = NH * s + h;
        hbase[h] = (int64_t)t * VSe;
        hlen[h] = t < C ? (int)max((int64_t)0, min((int64_t)VSe, p.V - hbase[h])) : 0;
        hbulk[h] = (hlen[h] * ES) / 16 * 16 / ES;
        for (int r = 0; r < HREG; ++r)
            if (r * WCH < hlen[h]) amask |= 1u << (h * HREG + r);
    }
    const int nact = __popc(amask);         // regions (pass-1 warps, pass-2 warps) with data
    const int np2 = nact;
    {
        uint32_t* r32 = reinterpret_cast<uint32_t*>(ring);
        for (int h = 0; h < NH; ++h) {
            const int w0 = (h * VS + hbulk[h]) * ES / 4, w1 = (h + 1) * VS * ES / 4;
            const int per_row = w1 - w0;
            for (int e = tid; e < S * L * per_row; e += blockDim.x) {
                const int row = e / per_row;
                r32[(size_t)row * (RS * ES / 4) + w0 + (e - row * per_row)] = 0xF1F1F1F1u;
            }
        }
    }
    if (warp == W_PROD) {
        if (lane == 0) {
            // empty: one arrival per region (pass-1 warps for T items, pass-2 warps for R items)
            // a T item's stage is released by its NSPLIT * nact pass-1 warps, an R item's by the
            // nact pass-2 warps (NSPLIT arrivals each)
            for (int s = 0; s < S; ++s) { mbar_init(&c.full[s], 1); mbar_init(&c.empty[s], nact * NSPLIT); }
            for (int r = 0; r < R1; ++r) { mbar_init(&c.r1_full[r], nact * NSPLIT); mbar_init(&c.r1_empty[r], 1); }
            for (int r = 0; r < R2; ++r) { mbar_init(&c.r2_full[r], np2); mbar_init(&c.r2_empty[r], 1); }
            for (int k = 0; k < NQ; ++k) {
                mbar_init(&c.rowf_full[k], 1);
                mbar_init(&c.rowf_empty[k], np2);
                mbar_init(&c.pub[k], LSE ? (uint32_t)(nact * NSPLIT) : 1u);
            }
            for (int q = 0; q < NT; ++q) { mbar_init(&c.tm_full[q], nact * NSPLIT); mbar_init(&c.tm_empty[q], np2); }
            fence_mbar_init();
        }
        __syncwarp();
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&c.taddr)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid < NQ) c.clampw[tid] = 0u;
    if (blockIdx.x == 0 && p.board) {       // the tail's exact-draw job board, for this call
        for (int t = tid; t < 4 + EXJ_MAX * (int)(sizeof(ExactJob) / 4); t += blockDim.x)
            reinterpret_cast<uint32_t*>(p.board)[t] = 0u;
    }
    if (tid < R1) c.p1cnt[tid] = 0u;
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");

    auto stamp = [&](int j, int k) {
#if defined(MSD_TRACE) && !defined(MSD_PROF)
        if (p.trace) p.trace[((int64_t)(grp + j * kgrp) * Cc + sfix) * 16 + k] = globaltimer();
#endif
    };
    auto item = [&](int j, int64_t& u, int64_t& b, int64_t& i) {
        const uint32_t uu = (uint32_t)(grp + j * kgrp);
        const uint32_t bb = __umulhi(uu, p.kinv);
        u = uu;
        b = bb;
        i = uu - bb * (uint32_t)p.K;
    };
    // TMEM column base of region w (lane quadrant w & 3, column block w >> 2)
    auto tcol = [&](int w) { return c.taddr + ((uint32_t)((w & 3) * 32) << 16) + (uint32_t)((w >> 2) * TCOLS); };

    // Publisher (one full warp; run by the last pass-1 warp of the item, or the publisher warp):
    // lane = 8 l + w: row l, region w (L <= 4).  Each lane sums its region's sub-records, scales
    // them by 2^((m_w - m_s) log2 e) relative to the tail slice's maximum m_s (1 when the region
    // holds the maximum) and the HREG lanes of each half reduce with 2 shuffle levels: one record
    // per (row, tail slice NH s + w / HREG).
    static_assert(NCW == 8 && HREG == 4 && L * NCW <= 32, "publisher lane layout");
    auto publish = [&](int j) {
        const int l = lane >> 3, w = lane & 7;
        const bool inrow = l < L;
        const bool act = inrow && ((amask >> w) & 1u);
        const int tslice = NH * s + w / HREG;   // this lane's tail slice
        int64_t u, b, i;
        item(j, u, b, i);
        const int k = j & (NQ - 1);
        const int r1 = j & (R1 - 1);
        // the NSPLIT pass-1 warps of region w (each with its own warp maximum)
        float Sh[NSPLIT], wmh[NSPLIT], cmh[NSPLIT];
        double Sdh[NSPLIT], Khd[NSPLIT];
        int ah[NSPLIT];
        float wm = -INFINITY;
#pragma unroll
        for (int h = 0; h < NSPLIT; ++h) {
            Sh[h] = cmh[h] = 0.f;
            Sdh[h] = Khd[h] = 0.0;
            wmh[h] = -INFINITY;
            ah[h] = 0x7fffffff;
            if (act) {
                const int wq = w + NCW * h;
                const float4 s4 = *reinterpret_cast<const float4*>(&c.r1S[r1][l][wq][0]);
                const float4 k4 = *reinterpret_cast<const float4*>(&c.r1K[r1][l][wq][0]);
                Sh[h] = (s4.x + s4.y) + (s4.z + s4.w);
                Sdh[h] = ((double)s4.x + (double)s4.y) + ((double)s4.z + (double)s4.w);
                Khd[h] = ((double)k4.x + (double)k4.y) + ((double)k4.z + (double)k4.w);
                wmh[h] = c.wmx[k][l][wq];
                if (l > 0) cmh[h] = wmh[h] - c.wmx[k][l - 1][wq];   // the centring offset m_l - m_{l-1}
                if (GREEDY) ah[h] = c.r1A[r1][l][wq];
                wm = max_nan_f32(wm, wmh[h]);
            }
        }
        __syncwarp();
        if (lane == 0) {
            c.p1cnt[r1] = 0u;               // the next item of this record slot counts from 0
            mbar_arrive(&c.r1_empty[r1]);
        }
        // tail-slice maximum of the row (NaN-propagating) over the half's HREG lanes
        float msl = wm;
#pragma unroll
        for (int o = HREG / 2; o > 0; o >>= 1) msl = max_nan_f32(msl, __shfl_xor_sync(0xffffffffu, msl, o));
        // each warp's records scaled to the slice maximum (factor 1 when the warp holds it)
        float Sx = 0.f, fh[NSPLIT];
        double Kxd = 0.0;
        int ax = 0x7fffffff;
#pragma unroll
        for (int h = 0; h < NSPLIT; ++h) {
            float f = wmh[h] == msl ? 1.f : ex2f((wmh[h] - msl) * l2s);
            if (!(wmh[h] > NEG_MASKED)) f = (act && !(msl > NEG_MASKED)) ? 1.f : 0.f;   // masked warp region
            fh[h] = f;
            Sx += Sh[h] * f;
            // KL numerator sum e (z_l - z_{l-1}) in float64: centred sum plus offset times the sum
            if (l > 0 && f != 0.f) Kxd += (double)f * (Khd[h] + (double)cmh[h] * Sdh[h]);
            if (wmh[h] == msl) ax = min(ax, ah[h]);
        }
#pragma unroll
        for (int o = HREG / 2; o > 0; o >>= 1) {
            Sx += __shfl_xor_sync(0xffffffffu, Sx, o);
            if (GREEDY) ax = min(ax, __shfl_xor_sync(0xffffffffu, ax, o));
        }
        if (lane == 0) stamp(j, 9);
        // lanes 8 l and 8 l + HREG publish row l's exchange records of the two tail slices first:
        // the other slices wait for them (self-validating: sum != 0, the slice maximum's entry
        // has e = 1 in the sum); this CTA's fetcher may start polling
        const bool pub_lane = inrow && (w % HREG) == 0 && w / HREG < NH && tslice < C;
        const size_t idx = ((size_t)u * L + l) * C + tslice;
        if (pub_lane)
            st_relaxed_u64(reinterpret_cast<unsigned long long*>(p.partms) + idx,
                           ((unsigned long long)__float_as_uint(Sx) << 32) | __float_as_uint(msl));
#if !MSD_PUB_LATE
        __syncwarp();
        if (lane == 0) {
            stamp(j, 5);
            if (!LSE) mbar_arrive(&c.pub[k]);
        }
#endif
        // then the tail's Partial, off the exchange's critical path: the slice sum again in
        // float64 from the sub-records (the row normalisers' precision decides the KL and
        // acceptance errors of the tail), the KL numerator in fp32
        // (hardware float -> double conversions: off the latency path, few instructions)
        double Sd = 0.0;
#pragma unroll
        for (int h = 0; h < NSPLIT; ++h) Sd += Sdh[h] * (double)fh[h];
#pragma unroll
        for (int o = HREG / 2; o > 0; o >>= 1) {
            Sd += __shfl_xor_sync(0xffffffffu, Sd, o);
            Kxd += __shfl_xor_sync(0xffffffffu, Kxd, o);
        }
        if (pub_lane) {
            Partial pr;
            pr.m = msl;                                   // raw units (the tail scales exponents)
            pr.amax = GREEDY ? ax : 0;
            pr.S = Sd;
            pr.Kl = Kxd * (double)sc;
            p.partials[idx] = pr;
        }
#if MSD_PUB_LATE
        __syncwarp();
        if (lane == 0) {
            stamp(j, 5);
            if (!LSE) mbar_arrive(&c.pub[k]);
        }
#endif
    };

    const bool p1only = (p.dbg & 1) != 0;   // debug: pass 1 + TMA ring only (results invalid)
    if (p1only && warp != W_PROD && warp < W_P1) {
    } else if (warp >= W_P1) {
        // ================================================================ pass-1 warps
        // Two groups of NCW warps take alternate items, so one group's reductions and barrier
        // waits overlap the other group's exponentials.  Reference: the warp maximum of the
        // row (the dominant entries then have |z - m| small, so the fp32 exponent argument
        // keeps full relative accuracy).  Rows are processed in two 8-element halves.
        const int g1 = (warp - W_P1) / NW1;
        const int wi = (warp - W_P1) % NW1;     // warp of the item (record index)
        const int rg = wi % NCW;                // element region
        const int hs = wi / NCW;                // split of the region: vectors / quarters of this warp
        constexpr int QPW = (CET / 8) / NSPLIT; // 8-element quarters per warp and row
        constexpr int VPW = NV / NSPLIT;        // vectors per warp and row
        const int hh = rg / HREG;               // its half (tail slice NH s + hh)
        const int gofs = (int)hbase[hh] - hh * VS;   // ring-row index -> vocabulary id
        if ((amask >> rg) & 1u) {
            PROF_DECL
            const uint32_t tbase = tcol(rg);
            Cursor cu;
            for (int x = 0; x < g1; ++x) cu.next(S, PP, PT, NT);
            for (; cu.j < n_my;) {
                const int j = cu.j;
                int64_t u, b, i;
                item(j, u, b, i);
                const bool isT = cu.isT(PT);
                const int q = cu.q;
                const int k = j & (NQ - 1);
                const int r1 = j & (R1 - 1);
                Tin* stage = ring + (size_t)cu.st * L * RS;
                mbar_wait(&c.full[cu.st], (uint32_t)cu.sph);
                if (p.dbg & 4) {   // debug: the TMA ring alone (no pass-1 arithmetic)
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&c.empty[cu.st]);
                    for (int x = 0; x < NG1; ++x) cu.next(S, PP, PT, NT);
                    continue;
                }
                PROF(0)
                if (wi == 0 && lane == 0) stamp(j, 1);
                // a row length that is not a multiple of 16 bytes: patch the straddling vector
                if (hbulk[hh] != hlen[hh])
                    repair_stage<Tin, L, NV>(stage, RS, p.lv, b, i, hbase[hh], rg, lane, hbulk[hh], hlen[hh],
                                             hs * VPW, (hs + 1) * VPW);
                // per-thread then per-warp max of every row (NaN-propagating)
                float wm[L];
#pragma unroll
                for (int l = 0; l < L; ++l) {
                    float tm = -INFINITY;
#pragma unroll
                    for (int jv = hs * VPW; jv < (hs + 1) * VPW; ++jv) {
                        const uint4 r = *reinterpret_cast<const uint4*>(stage + (size_t)l * RS + vec_index<Tin>(rg, lane, jv));
                        if (ES == 2) {
                            const uint32_t mx = max_nan_bf16x2(max_nan_bf16x2(r.x, r.y), max_nan_bf16x2(r.z, r.w));
                            tm = max_nan_f32(tm, max_nan_f32(bf16lo(mx), bf16hi(mx)));
                        } else {
                            tm = max_nan_f32(max_nan_f32(tm, max_nan_f32(__uint_as_float(r.x), __uint_as_float(r.y))),
                                             max_nan_f32(__uint_as_float(r.z), __uint_as_float(r.w)));
                        }
                    }
                    wm[l] = redux_max_nan(tm);
                }
                // record slot k free (pass 2 of item j - NQ has read it), TMEM slot q free,
                // record ring slot r1 free
                if (j >= NQ && !p1only) mbar_wait(&c.rowf_empty[k], (uint32_t)(((j / NQ) - 1) & 1));
                if (isT && cu.tj >= NT && !p1only) {
                    mbar_wait(&c.tm_empty[q], (uint32_t)(cu.tph ^ 1));
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                }
                if (j >= R1 && !p1only) mbar_wait(&c.r1_empty[r1], (uint32_t)(((j / R1) - 1) & 1));
                if (wi == 0 && lane == 0) stamp(j, 2);
                PROF(1)
                float Sv[L], Kv[L];
                int am[L];
                // one pass over the thread's elements, half-major (all rows of half 0, then of
                // half 1); e parked in TMEM (T items)
                auto run = [&](bool clamp) {
                    float2 s2[L], k2[L];
#pragma unroll
                    for (int l = 0; l < L; ++l) {
                        s2[l] = k2[l] = make_float2(0.f, 0.f);
                        am[l] = 0x7fffffff;
                    }
#pragma unroll
                    for (int h = hs * QPW; h < (hs + 1) * QPW; ++h) {
                        float2 yprev[4];
#pragma unroll
                        for (int l = 0; l < L; ++l) {
                            float e[8];
                            float2 y[4];
                            half_exp<Tin>(stage + (size_t)l * RS, rg, lane, h, wm[l], clamp, e, y, l2s);
                            const float2 e01 = __fadd2_rn(make_float2(e[0], e[1]), make_float2(e[2], e[3]));
                            const float2 e23 = __fadd2_rn(make_float2(e[4], e[5]), make_float2(e[6], e[7]));
                            s2[l] = __fadd2_rn(s2[l], __fadd2_rn(e01, e23));
                            if (l > 0) {
                                // KL numerator sum e_l (z_l - z_{l-1}) = sum e_l (y_l - y_{l-1}) +
                                // (m_l - m_{l-1}) sum e_l: the centred differences y_l - y_{l-1}
                                // (exact in fp32) are accumulated here, the offset term is added
                                // by the publisher in float64 -- a constant logit offset between
                                // the levels never enters the fp32 sums (R18)
                                const float2 neg1 = make_float2(-1.f, -1.f);
                                float2 ka = __fmul2_rn(make_float2(e[0], e[1]), __ffma2_rn(yprev[0], neg1, y[0]));
                                float2 kb = __fmul2_rn(make_float2(e[2], e[3]), __ffma2_rn(yprev[1], neg1, y[1]));
                                ka = __ffma2_rn(make_float2(e[4], e[5]), __ffma2_rn(yprev[2], neg1, y[2]), ka);
                                kb = __ffma2_rn(make_float2(e[6], e[7]), __ffma2_rn(yprev[3], neg1, y[3]), kb);
                                k2[l] = __fadd2_rn(k2[l], __fadd2_rn(ka, kb));
                            }
#pragma unroll
                            for (int pp = 0; pp < 4; ++pp) {
                                yprev[pp] = y[pp];
                                if (GREEDY) {
                                    const int ib = gofs + half_index<Tin>(rg, lane, h, pp);
                                    if (y[pp].x == 0.f) am[l] = min(am[l], ib);
                                    if (y[pp].y == 0.f) am[l] = min(am[l], ib + 1);
                                }
                            }
                            if (isT) tm_st8(tbase + (uint32_t)(q * CET * L + l * CET + h * 8), e);
                        }
                    }
#pragma unroll
                    for (int l = 0; l < L; ++l) {
                        Sv[l] = s2[l].x + s2[l].y;
                        Kv[l] = k2[l].x + k2[l].y;
                    }
                };
                // fast path: bf16 rows whose warp maxima are finite (no masked / NaN / +inf
                // chunk); -inf entries inside a finite chunk are caught by the finiteness check.
                // Otherwise (and for f32 logits): the -1e30 clamp.
                bool fast = ES == 2;
#pragma unroll
                for (int l = 0; l < L; ++l) fast = fast && (wm[l] > NEG_MASKED) && (wm[l] < INFINITY);
                if (fast) {
                    run(false);
                    bool ok = true;
#pragma unroll
                    for (int l = 0; l < L; ++l) ok = ok && isfinite(Sv[l]) && isfinite(Kv[l]);
                    fast = __all_sync(0xffffffffu, ok);
                    if (!fast && isT) tm_wait_st();
                }
                if (!fast) {
#pragma unroll
                    for (int l = 0; l < L; ++l) {
                        float tm = -INFINITY;
#pragma unroll
                        for (int jv = hs * VPW; jv < (hs + 1) * VPW; ++jv) {
                            float xs[VEC];
                            unpack_clamped<Tin>(*reinterpret_cast<const uint4*>(stage + (size_t)l * RS + vec_index<Tin>(rg, lane, jv)), xs);
#pragma unroll
                            for (int kk = 0; kk < VEC; ++kk) tm = max_nan_f32(tm, xs[kk]);
                        }
                        wm[l] = redux_max_nan(tm);
                    }
                    run(true);
                }
                PROF(2)
#pragma unroll
                for (int l = 0; l < L; ++l) {
                    Sv[l] = fold4(Sv[l]);
                    if (l > 0) Kv[l] = fold4(Kv[l]);
                }
                if (GREEDY) {
#pragma unroll
                    for (int l = 0; l < L; ++l) am[l] = redux_min_s32(am[l]);
                }
                // a T item's slice has been consumed: hand the ring stage back to the producer
                // (an R item's stage is released by pass 2)
                __syncwarp();
                if (lane == 0) {
                    if (isT || p1only) mbar_arrive(&c.empty[cu.st]);
#pragma unroll
                    for (int l = 0; l < L; ++l) c.wmx[k][l][wi] = wm[l];
                    const uint32_t bit = 1u << wi;
                    if (fast) atomicAnd(&c.clampw[k], ~bit);
                    else atomicOr(&c.clampw[k], bit);
                    if (LSE && !p1only) mbar_arrive(&c.pub[k]);     // this warp's maxima are out
                }
                PROF(3)
                if (lane < NSUB1) {
#pragma unroll
                    for (int l = 0; l < L; ++l) {
                        c.r1S[r1][l][wi][lane] = Sv[l];
                        c.r1K[r1][l][wi][lane] = Kv[l];
                    }
                    if (GREEDY && lane == 0) {
#pragma unroll
                        for (int l = 0; l < L; ++l) c.r1A[r1][l][wi] = am[l];
                    }
                }
                PROF(4)
                if (isT) {
                    tm_wait_st();
                    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                }
                __syncwarp();
                if (wi == 0 && lane == 0) stamp(j, 3);
#if defined(MSD_TRACE) && !defined(MSD_PROF)
                if (lane == 0 && p.trace)
                    atomicMax(p.trace + ((int64_t)(grp + j * kgrp) * Cc + sfix) * 16 + 7, (unsigned long long)globaltimer());
#endif
                if (lane == 0 && !p1only) {
                    if (!MSD_INLINE_PUB) mbar_arrive(&c.r1_full[r1]);
                    if (isT) mbar_arrive(&c.tm_full[q]);
                }
#if MSD_INLINE_PUB
                if (!p1only) {
                    // the last pass-1 warp of the item publishes its records at once (no wake-up
                    // of a publisher warp): fence + counter, like a last-block reduction
                    uint32_t last = 0;
                    if (lane == 0) {
                        __threadfence_block();
                        last = atomicAdd(&c.p1cnt[r1], 1u) == (uint32_t)(nact - 1) ? 1u : 0u;
                    }
                    if (__shfl_sync(0xffffffffu, last, 0)) {
                        __threadfence_block();
                        publish(j);
                    }
                }
#endif
                PROF(5)
                PROF_ITEM
                for (int x = 0; x < NG1; ++x) cu.next(S, PP, PT, NT);
            }
            PROF_FLUSH(0)
        }
    } else if (warp >= W_P2) {
        // ================================================================ pass-2 warps
        // warp W_P2 + vw handles regions vw, vw + NCW2, ... (the same TMEM lane quadrant as
        // pass-1 warp vw: NCW2 is a multiple of 4), one after the other for every item
        const int vw = warp - W_P2;
        uint32_t mine = 0;
        for (int rr = 0; rr < NPR; ++rr) mine |= amask & (1u << (vw + NCW2 * rr));
        if (mine) {
            PROF_DECL
            Cursor cu;
            for (; cu.j < n_my; cu.next(S, PP, PT, NT)) {
              for (int rr = 0; rr < NPR; ++rr) {
                const int v = vw + NCW2 * rr;
                if (!((amask >> v) & 1u)) continue;
                const int j = cu.j;
                const bool isT = cu.isT(PT);
                const int q = cu.q;
                const int k = j & (NQ - 1);
                const int r2 = j & (R2 - 1);
                mbar_wait_lat(&c.rowf_full[k], (uint32_t)((j / NQ) & 1));
                PROF(0)
                // factors of the region's NSPLIT pass-1 warps (chunk ch belongs to split ch NSPLIT / 2)
                float rh[L][NSPLIT], sc[L][NSPLIT], wm[L][NSPLIT];
                const uint32_t cw = c.clampw[k];
#pragma unroll
                for (int l = 0; l < L; ++l) {
#pragma unroll
                    for (int h = 0; h < NSPLIT; ++h) {
                        rh[l][h] = l > 0 ? c.rowf[k][l][v + NCW * h].rho : 0.f;
                        sc[l][h] = l > 0 ? c.rowf[k][l][v + NCW * h].scale : 0.f;
                        wm[l][h] = c.wmx[k][l][v + NCW * h];
                    }
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&c.rowf_empty[k]);
                float acc[L];
#pragma unroll
                for (int l = 0; l < L; ++l) acc[l] = 0.f;
                // residual of the pair (l-1, l) over a 16-element chunk: sum max(e_l - rho e_{l-1}, 0)
                float2 a2[L];
#pragma unroll
                for (int l = 0; l < L; ++l) a2[l] = make_float2(0.f, 0.f);
                auto pair = [&](int l, int hc, const float* ea, const float* eb) {
                    const float2 nr = make_float2(-rh[l][hc], -rh[l][hc]);
                    float2 x = make_float2(0.f, 0.f), xb = make_float2(0.f, 0.f);
#pragma unroll
                    for (int kk = 0; kk < CH; kk += 2) {
                        float2 t = __ffma2_rn(make_float2(eb[kk], eb[kk + 1]), nr, make_float2(ea[kk], ea[kk + 1]));
                        t.x = fmaxf(t.x, 0.f);
                        t.y = fmaxf(t.y, 0.f);
                        if (kk & 2) xb = __fadd2_rn(xb, t);
                        else x = __fadd2_rn(x, t);
                    }
                    const float2 xs = __fadd2_rn(x, xb);
                    a2[l] = __ffma2_rn(xs, make_float2(sc[l][hc], sc[l][hc]), a2[l]);
                };
                if (isT) {
                    mbar_wait_lat(&c.tm_full[q], (uint32_t)cu.tph);
                    if (v == 0 && lane == 0) stamp(j, 12);
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                    PROF(1)
                    const uint32_t tb = tcol(v) + (uint32_t)(q * CET * L);
#pragma unroll
                    for (int ch = 0; ch < CET / CH; ++ch) {
                        const int hc = ch * NSPLIT / (CET / CH);
                        float ea[CH], eb[CH], ec[CH];
                        tm_ld16(tb + (uint32_t)(ch * CH), eb);
                        tm_ld16(tb + (uint32_t)(CET + ch * CH), ea);
                        if (L > 2) tm_ld16(tb + (uint32_t)(2 * CET + ch * CH), ec);
                        tm_wait_ld();
                        pair(1, hc, ea, eb);
                        if (L > 2) pair(2, hc, ec, ea);
#pragma unroll
                        for (int l = 3; l < L; ++l) {
#pragma unroll
                            for (int kk = 0; kk < CH; ++kk) eb[kk] = ec[kk];
                            tm_ld16(tb + (uint32_t)(l * CET + ch * CH), ec);
                            tm_wait_ld();
                            pair(l, hc, ec, eb);
                        }
                    }
                    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&c.tm_empty[q]);
                    PROF(2)
                } else {
                    // R item: recompute e from the kept ring stage (already complete: full[st]
                    // cannot advance before the stage is released here)
                    mbar_wait(&c.full[cu.st], (uint32_t)cu.sph);
                    if (v == 0 && lane == 0) stamp(j, 12);
                    PROF(1)
                    const Tin* stage = ring + (size_t)cu.st * L * RS;
                    const bool skip_r = (p.dbg & 2) != 0;   // debug: R items skip the recomputation
                    if (!skip_r) {
                        constexpr int NVC = CH / VEC;      // vectors per chunk
#pragma unroll
                        for (int ch = 0; ch < CET / CH; ++ch) {
                            const int hc = ch * NSPLIT / (CET / CH);
                            const bool clamp = ((cw >> (v + NCW * hc)) & 1u) || ES == 4;
                            float eprev[CH];
#pragma unroll
                            for (int l = 0; l < L; ++l) {
                                uint4 raw[NVC];
#pragma unroll
                                for (int jv = 0; jv < NVC; ++jv)
                                    raw[jv] = *reinterpret_cast<const uint4*>(stage + (size_t)l * RS +
                                                                              vec_index<Tin>(v, lane, ch * NVC + jv));
                                float e[CH];
                                float2 y[CH / 2];
                                row_exp<Tin>(raw, wm[l][hc], clamp, e, y, l2s);
                                if (l > 0) pair(l, hc, e, eprev);
#pragma unroll
                                for (int kk = 0; kk < CH; ++kk) eprev[kk] = e[kk];
                            }
                        }
                    }
                    __syncwarp();
                    if (lane == 0) mbar_arrive_cnt(&c.empty[cu.st], (uint32_t)NSPLIT);
                    PROF(2)
                }
#pragma unroll
                for (int l = 1; l < L; ++l) acc[l] = a2[l].x + a2[l].y;
#pragma unroll
                for (int l = 1; l < L; ++l) acc[l] = fold4(acc[l]);
                PROF(3)
                if (j >= R2) mbar_wait(&c.r2_empty[r2], (uint32_t)(((j / R2) - 1) & 1));
                if (lane < NSUB) {
#pragma unroll
                    for (int l = 1; l < L; ++l) c.r2R[r2][l][v][lane] = acc[l];
                }
                __syncwarp();
                if (v == 0 && lane == 0) stamp(j, 13);
                if (lane == 0) mbar_arrive(&c.r2_full[r2]);
                PROF(4)
                PROF_ITEM
              }   // regions of this warp
            }
            PROF_FLUSH(1)
        }
    } else if (warp == W_PROD) {
        // ================================================================ TMA producer
        PROF_DECL
        if (lane == 0) {
            const uint64_t pol = policy_evict_first();
            uint32_t hb[NH], bytes = 0;              // [hbulk_h, VS) of each half holds the pad
#pragma unroll
            for (int h = 0; h < NH; ++h) {
                hb[h] = (uint32_t)(hbulk[h] * ES);
                bytes += hb[h];
            }
            // items j + 1 .. j + pf_dist requested into L2 ahead of their shared-memory copies
            // (cp.async.bulk.prefetch: no smem, no barrier): the copies then complete at L2
            // latency, which narrows the spread of a group's CTAs (Llama-3 core 1.004 -> 0.980 ms
            // at distance 2; 3..8 measured in between)
            const int pfd = p.pf_dist;
            auto prefetch = [&](int jj) {
                if (jj >= n_my) return;
                int64_t u2, b2, i2;
                item(jj, u2, b2, i2);
#pragma unroll
                for (int l = 0; l < L; ++l) {
                    const Tin* src = reinterpret_cast<const Tin*>(p.lv.ptr[l]) + b2 * p.lv.bs[l] + i2 * p.lv.ld[l];
#pragma unroll
                    for (int h = 0; h < NH; ++h)
                        if (hb[h]) bulk_prefetch_l2(src + hbase[h], hb[h]);
                }
            };
            for (int jj = 1; jj < pfd; ++jj) prefetch(jj);
            Cursor cu;
            for (; cu.j < n_my; cu.next(S, PP, PT, NT)) {
                const int j = cu.j;
                if (pfd) prefetch(j + pfd);
                if (j >= S) mbar_wait(&c.empty[cu.st], (uint32_t)(cu.sph ^ 1));
                PROF(0)
                int64_t u, b, i;
                item(j, u, b, i);
                stamp(j, 0);
                if (bytes) {
                    mbar_arrive_expect_tx(&c.full[cu.st], bytes * L);
#pragma unroll
                    for (int l = 0; l < L; ++l) {
                        Tin* dst = ring + ((size_t)cu.st * L + l) * RS;
                        const Tin* src = reinterpret_cast<const Tin*>(p.lv.ptr[l]) + b * p.lv.bs[l] + i * p.lv.ld[l];
#pragma unroll
                        for (int h = 0; h < NH; ++h)
                            if (hb[h]) bulk_g2s(dst + h * VS, src + hbase[h], hb[h], &c.full[cu.st], pol);
                    }
                } else {
                    mbar_arrive(&c.full[cu.st]);   // nothing to copy (a slice past the row end)
                }
                PROF(1)
                PROF_ITEM
            }
        }
        PROF_FLUSH(5)
    } else if (warp == W_PUB) {
        // ================================================================ publisher
        // lane = 8 l + w: row l, region w (L <= 4).  Each lane sums its region's sub-records,
        // scales them by 2^((m_w - m_s) log2 e) relative to the tail slice's maximum m_s (1 when
        // the region holds the maximum) and the HREG lanes of each half reduce with 2 shuffle
        // levels: one record per (row, tail slice NH s + w / HREG).
        PROF_DECL
#if !MSD_INLINE_PUB
        for (int j = 0; j < n_my; ++j) {
            mbar_wait_lat(&c.r1_full[j & (R1 - 1)], (uint32_t)((j / R1) & 1));
            if (lane == 0) stamp(j, 8);
            PROF(0)
            publish(j);
            PROF(1)
            PROF_ITEM
        }
#endif
        PROF_FLUSH(2)
    } else if (warp >= W_FETCH0 && warp < W_FETCH0 + NFETCH) {
        // ================================================================ fetchers (pass-2 factors)
        PROF_DECL
        const int f = warp - W_FETCH0;
        const int LC = L * C;     // <= FBUF (checked on the host)
        unsigned long long* fb = c.fbuf[f];
        for (int j = f; j < n_my; j += NFETCH) {
            int64_t u, b, i;
            item(j, u, b, i);
            const int k = j & (NQ - 1);
            if (lane == 0) stamp(j, 6);
            // producer-supplied normalisers: lane l's row, in flight while the pass-1 warps finish
            double lz = 0.0;
            if (LSE && lane < L) lz = __ldg(p.lse + ((size_t)lane * p.B + b) * p.K + i);
            // the other slices of the unit are published around the time this one is: poll only
            // from then on (polls steal issue slots and L2 bandwidth)
            // (LSE: pub[k] is arrived by the pass-1 warps themselves -- only their maxima are needed)
            mbar_wait_lat(&c.pub[k], (uint32_t)((j / NQ) & 1));
            const uint64_t t0 = globaltimer();
            PROF(4)
            // stage the unit's records; a record whose sum is still 0 is not yet visible
            const unsigned long long* pm = reinterpret_cast<const unsigned long long*>(p.partms) + (size_t)u * LC;
            // producer-supplied row normalisers (msd_chain_verify_lse): nothing to exchange
            while (!LSE) {
                // all loads in flight before any use (one round trip), then stage in smem
                constexpr int MAXB = FBUF / 32;
                unsigned long long rr[MAXB];
#pragma unroll
                for (int t = 0; t < MAXB; ++t) {
                    const int idx = t * 32 + lane;
                    rr[t] = idx < LC ? ld_relaxed_u64_nc(pm + idx) : 0x100000000ull;
                }
                bool ok = true;
#pragma unroll
                for (int t = 0; t < MAXB; ++t) {
                    const int idx = t * 32 + lane;
                    if (idx < LC) fb[idx] = rr[t];
                    ok &= (uint32_t)(rr[t] >> 32) != 0u;
                }
                if (__all_sync(0xffffffffu, ok)) break;
                if (globaltimer() - t0 > 4000000000ull) {
                    if (lane == 0) {
                        atomicOr(p.err, 1u);
                        atomicOr(&p.flags[b], (uint32_t)MSD_F_TIMEOUT);
                    }
                    break;
                }
                __nanosleep(MSD_POLL_NS);
            }
            __syncwarp();
            if (lane == 0) stamp(j, 4);
            PROF(0)
            // row normalisers N_l from the C slice records, relative to this slice's own record
            // reference R_l (fp32).  A slice reference more than 2^127 above R_l, or a masked
            // own slice, falls back to the maximum reference.
            float Rl[L], Sl[L];
            if (LSE) {
                // reference: this CTA's own maximum of the row (its pass-1 warps' maxima); the
                // normaliser relative to it, exp(lse - ref sc) >= 1, from the supplied float64 LSE
                // (lane l computes row l, then every lane gets all rows)
                float mr = -INFINITY;
                if (lane < L)
                    for (int w = 0; w < NW1; ++w)
                        if ((amask >> (w % NCW)) & 1u) mr = fmaxf(mr, c.wmx[k][lane][w]);
                if (!(mr > NEG_MASKED)) mr = (float)(lz / (double)sc);
                const double x = (double)mr * (double)sc - lz;       // <= 0 up to the rounding of mr
                // exp(-x) for -x >= 0 (dexp_neg's reduction holds for arguments up to ~700 either sign)
                const float sn = lane < L ? (float)dexp_neg(-x) : 0.f;
#pragma unroll
                for (int l = 0; l < L; ++l) {
                    Rl[l] = __shfl_sync(0xffffffffu, mr, l);
                    Sl[l] = __shfl_sync(0xffffffffu, sn, l);
                }
            } else {
#pragma unroll
            for (int l = 0; l < L; ++l) {
                Rl[l] = __uint_as_float((uint32_t)fb[l * C + NH * s]);   // first tail slice's record
                Sl[l] = 0.f;
            }
            for (int t = lane; t < C; t += 32) {
#pragma unroll
                for (int l = 0; l < L; ++l) {
                    const unsigned long long r = fb[l * C + t];
                    const float vm = __uint_as_float((uint32_t)r);
                    if (vm > NEG_MASKED)
                        Sl[l] = fmaf(__uint_as_float((uint32_t)(r >> 32)), ex2f((vm - Rl[l]) * l2s), Sl[l]);
                }
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
                for (int l = 0; l < L; ++l) Sl[l] += __shfl_xor_sync(0xffffffffu, Sl[l], o);
            }
            bool slow = false;
#pragma unroll
            for (int l = 0; l < L; ++l) slow = slow || !(Rl[l] > NEG_MASKED) || !(Sl[l] < INFINITY);
            if (slow) {
#pragma unroll
                for (int l = 0; l < L; ++l) Rl[l] = -INFINITY;
                for (int t = lane; t < C; t += 32) {
#pragma unroll
                    for (int l = 0; l < L; ++l) Rl[l] = fmaxf(Rl[l], __uint_as_float((uint32_t)fb[l * C + t]));
                }
#pragma unroll
                for (int l = 0; l < L; ++l) {
                    Rl[l] = warp_max(Rl[l]);
                    Sl[l] = 0.f;
                }
                for (int t = lane; t < C; t += 32) {
#pragma unroll
                    for (int l = 0; l < L; ++l) {
                        const unsigned long long r = fb[l * C + t];
                        const float vm = __uint_as_float((uint32_t)r);
                        if (vm > NEG_MASKED)
                            Sl[l] = fmaf(__uint_as_float((uint32_t)(r >> 32)), exp2f_fma((vm - Rl[l]) * l2s), Sl[l]);
                    }
                }
#pragma unroll
                for (int l = 0; l < L; ++l) Sl[l] = warp_sum(Sl[l]);
            }
            }   // exchange records
            PROF(1)
            if (j >= NQ) mbar_wait(&c.rowf_empty[k], (uint32_t)(((j / NQ) - 1) & 1));
            PROF(2)
            // per pass-1-warp factors: x = NW1 (l - 1) + w for warp w and the pair ending at row l
            for (int x = lane; x < (L - 1) * NW1; x += 32) {
                const int w = x % NW1, l = 1 + x / NW1;
                if ((amask >> (w % NCW)) & 1u) {
                    float Ma = Rl[0], Mb = Rl[0], Sa = Sl[0], Sb = Sl[0];
#pragma unroll
                    for (int r = 1; r < L; ++r)
                        if (r == l) { Ma = Rl[r]; Sa = Sl[r]; Mb = Rl[r - 1]; Sb = Sl[r - 1]; }
                    const float wa = c.wmx[k][l][w], wb = c.wmx[k][l - 1][w];
                    const float ca = (wa > NEG_MASKED && Ma > NEG_MASKED) ? ex2f((wa - Ma) * l2s) : 0.f;
                    const float cb = (wb > NEG_MASKED && Mb > NEG_MASKED) ? ex2f((wb - Mb) * l2s) : 0.f;
                    const bool skip = !(ca > 0.f) || !(Sa > 0.f) || !(Sb > 0.f) || !isfinite(Sa) || !isfinite(Sb) ||
                                      !isfinite(ca) || !isfinite(cb);
                    WF wf;
                    // identical rows must give rho = 1 exactly (zero residual), which the
                    // Newton reciprocal alone does not guarantee
                    const float num = cb * Sa, den = Sb * ca;
                    wf.rho = skip ? 0.f : (num == den ? 1.f : __fdiv_rn(num, den));
                    wf.scale = skip ? 0.f : __fdiv_rn(ca, Sa);
                    c.rowf[k][l][w] = wf;
                }
            }
            __syncwarp();
            if (lane == 0) {
                stamp(j, 10);
                mbar_arrive(&c.rowf_full[k]);
            }
            PROF(3)
            PROF_ITEM
        }
        PROF_FLUSH(3)
    } else if (warp == W_RED) {
        // ================================================================ reducer (slice residual)
        PROF_DECL
        // lane = 4 v + t: region v (half v / HREG), sub-record t; each half's 16 lanes fold
        static_assert(NCW * NSUB == 32 && HREG * NSUB == 16, "reducer lane layout");
        const int v = lane >> 2, t = lane & 3;
        const bool act = (amask >> v) & 1u;
        const int tslice = NH * s + v / HREG;
        for (int j = 0; j < n_my; ++j) {
            int64_t u, b, i;
            item(j, u, b, i);
            const int r2 = j & (R2 - 1);
            mbar_wait_lat(&c.r2_full[r2], (uint32_t)((j / R2) & 1));
            PROF(0)
            float R[L];
#pragma unroll
            for (int l = 1; l < L; ++l) {
                float d = act ? c.r2R[r2][l][v][t] : 0.f;
#pragma unroll
                for (int o = HREG * NSUB / 2; o > 0; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
                R[l] = d;
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&c.r2_empty[r2]);
            if ((lane % (HREG * NSUB)) == 0 && lane / (HREG * NSUB) < NH && tslice < C) {
#pragma unroll
                for (int l = 1; l < L; ++l) p.resid[((size_t)u * (L - 1) + (l - 1)) * C + tslice] = f2d_alu(R[l]);
            }
            if (lane == 0) stamp(j, 15);
            PROF(1)
            PROF_ITEM
        }
        PROF_FLUSH(4)
    }

    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (warp == W_PROD) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(c.taddr));
}


template <typename Tin, int L, bool G, bool LSE>
static cudaError_t launch_one(const CoreParams& p0, cudaStream_t s) {
    CoreParams p = p0;
    const int ES = (int)sizeof(Tin);
    const int NT = core_tslots(L);
    const int NH = ES == 2 ? 2 : 1;          // tail slices per item
    p.rs = NH * VS;
    const size_t ctl = align_up(sizeof(Ctl<L>), 128);
    const size_t stage_bytes = (size_t)L * p.rs * ES;
    int S = (int)((SMEM_BUDGET - ctl - 256) / stage_bytes);
    S = std::min(S, std::min(SMAX, g_knobs.stages > 0 ? (int)g_knobs.stages : SMAX));
    if (S < 2) return cudaErrorInvalidConfiguration;
    p.stages = S;
    // item pattern: T items use the NT TMEM slots; R items keep their ring stage.  Of the S
    // stages ~4 are needed in flight for the TMA; the rest may hold R items.
    int pt = g_knobs.pat_t >= 0 ? (int)g_knobs.pat_t : NT, pr = g_knobs.pat_r;
    if (pr < 0) pr = std::max(0, std::min(2, S - 3));
    if (pt < 1) pt = 1;
    p.pat_t = pt;
    p.pat_p = pt + pr;
    // L2 prefetch distance: 2 items (core_dbg bits 8..11 = distance + 1 override it)
    p.pf_dist = ((g_knobs.core_dbg >> 8) & 15) ? ((g_knobs.core_dbg >> 8) & 15) - 1 : 2;
    const size_t smem = ctl + (size_t)S * stage_bytes + 128;
    auto k = core_kernel<Tin, L, G, LSE>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int dev = 0, nsm = 0, occ = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, CORE_THREADS, smem);
    if (e != cudaSuccess) return e;
    if (occ < 1) return cudaErrorInvalidConfiguration;
    if (L * p.C > FBUF) return cudaErrorInvalidValue;   // vocabulary too large for the exchange buffer
    // one CTA per SM (it owns all 512 TMEM columns); k = floor(nsm / Cc) groups of
    // Cc = ceil(C / NH) CTAs
    const int Cc = (p.C + NH - 1) / NH;
    int64_t kg = nsm / Cc;
    if (kg < 1) return cudaErrorInvalidConfiguration;
    if (kg > p.U) kg = p.U;
    const int64_t grid = kg * Cc;
    void* args[] = {&p};
    return cudaLaunchCooperativeKernel((const void*)k, dim3((unsigned)grid), dim3(CORE_THREADS), args, smem, s);
}

cudaError_t launch_core(const CoreParams& p, int bf16, int greedy, cudaStream_t s) {
#define MSD_CASE(TY, LL)                                                         \
    if (p.L == LL) {                                                             \
        if (p.lse) return greedy ? launch_one<TY, LL, true, true>(p, s) : launch_one<TY, LL, false, true>(p, s); \
        return greedy ? launch_one<TY, LL, true, false>(p, s) : launch_one<TY, LL, false, false>(p, s);         \
    }
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
