// msd_core.cu -- the streaming pass over every logit row at the draft positions.
//
// Rows a1 (Eq. 1 normaliser) and a5 (Eq. 5 DTV; KL) of the
// hot path, for all L chain levels at once so every logit byte is read from HBM
// exactly once.
//
// Decomposition.  A *unit* is one (request b, draft position i < K) and owns the L
// rows Z_l[b, i, :].  A unit is cut into C slices of VS = 4096 vocabulary entries;
// an *item* is (unit, slice).  The kernel is persistent and cooperative (one CTA per
// SM): CTA g processes items g, g+G, g+2G, ...; the C items of a unit run on C CTAs,
// which exchange per-slice (max, sum) records through global memory.
//
// Warp specialisation (16 compute + 7 service warps):
//   compute  pass 1 of item j: per-warp max of each row (the only cross-lane step),
//            e_v = 2^((z_v - m_w) log2 e) -- one MUFU.EX2 per element --, per-thread sums
//            (S, KL numerator) to shared memory, e_v parked in TMEM (tcgen05.st);
//            then pass 2 of item j-LAG: e_v back from TMEM (tcgen05.ld), per-thread residual
//            sum_v max(p_v - q_v, 0) of every adjacent pair to shared memory.
//   producer TMA bulk copies (cp.async.bulk) of the L row slices into an S-stage ring.
//   publisher folds pass-1 records into the slice record (float64 combine), publishes a
//            self-validating 64-bit (max, sum) record per row with a relaxed store and bumps
//            the unit counter with a relaxed red (no fence on the critical path).
//   fetchers (4, items j = f mod 4) poll the unit counter, load the unit's C records in one
//            round trip (re-loading if one is not yet visible), combine them (float64) into
//            the row normalisers and derive the per-warp pass-2 factors of this slice.
//   reducer  folds pass-2 records into the slice residual R_s (float64).
// The exchange latency hides behind LAG items of pass 1: TMEM holds LAG+1 items of
// exponentials per compute thread (128 columns / (8 L)).
#include "msd_common.cuh"
#include "msd_internal.h"

namespace msd {

constexpr int NCW = 8;                 // pass-1 warps (pass-2 warps: NCW .. 2 NCW - 1)
constexpr int CTH = NCW * 32;          // pass-1 threads
constexpr int CET = VS / CTH;          // elements per pass-1 thread per row (16)
constexpr int NFETCH = 5;
constexpr int W_P2 = NCW, W_PROD = 2 * NCW, W_PUB = 2 * NCW + 1, W_FETCH0 = 2 * NCW + 2,
              W_RED = W_FETCH0 + NFETCH;
constexpr int CORE_THREADS = (W_RED + 1) * 32;
constexpr int SMAX = 6;
constexpr int FBUF = 192;              // records per fetcher staging buffer (L * C <= 192)
constexpr int SMEM_BUDGET = 227 * 1024;
constexpr int NRMAX = 8;
constexpr int R1 = 3, R2 = 3;          // pass-1 / pass-2 record rings
constexpr int NSUB = 4;                // per-warp records after a 3-step shuffle fold (lanes 0..3)
static_assert(CET == 16, "two 16-byte bf16 vectors per thread and row");

struct WF {                // pass-2 factors of one (row, warp) of the current slice
    float rho;             // rho = c_b S_a / (S_b c_a)  (pair ending at this row)
    float scale;           // c_a / S_a
};
template <int L>
struct Ctl {
    uint64_t full[SMAX], empty[SMAX];
    uint64_t r1_full[R1], r1_empty[R1], r2_full[R2], r2_empty[R2];
    uint64_t rowf_full[NRMAX], rowf_empty[NRMAX];
    uint64_t tm_full[NRMAX], tm_empty[NRMAX];   // TMEM item slots: pass-1 warps -> pass-2 warps
    uint32_t taddr;
    float wmx[NRMAX][L][NCW];               // per-warp max of each row, per item slot
    float r1S[R1][L][NCW][NSUB];            // pass-1 partial sums
    float r1K[R1][L][NCW][NSUB];            // pass-1 KL numerators (relative to the warp shift)
    int r1A[R1][L][NCW];                    // greedy: first argmax index per warp
    WF rowf[NRMAX][L][NCW];
    float r2R[R2][L][NCW][NSUB];            // pass-2 residual partials
    float r2scale[R2][L][NCW];
    unsigned long long fbuf[NFETCH][FBUF];       // fetcher staging of a unit's records
};

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void red_add_release(uint32_t* p, uint32_t v) {
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_relaxed_u32(const uint32_t* p) {
    uint32_t r;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(r) : "l"(p) : "memory");
    return r;
}
__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p) {
    unsigned long long r;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(r) : "l"(p) : "memory");
    return r;
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
__device__ __forceinline__ void tm_st8(uint32_t ta, const float* v) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(ta), "f"(v[0]),
                 "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7])
                 : "memory");
}
__device__ __forceinline__ void tm_ld8(uint32_t ta, float* v) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7])
                 : "r"(ta)
                 : "memory");
}
__device__ __forceinline__ void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tm_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ uint32_t clamp_bf16x2(uint32_t w) { return max_nan_bf16x2(w, 0xF149F149u); }

// fold a per-lane value into lanes 0..3 (lane k holds the sum over lanes == k mod 4)
__device__ __forceinline__ float fold4(float v) {
    v += __shfl_xor_sync(0xffffffffu, v, 16);
    v += __shfl_xor_sync(0xffffffffu, v, 8);
    v += __shfl_xor_sync(0xffffffffu, v, 4);
    return v;
}

// TMA ring depth: 4 stages of 24-32 KB (bf16, L = 3-4) keep ~2 us of HBM data in flight.
#ifndef MSD_RING_BYTES
#define MSD_RING_BYTES 98304
#endif
__host__ __device__ constexpr int core_stages(int L, int es) {
    return (MSD_RING_BYTES / (L * VS * es)) < 2 ? 2
         : ((MSD_RING_BYTES / (L * VS * es)) > SMAX ? SMAX : (MSD_RING_BYTES / (L * VS * es)));
}
// item slots of parked exponentials: TMEM holds 256 / (16 L) items per pass-1 warp; the
// shared memory left after the ring and the control block adds 1-2 more (L = 3, 4).
__host__ __device__ constexpr int core_tslots(int L) { return 256 / (CET * L); }
__host__ __device__ constexpr int core_sslots_raw(int L, int es, int ctl_bytes) {
    return (SMEM_BUDGET - core_stages(L, es) * L * VS * es - ctl_bytes - 1024) / (L * CET * CTH * 4);
}
#ifndef MSD_SSLOTS_MAX
#define MSD_SSLOTS_MAX 0   // measured: parking items in shared memory costs more than it hides
#endif
__host__ __device__ constexpr int cmin(int a, int b) { return a < b ? a : b; }
__host__ __device__ constexpr int core_sslots(int L, int es, int ctl_bytes) {
    return core_sslots_raw(L, es, ctl_bytes) < 0
               ? 0
               : cmin(cmin(core_sslots_raw(L, es, ctl_bytes), MSD_SSLOTS_MAX), NRMAX - core_tslots(L));
}

// elements (2 pp, 2 pp + 1) of a thread's 16-byte vector as a float pair
template <typename Tin>
__device__ __forceinline__ float2 elem_pair(const uint4& r, int pp);
template <>
__device__ __forceinline__ float2 elem_pair<__nv_bfloat16>(const uint4& r, int pp) {
    const uint32_t w = pp == 0 ? r.x : pp == 1 ? r.y : pp == 2 ? r.z : r.w;
    return make_float2(bf16lo(w), bf16hi(w));
}
template <>
__device__ __forceinline__ float2 elem_pair<float>(const uint4& r, int pp) {
    return pp == 0 ? make_float2(__uint_as_float(r.x), __uint_as_float(r.y))
                   : make_float2(__uint_as_float(r.z), __uint_as_float(r.w));
}

// The VEC-element vector that straddles the end of a row: the bulk-copied part from shared
// memory, the tail (< 16 bytes) from global memory, -inf past the row.  Out of line so the
// pass-1 loop stays compact in the instruction cache.
template <typename Tin>
__device__ __noinline__ uint4 load_straddle(const Tin* sl, const Tin* g, int e0, int len_bulk, int len) {
    constexpr int VEC = Elem<Tin>::VEC;
    Tin xs[VEC];
#pragma unroll
    for (int k = 0; k < VEC; ++k) {
        const int ee = e0 + k;
        Tin z = (Tin)(-INFINITY);
        if (ee < len_bulk) z = sl[ee];
        else if (ee < len) z = g[ee];
        xs[k] = z;
    }
    return *reinterpret_cast<const uint4*>(xs);
}

// An item whose slice is not a whole number of bulk-copied vectors of length VSe (the last
// slice of a row, or a row length that is not a multiple of 16 bytes): each thread rewrites
// its own vectors of the ring stage -- -inf past the row, the straddling vector element-wise
// from the ring and global memory -- so the pass-1 loads stay unconditional.  Out of line.
template <typename Tin, int L, int NV>
__device__ __noinline__ void repair_stage(Tin* stage, const LevelDesc& lv, int64_t b, int64_t i, int64_t base,
                                          int tid, int len_bulk, int len, int vse) {
    constexpr int VEC = Elem<Tin>::VEC;
    constexpr int ES = (int)sizeof(Tin);
    for (int l = 0; l < L; ++l) {
        Tin* sl = stage + (size_t)l * VS;
        for (int jv = 0; jv < NV; ++jv) {
            const int e0 = (jv * CTH + tid) * VEC;
            if (e0 + VEC <= len_bulk || e0 >= vse) continue;
            uint4 v;
            if (e0 >= len) {
                v = ES == 2 ? make_uint4(0xFF80FF80u, 0xFF80FF80u, 0xFF80FF80u, 0xFF80FF80u)
                            : make_uint4(0xFF800000u, 0xFF800000u, 0xFF800000u, 0xFF800000u);
            } else {
                v = load_straddle<Tin>(sl, reinterpret_cast<const Tin*>(lv.ptr[l]) + b * lv.bs[l] + i * lv.ld[l] + base,
                                       e0, len_bulk, len);
            }
            *reinterpret_cast<uint4*>(sl + e0) = v;
        }
    }
    // these generic-proxy writes precede the next bulk copy (async proxy) into the stage
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

template <typename Tin, int L, bool GREEDY>
__global__ void __launch_bounds__(CORE_THREADS, 1) core_kernel(CoreParams p) {
    constexpr int VEC = Elem<Tin>::VEC;
    constexpr int NV = CET / VEC;           // 1 (bf16) or 2 (f32) vectors per thread and row
    constexpr int ES = (int)sizeof(Tin);
    constexpr int NT = core_tslots(L);                       // TMEM item slots
    constexpr int NSS = core_sslots(L, ES, (int)sizeof(Ctl<L>)); // shared-memory item slots
    constexpr int NR = NT + NSS;
    static_assert(NR <= NRMAX && NT >= 2, "item slots");
    extern __shared__ __align__(128) unsigned char smem[];
    constexpr int S = core_stages(L, ES);
    Tin* ring = reinterpret_cast<Tin*>(smem);
    Ctl<L>& c = *reinterpret_cast<Ctl<L>*>(smem + align_up((size_t)S * L * VS * ES, 128));
    // shared-memory exponential slots: [slot][row][k][pass-1 thread] (conflict-free)
    float* xslot = reinterpret_cast<float*>(smem + align_up((size_t)S * L * VS * ES, 128) + align_up(sizeof(Ctl<L>), 128));

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int C = p.C;
    const int VSe = p.VSe;
    // group scheduling: the grid is k groups of C CTAs; CTA (group, s) handles slice s of
    // units group, group + k, ... -- a unit's C slices always run together on one group
    const int kgrp = gridDim.x / C;
    const int grp = blockIdx.x / C, sfix = blockIdx.x % C;
    const int n_my = grp < kgrp && grp < p.U ? (p.U - grp + kgrp - 1) / kgrp : 0;

    // the ring tail [VSe, VS) of every row is never written by the bulk copies: -inf once, so
    // that clean items load whole vectors unconditionally
    for (int e = tid; e < S * L * (VS - VSe); e += blockDim.x) {
        const int row = e / (VS - VSe);
        ring[(size_t)row * VS + VSe + (e - row * (VS - VSe))] = (Tin)(-INFINITY);
    }
    if (warp == W_PROD) {
        if (lane == 0) {
            for (int s = 0; s < S; ++s) { mbar_init(&c.full[s], 1); mbar_init(&c.empty[s], NCW); }
            for (int r = 0; r < R1; ++r) { mbar_init(&c.r1_full[r], NCW); mbar_init(&c.r1_empty[r], 1); }
            for (int r = 0; r < R2; ++r) { mbar_init(&c.r2_full[r], NCW); mbar_init(&c.r2_empty[r], 1); }
            for (int q = 0; q < NR; ++q) {
                mbar_init(&c.rowf_full[q], 1);
                mbar_init(&c.rowf_empty[q], NCW);
                mbar_init(&c.tm_full[q], NCW);
                mbar_init(&c.tm_empty[q], NCW);
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

    auto stamp = [&](int j, int k) {
        if (p.trace && !(p.dbg & 64)) p.trace[((int64_t)(grp + j * kgrp) * C + sfix) * 16 + k] = globaltimer();
    };
    // (no runtime integer division on the hot loops: it would issue on the busy MUFU pipe)
    auto item = [&](int j, int64_t& u, int& s, int64_t& b, int64_t& i) {
        const uint32_t uu = (uint32_t)(grp + j * kgrp);
        const uint32_t bb = __umulhi(uu, p.kinv);
        u = uu;
        s = sfix;
        b = bb;
        i = uu - bb * (uint32_t)p.K;
    };

    const bool dbg_idle = p.dbg != 0 && warp >= NCW && (warp != W_PROD || (p.dbg & 32));
    if (dbg_idle) {
    } else if (warp < NCW) {
        // ================================================================ pass-1 warps
        const uint32_t tbase = c.taddr + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)((warp >> 2) * 256);
#ifdef MSD_PHASE_PROF
        long long pc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#endif
        for (int j = 0; j < n_my; ++j) {
            int64_t u, b, i;
            int s;
            item(j, u, s, b, i);
            const int st = (int)(j % S);
            const int q = (int)(j % NR);
            const int r1 = (int)(j % R1);
            const int64_t base = (int64_t)s * VSe;
            const int len = (int)max((int64_t)0, min((int64_t)VSe, p.V - base));
            const int len_bulk = (len * ES) / 16 * 16 / ES;
#ifdef MSD_PHASE_PROF
            long long ck0 = clock64();
#endif
            if (!(p.dbg & 32)) mbar_wait(&c.full[st], (uint32_t)((j / S) & 1));
#ifdef MSD_PHASE_PROF
            long long ck1 = clock64();
#endif
            if (tid == 0) stamp(j, 1);
            uint4 raw[L][NV];
            float tmax[L];
            // a row length that is not a multiple of 16 bytes: patch the straddling vector
            if (len_bulk != len) repair_stage<Tin, L, NV>(ring + (size_t)st * L * VS, p.lv, b, i, base, tid, len_bulk, len, VSe);
            // every vector from the ring ([VSe, VS) holds -inf from the prologue)
#pragma unroll
            for (int l = 0; l < L; ++l) {
                const Tin* sl = ring + ((size_t)st * L + l) * VS;
#pragma unroll
                for (int jv = 0; jv < NV; ++jv) raw[l][jv] = *reinterpret_cast<const uint4*>(sl + (jv * CTH + tid) * VEC);
            }
#pragma unroll
            for (int l = 0; l < L; ++l) {
                float tm = -INFINITY;
                if (ES == 2) {
                    uint32_t mx = 0xFF80FF80u;
#pragma unroll
                    for (int jv = 0; jv < NV; ++jv) {
                        uint4& r = raw[l][jv];
                        r.x = clamp_bf16x2(r.x); r.y = clamp_bf16x2(r.y);
                        r.z = clamp_bf16x2(r.z); r.w = clamp_bf16x2(r.w);
                        mx = max_nan_bf16x2(mx, max_nan_bf16x2(max_nan_bf16x2(r.x, r.y), max_nan_bf16x2(r.z, r.w)));
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
                tmax[l] = tm;
            }
            // the slice is in registers now: hand the ring stage back to the producer
            __syncwarp();
            if (lane == 0 && !(p.dbg & 32)) mbar_arrive(&c.empty[st]);
            // per-warp max of all rows, the shuffle chains interleaved
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
                for (int l = 0; l < L; ++l) tmax[l] = fmaxf(tmax[l], __shfl_xor_sync(0xffffffffu, tmax[l], o));
            }
#ifdef MSD_PHASE_PROF
            long long ck2 = clock64();
#endif
            if (p.dbg & 8) continue;   // debug: TMA ring only
            if (j >= NR && !p.dbg) {   // slot q (TMEM and wmx) must have been released by the pass-2 warps
                mbar_wait(&c.tm_empty[q], (uint32_t)(((j / NR) - 1) & 1));
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            }
            if (tid == 0) stamp(j, 2);
#ifdef MSD_PHASE_PROF
            long long ck3 = clock64();
#endif
            if (lane == 0) {
#pragma unroll
                for (int l = 0; l < L; ++l) c.wmx[q][l][warp] = tmax[l];
            }
            float Sv[L], Kv[L];
            int am[L];
            float2 yprev[CET / 2];
#pragma unroll
            for (int l = 0; l < L; ++l) {
                // y = z - m_w exactly (bf16 / clamped inputs), e = 2^(y log2 e) on the MUFU; the
                // rest in packed fp32 pairs (FADD2 / FMUL2 / FFMA2): sum e and the KL numerator
                // sum e (y_l - y_{l-1}) = sum e ((z_l - z_{l-1}) - (m_l - m_{l-1}))
                const float2 nm = make_float2(-tmax[l], -tmax[l]);
                const float2 l2e = make_float2(LOG2E, LOG2E);
                const float2 neg1 = make_float2(-1.f, -1.f);
                float e[CET];
                float2 s2 = make_float2(0.f, 0.f), k2 = make_float2(0.f, 0.f);
                am[l] = 0x7fffffff;
#pragma unroll
                for (int pp = 0; pp < CET / 2; ++pp) {
                    const float2 xv = elem_pair<Tin>(raw[l][(2 * pp) / VEC], pp % (VEC / 2));
                    const float2 y = __fadd2_rn(xv, nm);
                    const float2 t = __fmul2_rn(y, l2e);
                    const float2 ev = make_float2(ex2f(t.x), ex2f(t.y));
                    e[2 * pp] = ev.x;
                    e[2 * pp + 1] = ev.y;
                    s2 = __fadd2_rn(s2, ev);
                    if (l > 0) k2 = __ffma2_rn(ev, __ffma2_rn(yprev[pp], neg1, y), k2);
                    yprev[pp] = y;
                    if (GREEDY) {
                        const int k0 = 2 * pp;
                        const int i0 = (int)(base + ((k0 / VEC) * CTH + tid) * VEC + (k0 % VEC));
                        if (xv.x == tmax[l]) am[l] = min(am[l], i0);
                        if (xv.y == tmax[l]) am[l] = min(am[l], i0 + 1);
                    }
                }
                if (q < NT) {
                    tm_st16(tbase + (uint32_t)(q * CET * L + l * CET), e);
                } else {
                    float* xs = xslot + ((size_t)((q - NT) * L + l) * CET) * CTH + tid;
#pragma unroll
                    for (int k = 0; k < CET; ++k) xs[k * CTH] = e[k];
                }
                Sv[l] = s2.x + s2.y;
                Kv[l] = k2.x + k2.y;
            }
#ifdef MSD_PHASE_PROF
            long long ck4 = clock64();
#endif
#pragma unroll
            for (int l = 0; l < L; ++l) {
                Sv[l] = fold4(Sv[l]);
                if (l > 0) Kv[l] = fold4(Kv[l]);
            }
            if (GREEDY) {
#pragma unroll
                for (int l = 0; l < L; ++l) am[l] = warp_min_i(am[l]);
            }
#ifdef MSD_PHASE_PROF
            long long ck5 = clock64();
#endif
            if (j >= R1 && !p.dbg) mbar_wait(&c.r1_empty[r1], (uint32_t)(((j / R1) - 1) & 1));
            if (lane < NSUB) {
#pragma unroll
                for (int l = 0; l < L; ++l) {
                    c.r1S[r1][l][warp][lane] = Sv[l];
                    c.r1K[r1][l][warp][lane] = Kv[l];
                }
                if (GREEDY && lane == 0) {
#pragma unroll
                    for (int l = 0; l < L; ++l) c.r1A[r1][l][warp] = am[l];
                }
            }
#ifdef MSD_PHASE_PROF
            long long ck6 = clock64();
#endif
            tm_wait_st();
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            __syncwarp();
            if (tid == 0) stamp(j, 3);
#ifdef MSD_PHASE_PROF
            if (p.dbg & 64) {   // debug: pass-1 phase cycle profile (register accumulators)
                long long ck7 = clock64();
                pc[0] += ck1 - ck0; pc[1] += ck2 - ck1; pc[2] += ck3 - ck2; pc[3] += ck4 - ck3;
                pc[4] += ck5 - ck4; pc[5] += ck6 - ck5; pc[6] += ck7 - ck6; pc[7] += 1;
            }
#endif
            if (lane == 0) {
                if (!p.dbg) {
                    mbar_arrive(&c.r1_full[r1]);
                    mbar_arrive(&c.tm_full[q]);
                }
            }
        }
#ifdef MSD_PHASE_PROF
        if ((p.dbg & 64) && p.trace && lane == 0)
            for (int k = 0; k < 8; ++k) atomicAdd(p.trace + warp * 8 + k, (unsigned long long)pc[k]);
#endif
    } else if (warp < W_PROD) {
        // ================================================================ pass-2 warps
        // warp NCW + w reads the TMEM lanes / columns written by pass-1 warp w
        const int w = warp - W_P2;
        const uint32_t tbase = c.taddr + ((uint32_t)((w & 3) * 32) << 16) + (uint32_t)((w >> 2) * 256);
        for (int j = 0; j < n_my; ++j) {
            const int q = (int)(j % NR);
            const int r2 = (int)(j % R2);
            mbar_wait(&c.rowf_full[q], (uint32_t)((j / NR) & 1));
            if (w == 0 && lane == 0) stamp(j, 11);
            float rh[L], sc[L];
#pragma unroll
            for (int l = 1; l < L; ++l) {
                rh[l] = c.rowf[q][l][w].rho;
                sc[l] = c.rowf[q][l][w].scale;
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&c.rowf_empty[q]);
            mbar_wait(&c.tm_full[q], (uint32_t)((j / NR) & 1));
            if (w == 0 && lane == 0) stamp(j, 12);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            float ev[L][CET];
            if (q < NT) {
#pragma unroll
                for (int l = 0; l < L; ++l) tm_ld16(tbase + (uint32_t)(q * CET * L + l * CET), ev[l]);
                tm_wait_ld();
            } else {
#pragma unroll
                for (int l = 0; l < L; ++l) {
                    const float* xs = xslot + ((size_t)((q - NT) * L + l) * CET) * CTH + w * 32 + lane;
#pragma unroll
                    for (int k = 0; k < CET; ++k) ev[l][k] = xs[k * CTH];
                }
            }
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive(&c.tm_empty[q]);
            float acc[L];
#pragma unroll
            for (int l = 1; l < L; ++l) {
                float a = 0.f;
#pragma unroll
                for (int k = 0; k < CET; ++k) {
                    a += fmaxf(fmaf(-ev[l - 1][k], rh[l], ev[l][k]), 0.f);
                }
                acc[l] = a;
            }
#pragma unroll
            for (int l = 1; l < L; ++l) acc[l] = fold4(acc[l]);
            if (j >= R2) mbar_wait(&c.r2_empty[r2], (uint32_t)(((j / R2) - 1) & 1));
            if (lane < NSUB) {
#pragma unroll
                for (int l = 1; l < L; ++l) c.r2R[r2][l][w][lane] = acc[l];
            }
            if (lane == 0) {
#pragma unroll
                for (int l = 1; l < L; ++l) c.r2scale[r2][l][w] = sc[l];
            }
            __syncwarp();
            if (w == 0 && lane == 0) stamp(j, 13);
            if (lane == 0) mbar_arrive(&c.r2_full[r2]);
        }
    } else if (warp == W_PROD) {
        // ================================================================ TMA producer
        if (lane == 0) {
            const uint64_t pol = policy_evict_first();
            for (int j = 0; j < n_my; ++j) {
                const int st = (int)(j % S);
                if (j >= S) mbar_wait(&c.empty[st], (uint32_t)(((j / S) - 1) & 1));
                int64_t u, b, i;
                int s;
                item(j, u, s, b, i);
                const int64_t len = max((int64_t)0, min((int64_t)VSe, p.V - (int64_t)s * VSe));
                const uint32_t bytes = (uint32_t)((len * ES) / 16 * 16);
                // the last slice of a row: pad [bulk end, VSe) from the constant pad buffer so
                // the pass-1 loads stay unconditional (the copy engine does the fill)
                const uint32_t pad = (uint32_t)(VSe * ES) - bytes;
                stamp(j, 0);
                mbar_arrive_expect_tx(&c.full[st], (bytes + pad) * L);
#pragma unroll
                for (int l = 0; l < L; ++l) {
                    Tin* dst = ring + ((size_t)st * L + l) * VS;
                    if (bytes) {
                        const Tin* src = reinterpret_cast<const Tin*>(p.lv.ptr[l]) + b * p.lv.bs[l] +
                                         i * p.lv.ld[l] + (int64_t)s * VSe;
                        bulk_g2s(dst, src, bytes, &c.full[st], pol);
                    }
                    if (pad) bulk_g2s(reinterpret_cast<unsigned char*>(dst) + bytes, p.pad, pad, &c.full[st], pol);
                }
            }
        }
    } else if (warp == W_PUB) {
        // ================================================================ publisher
        // lane = 4 * w + t: pass-1 warp w, record t (of NSUB)
        const int w = lane >> 2, t = lane & 3;
        for (int j = 0; j < n_my; ++j) {
            int64_t u, b, i;
            int s;
            item(j, u, s, b, i);
            const int q = (int)(j % NR);
            const int r1 = (int)(j % R1);
            mbar_wait(&c.r1_full[r1], (uint32_t)((j / R1) & 1));
            float Sw[L], Kw[L], wm[L];
            int aw[L];
#pragma unroll
            for (int l = 0; l < L; ++l) {
                Sw[l] = c.r1S[r1][l][w][t];
                Kw[l] = c.r1K[r1][l][w][t];
                wm[l] = c.wmx[q][l][w];
                aw[l] = (GREEDY && t == 0) ? c.r1A[r1][l][w] : 0x7fffffff;
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&c.r1_empty[r1]);
            // slice combine in fp32 (per-warp factors on the MUFU); the KL numerator is kept
            // relative to the slice shift sigma = m_s,l - m_s,l-1 (restored in float64 by the tail)
            unsigned long long rec[L];
            Partial pr[L];
            float msl[L];
#pragma unroll
            for (int l = 0; l < L; ++l) {
                float ms = wm[l];
#pragma unroll
                for (int o = 16; o > 2; o >>= 1) ms = fmaxf(ms, __shfl_xor_sync(0xffffffffu, ms, o));
                msl[l] = ms;
            }
            float Sx[L], Kx[L];
            int ax[L];
#pragma unroll
            for (int l = 0; l < L; ++l) {
                float f = exp2f_fma((wm[l] - msl[l]) * LOG2E);   // FMA pipe: MUFU is busy
                if (!(wm[l] > NEG_MASKED)) f = (msl[l] > NEG_MASKED) ? 0.f : 1.f;   // fully masked warp
                Sx[l] = Sw[l] * f;
                Kx[l] = 0.f;
                if (l > 0 && f != 0.f) {
                    const float dsh = (wm[l] - wm[l > 0 ? l - 1 : 0]) - (msl[l] - msl[l > 0 ? l - 1 : 0]);
                    Kx[l] = f * fmaf(dsh, Sw[l], Kw[l]);
                }
                ax[l] = (wm[l] == msl[l]) ? aw[l] : 0x7fffffff;
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
                for (int l = 0; l < L; ++l) {
                    Sx[l] += __shfl_xor_sync(0xffffffffu, Sx[l], o);
                    if (l > 0) Kx[l] += __shfl_xor_sync(0xffffffffu, Kx[l], o);
                    if (GREEDY) ax[l] = min(ax[l], __shfl_xor_sync(0xffffffffu, ax[l], o));
                }
            }
#pragma unroll
            for (int l = 0; l < L; ++l) {
                rec[l] = ((unsigned long long)__float_as_uint(Sx[l]) << 32) | __float_as_uint(msl[l]);
                pr[l].m = msl[l];
                pr[l].amax = ax[l];
                pr[l].S = f2d_alu(Sx[l]);
                pr[l].Kl = f2d_alu(Kx[l]);     // relative to the slice shift (see the tail)
            }
            // lane 0 issues every record store and then the counter increment with release
            // semantics, so a fetcher that sees the count complete sees every record
            if (lane == 0) {
#pragma unroll
                for (int l = 0; l < L; ++l) {
                    const size_t idx = ((size_t)u * L + l) * C + s;
                    p.partials[idx] = pr[l];
                    st_relaxed_u64(reinterpret_cast<unsigned long long*>(p.partms) + idx, rec[l]);
                }
                stamp(j, 5);
            }
        }
    } else if (warp >= W_FETCH0 && warp < W_FETCH0 + NFETCH) {
        // ================================================================ fetchers (pass-2 factors)
        const int f = warp - W_FETCH0;
        const int LC = L * C;     // <= FBUF (checked on the host)
        unsigned long long* fb = c.fbuf[f];
        for (int j = f; j < n_my; j += NFETCH) {
            int64_t u, b, i;
            int s;
            item(j, u, s, b, i);
            const int q = (int)(j % NR);
            const uint64_t t0 = globaltimer();
            if (lane == 0) stamp(j, 6);
            if (lane == 0) stamp(j, 7);
            // stage the unit's records; a record whose sum is still 0 is not yet visible
            const unsigned long long* pm = reinterpret_cast<const unsigned long long*>(p.partms) + (size_t)u * LC;
            while (true) {
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
                __nanosleep(32);
            }
            __syncwarp();
            if (lane == 0) stamp(j, 4);
            // row normalisers from the C slice records, all L rows interleaved.  fp32 on the
            // FMA pipe: the slice sums are fp32-accurate already and FP64 is slow on this part.
            float Ml[L], Sl[L];
            {
#pragma unroll
                for (int l = 0; l < L; ++l) Ml[l] = -INFINITY;
                for (int t = lane; t < C; t += 32) {
#pragma unroll
                    for (int l = 0; l < L; ++l) Ml[l] = fmaxf(Ml[l], __uint_as_float((uint32_t)fb[l * C + t]));
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
                    for (int l = 0; l < L; ++l) Ml[l] = fmaxf(Ml[l], __shfl_xor_sync(0xffffffffu, Ml[l], o));
                }
#pragma unroll
                for (int l = 0; l < L; ++l) Sl[l] = 0.f;
                for (int t = lane; t < C; t += 32) {
#pragma unroll
                    for (int l = 0; l < L; ++l) {
                        const unsigned long long r = fb[l * C + t];
                        const float vm = __uint_as_float((uint32_t)r);
                        if (vm > NEG_MASKED)
                            Sl[l] = fmaf(__uint_as_float((uint32_t)(r >> 32)), exp2f_fma((vm - Ml[l]) * LOG2E), Sl[l]);
                    }
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
                    for (int l = 0; l < L; ++l) Sl[l] += __shfl_xor_sync(0xffffffffu, Sl[l], o);
                }
            }
            // per-warp factors: lane = 8 (l - 1) + w for pass-1 warp w and the pair ending at row l
            if (lane == 0) stamp(j, 8);
            if (j >= NR) mbar_wait(&c.rowf_empty[q], (uint32_t)(((j / NR) - 1) & 1));
            if (lane == 0) stamp(j, 9);
            {
                const int w = lane & 7, l = 1 + (lane >> 3);
                if (l < L) {
                    float Ma = Ml[0], Mb = Ml[0], Sa = Sl[0], Sb = Sl[0];
#pragma unroll
                    for (int r = 1; r < L; ++r)
                        if (r == l) { Ma = Ml[r]; Sa = Sl[r]; Mb = Ml[r - 1]; Sb = Sl[r - 1]; }
                    const float wa = c.wmx[q][l][w], wb = c.wmx[q][l - 1][w];
                    const float ca = (wa > NEG_MASKED && Ma > NEG_MASKED) ? exp2f_fma((wa - Ma) * LOG2E) : 0.f;
                    const float cb = (wb > NEG_MASKED && Mb > NEG_MASKED) ? exp2f_fma((wb - Mb) * LOG2E) : 0.f;
                    const bool skip = !(ca > 0.f) || !(Sa > 0.f) || !(Sb > 0.f) || !isfinite(Sa) || !isfinite(Sb);
                    WF wf;
                    // identical rows must give rho = 1 exactly (zero residual), which the
                    // Newton reciprocal alone does not guarantee
                    const float num = cb * Sa, den = Sb * ca;
                    wf.rho = skip ? 0.f : (num == den ? 1.f : num * frcp_fma(den));
                    wf.scale = skip ? 0.f : ca * frcp_fma(Sa);
                    c.rowf[q][l][w] = wf;
                }
            }
            __syncwarp();
            if (lane == 0) {
                stamp(j, 10);
                mbar_arrive(&c.rowf_full[q]);
            }
        }
    } else if (warp == W_RED) {
        // ================================================================ reducer (slice residual)
        const int w = lane >> 2, t = lane & 3;
        for (int j = 0; j < n_my; ++j) {
            int64_t u, b, i;
            int s;
            item(j, u, s, b, i);
            const int r2 = (int)(j % R2);
            mbar_wait(&c.r2_full[r2], (uint32_t)((j / R2) & 1));
            if (lane == 0) stamp(j, 14);
            float R[L];
#pragma unroll
            for (int l = 1; l < L; ++l) {
                float d = c.r2R[r2][l][w][t] * c.r2scale[r2][l][w];
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
                R[l] = d;
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&c.r2_empty[r2]);
            if (lane >= 1 && lane < L) {
                float v = R[1];
#pragma unroll
                for (int l = 2; l < L; ++l)
                    if (lane == l) v = R[l];
                p.resid[((size_t)u * (L - 1) + (lane - 1)) * C + s] = f2d_alu(v);
            }
            if (lane == 0) stamp(j, 15);
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
    const int S = core_stages(L, ES);
    p.stages = S;
    const int nss = core_sslots(L, ES, (int)sizeof(Ctl<L>));
    const size_t smem = align_up(stage_bytes * S, 128) + align_up(sizeof(Ctl<L>), 128) +
                        (size_t)nss * L * CET * CTH * 4 + 128;
    auto k = core_kernel<Tin, L, G>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int dev = 0, nsm = 0, occ = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, CORE_THREADS, smem);
    if (e != cudaSuccess) return e;
    if (occ < 1) return cudaErrorInvalidConfiguration;
    if (L * p.C > FBUF) return cudaErrorInvalidValue;   // vocabulary too large for the exchange buffer
    // one CTA per SM (it owns all 512 TMEM columns); k = floor(nsm / C) groups of C CTAs
    int64_t kg = nsm / p.C;
    if (kg < 1) return cudaErrorInvalidConfiguration;
    if (kg > p.U) kg = p.U;
    const int64_t grid = kg * p.C;
    void* args[] = {&p};
    return cudaLaunchCooperativeKernel((const void*)k, dim3((unsigned)grid), dim3(CORE_THREADS), args, smem, s);
}

// 0xF1 bytes: bf16 0xF1F1 and f32 0xF1F1F1F1 are both ~ -2.4e30, i.e. masked (-inf after the
// -1e30 clamp) -- the fill of a row's last slice beyond the vocabulary
__device__ __align__(128) unsigned char g_pad[VS * 4];

cudaError_t core_pad(const void** out) {
    static bool done[64] = {};
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    void* ptr = nullptr;
    e = cudaGetSymbolAddress(&ptr, g_pad);
    if (e != cudaSuccess) return e;
    if (dev >= 0 && dev < 64 && !done[dev]) {
        e = cudaMemset(ptr, 0xF1, sizeof(g_pad));
        if (e != cudaSuccess) return e;
        e = cudaDeviceSynchronize();
        if (e != cudaSuccess) return e;
        done[dev] = true;
    }
    *out = ptr;
    return cudaSuccess;
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
