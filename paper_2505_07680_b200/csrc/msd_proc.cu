// msd_proc.cu -- top-k / top-p logits processors ("sets up sampling
// parameters (LogitsProcessorList)"; R19 / R23).
//
// Per logit row: the threshold tau (entries z < tau removed, ties at tau kept) of Hugging Face's
// TemperatureLogitsWarper -> TopKLogitsWarper -> TopPLogitsWarper order, then the processed row
// (removed entries = -inf) written to the output (in place allowed).  The verify path then runs on
// the processed rows (msd_chain_verify_proc applies the temperature inside its arithmetic).
//
// One CTA per row, every pass a streaming read of the row (the first from HBM, the rest from L2).
// The threshold is found by radix selection on the order-preserving integer key of the value
// (16-bit for bf16, 32-bit for f32), most significant digit first (10 bits, then the rest):
//   pass 0   row maximum M, non-finite check;
//   top-k    per digit a histogram of counts over the entries matching the digits chosen so far;
//            the bin where the count from the top reaches k (k reduced by the bins above);
//   top-p    the same with masses m = 2^((z - M) log2e / T) of the entries >= tau_k, accumulated
//            as 2^-40 fixed-point integers (exact, order-independent sums: every run takes the same
//            decision), the first level binning the mass exponent instead of a key digit (spreads
//            the bulk of the row over the bins); its total is the kept mass Z, the target p Z;
//   write    z >= tau ? z : -inf.
// Histogram bins are shared-memory integer atomics.  The top-p decision is a floating-point one:
// when the cumulative mass at the chosen key lies within 3e-7 Z of p Z the row is flagged NEAR_TIE.
#include "msd_common.cuh"
#include "msd_internal.h"

namespace msd {

constexpr int PT = 512;                  // threads per CTA
constexpr int PNW = PT / 32;
constexpr int NB = 1024;                 // bins of the first digit
constexpr double MFIX = 1099511627776.0; // 2^40: fixed-point scale of the masses
constexpr double TIE_P = 3e-7;           // top-p boundary tie band (relative to Z): above the worst-case
                                         // error of the masses (ex2.approx 2^-22 relative, 2^-41 fixed point)

template <typename Tin> struct PKey;
template <> struct PKey<__nv_bfloat16> {
    static constexpr int BITS = 16;
    __device__ static uint32_t bits(const __nv_bfloat16* row, int64_t v) {
        return (uint32_t)__bfloat16_as_ushort(row[v]);
    }
    __device__ static float val(uint32_t b) { return __uint_as_float(b << 16); }
    __device__ static uint32_t key(uint32_t b) {          // order-preserving (-0 == +0)
        if (b == 0x8000u) b = 0u;
        return (b & 0x8000u) ? (~b & 0xFFFFu) : (b | 0x8000u);
    }
    __device__ static uint32_t unkey(uint32_t k) { return (k & 0x8000u) ? (k & 0x7FFFu) : (~k & 0xFFFFu); }
    __device__ static void store(__nv_bfloat16* row, int64_t v, uint32_t b) { row[v] = __ushort_as_bfloat16((unsigned short)b); }
    static constexpr uint32_t NEG_INF = 0xFF80u;
};
template <> struct PKey<float> {
    static constexpr int BITS = 32;
    __device__ static uint32_t bits(const float* row, int64_t v) { return __float_as_uint(row[v]); }
    __device__ static float val(uint32_t b) { return __uint_as_float(b); }
    __device__ static uint32_t key(uint32_t b) {
        if (b == 0x80000000u) b = 0u;
        return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
    }
    __device__ static uint32_t unkey(uint32_t k) { return (k & 0x80000000u) ? (k & 0x7FFFFFFFu) : ~k; }
    __device__ static void store(float* row, int64_t v, uint32_t b) { row[v] = __uint_as_float(b); }
    static constexpr uint32_t NEG_INF = 0xFF800000u;
};

struct ProcShared {
    uint32_t cnt[NB];
    unsigned long long mass[NB];
    float red_f[PNW];
    int red_i[PNW];
    uint32_t sel_bin;
    unsigned long long sel_above, sel_in;
    int sel_found;
};

// Every entry of the row visited once per pass by the CTA: f(v, bits) for v < V (16-byte vectors
// where the row allows, scalars at the ragged end).
template <typename Tin, typename F>
__device__ __forceinline__ void for_row(const Tin* row, int64_t V, F f) {
    constexpr int VEC = 16 / (int)sizeof(Tin);
    const int64_t nv = V / VEC;
    const uint4* r4 = reinterpret_cast<const uint4*>(row);
    for (int64_t q = threadIdx.x; q < nv; q += PT) {
        const uint4 w = r4[q];
        const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
        for (int k = 0; k < VEC; ++k) {
            const uint32_t b = sizeof(Tin) == 2 ? ((ws[k / 2] >> (16 * (k & 1))) & 0xFFFFu) : ws[k];
            f(q * VEC + k, b);
        }
    }
    for (int64_t v = nv * VEC + threadIdx.x; v < V; v += PT) f(v, PKey<Tin>::bits(row, v));
}

// Digit d of a key: the first digit is the top 10 bits, then 10-bit digits, the last one shorter.
template <typename Tin>
struct Digits {
    static constexpr int NDIG = (PKey<Tin>::BITS + 9) / 10;
    __device__ static int shift(int d) { return PKey<Tin>::BITS - 10 * (d + 1) < 0 ? 0 : PKey<Tin>::BITS - 10 * (d + 1); }
    __device__ static int width(int d) { return (PKey<Tin>::BITS - 10 * d) < 10 ? PKey<Tin>::BITS - 10 * d : 10; }
};

// Choose, from the top bin down, the bin at which the cumulative value (counts or masses) of the
// bins reaches `target`; `above` = the sum of the bins above it, `in` = the chosen bin's own value.
// Warp 0, fixed order; nb bins.  found = 0 when the total stays below the target.
__device__ void pick_bin(ProcShared& sh, int nb, bool use_mass, unsigned long long target) {
    if (threadIdx.x >= 32) return;
    const int lane = threadIdx.x;
    const int per = (nb + 31) / 32;              // bins per lane, lane 0 owns the TOP bins
    unsigned long long loc = 0;
    for (int q = 0; q < per; ++q) {
        const int bin = nb - 1 - (lane * per + q);
        if (bin >= 0) loc += use_mass ? sh.mass[bin] : (unsigned long long)sh.cnt[bin];
    }
    unsigned long long incl = loc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long x = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += x;
    }
    const unsigned long long excl = incl - loc;
    const bool mine = excl < target && incl >= target;
    const unsigned hit = __ballot_sync(0xffffffffu, mine);
    if (lane == 0) sh.sel_found = hit ? 1 : 0;
    if (mine) {
        unsigned long long c = excl;
        for (int q = 0; q < per; ++q) {
            const int bin = nb - 1 - (lane * per + q);
            if (bin < 0) break;
            const unsigned long long x = use_mass ? sh.mass[bin] : (unsigned long long)sh.cnt[bin];
            if (c + x >= target && x > 0) {
                sh.sel_bin = (uint32_t)bin;
                sh.sel_above = c;
                sh.sel_in = x;
                break;
            }
            c += x;
        }
    }
}

template <typename Tin>
__global__ void __launch_bounds__(PT) proc_kernel(ProcParams p) {
    __shared__ ProcShared sh;
    using K = PKey<Tin>;
    using D = Digits<Tin>;
    const int64_t r = blockIdx.x;                 // row = b * rows + i
    const int64_t b = r / p.rows, i = r % p.rows;
    const Tin* row = reinterpret_cast<const Tin*>(p.in) + b * p.in_bs + i * p.in_ld;
    Tin* out = reinterpret_cast<Tin*>(p.out) + b * p.out_bs + i * p.out_ld;
    const int64_t V = p.V;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    // ---- pass 0: maximum, non-finite entries
    float mx = -INFINITY;
    int bad = 0;
    for_row<Tin>(row, V, [&](int64_t, uint32_t bits) {
        const float z = K::val(bits);
        if (isnan(z) || z == INFINITY) bad = 1;
        mx = fmaxf(mx, z);
    });
    mx = warp_max(mx);
    bad = __any_sync(0xffffffffu, bad);
    if (lane == 0) { sh.red_f[warp] = mx; sh.red_i[warp] = bad; }
    __syncthreads();
    float M = -INFINITY;
    bad = 0;
    for (int w = 0; w < PNW; ++w) { M = fmaxf(M, sh.red_f[w]); bad |= sh.red_i[w]; }
    __syncthreads();

    uint32_t key_tau = 0;                         // keep keys >= key_tau (0: everything)
    bool near = false;
    if (!bad) {
        // ---- top-k: radix selection of the k-th largest key by counts
        uint32_t key_k = 0;
        if (p.top_k > 0 && (int64_t)p.top_k < V) {
            uint32_t prefix = 0;
            unsigned long long target = (unsigned long long)p.top_k;
            for (int d = 0; d < D::NDIG; ++d) {
                const int sh_d = D::shift(d), nb = 1 << D::width(d);
                const int hs = sh_d + D::width(d);          // bits above this digit
                for (int t = threadIdx.x; t < nb; t += PT) sh.cnt[t] = 0u;
                __syncthreads();
                for_row<Tin>(row, V, [&](int64_t, uint32_t bits) {
                    const uint32_t k = K::key(bits);
                    if (hs >= K::BITS || (k >> hs) == (prefix >> hs))
                        atomicAdd(&sh.cnt[(k >> sh_d) & (uint32_t)(nb - 1)], 1u);
                });
                __syncthreads();
                pick_bin(sh, nb, false, target);
                __syncthreads();
                prefix |= sh.sel_bin << sh_d;
                target -= sh.sel_above;
                __syncthreads();
            }
            key_k = prefix;
        }
        // ---- top-p over the entries kept by top-k, by fixed-point masses.  Level A bins the
        // entries by their mass exponent (M - z) log2e / T in NB steps over [0, 40) -- monotone in
        // the value, so every bin is a contiguous key range, and the bulk of a row spreads over
        // many bins (few colliding atomics); masses below 2^-40 are 0 in fixed point and skipped
        // everywhere.  Then the key digits inside the chosen bin.
        uint32_t key_p = 0;
        if (p.top_p > 0.f && p.top_p < 1.f && M > -INFINITY) {
            const float l2s = LOG2E * p.inv_temp, bscale = (float)NB / 40.f;
            auto mass_of = [&](uint32_t bits, int* vb) -> unsigned long long {
                const float x = (M - K::val(bits)) * l2s;        // >= 0
                *vb = (int)fminf(x * bscale, (float)(NB - 1));
                return (unsigned long long)__float2ull_rn(ex2f(-x) * (float)MFIX);
            };
            for (int t = threadIdx.x; t < NB; t += PT) sh.mass[t] = 0ull;
            __syncthreads();
            for_row<Tin>(row, V, [&](int64_t, uint32_t bits) {
                if (K::key(bits) >= key_k) {
                    int vb;
                    const unsigned long long fx = mass_of(bits, &vb);
                    if (fx) atomicAdd(&sh.mass[vb], fx);
                }
            });
            __syncthreads();
            // kept mass Z (fixed order) and the target p Z
            if (threadIdx.x < 32) {
                unsigned long long z = 0;
                for (int t = lane; t < NB; t += 32) z += sh.mass[t];
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) z += __shfl_xor_sync(0xffffffffu, z, o);
                if (lane == 0) sh.sel_above = z;
            }
            __syncthreads();
            const unsigned long long Zfx = sh.sel_above;
            unsigned long long target = (unsigned long long)ceil((double)p.top_p * (double)Zfx);
            if (target == 0) target = 1;
            __syncthreads();
            // bin NB - 1 - vb: pick_bin scans from the top bin (the largest values have vb = 0)
            for (int t = threadIdx.x; t < NB / 2; t += PT) {
                const unsigned long long a = sh.mass[t];
                sh.mass[t] = sh.mass[NB - 1 - t];
                sh.mass[NB - 1 - t] = a;
            }
            __syncthreads();
            pick_bin(sh, NB, true, target);
            __syncthreads();
            const int vsel = NB - 1 - (int)sh.sel_bin;
            target -= sh.sel_above;
            unsigned long long above_total = sh.sel_above;
            __syncthreads();
            uint32_t prefix = 0;
            for (int d = 0; d < D::NDIG; ++d) {
                const int sh_d = D::shift(d), nb = 1 << D::width(d);
                const int hs = sh_d + D::width(d);
                for (int t = threadIdx.x; t < nb; t += PT) sh.mass[t] = 0ull;
                __syncthreads();
                for_row<Tin>(row, V, [&](int64_t, uint32_t bits) {
                    const uint32_t k = K::key(bits);
                    if (k >= key_k && (hs >= K::BITS || (k >> hs) == (prefix >> hs))) {
                        int vb;
                        const unsigned long long fx = mass_of(bits, &vb);
                        if (fx && vb == vsel) atomicAdd(&sh.mass[(k >> sh_d) & (uint32_t)(nb - 1)], fx);
                    }
                });
                __syncthreads();
                pick_bin(sh, nb, true, target);
                __syncthreads();
                prefix |= sh.sel_bin << sh_d;
                target -= sh.sel_above;
                above_total += sh.sel_above;
                if (d == D::NDIG - 1) {
                    // the chosen key's group: mass above it and including it vs p Z
                    const double tgt = (double)p.top_p * (double)Zfx;
                    const double lo = (double)above_total, hi = lo + (double)sh.sel_in;
                    near = fabs(hi - tgt) < TIE_P * (double)Zfx || fabs(lo - tgt) < TIE_P * (double)Zfx;
                }
                __syncthreads();
            }
            key_p = prefix;
        }
        key_tau = key_k > key_p ? key_k : key_p;
    }

    // ---- write the processed row (removed entries -inf); non-finite rows pass through unchanged
    const bool copy = p.out != p.in || !bad;
    if (copy) {
        for_row<Tin>(row, V, [&](int64_t v, uint32_t bits) {
            const bool keep = bad || K::key(bits) >= key_tau;
            if (keep) {
                if (p.out != p.in) K::store(out, v, bits);
            } else {
                K::store(out, v, K::NEG_INF);
            }
        });
    }
    if (threadIdx.x == 0) {
        if (p.tau) p.tau[r] = bad ? NAN : (key_tau == 0 ? -INFINITY : K::val(K::unkey(key_tau)));
        if (p.flags && (bad || near)) atomicOr(&p.flags[b], bad ? (uint32_t)MSD_F_NONFINITE : (uint32_t)MSD_F_NEAR_TIE);
    }
}

cudaError_t launch_proc(const ProcParams& p, int bf16, cudaStream_t s) {
    const int64_t n = (int64_t)p.B * p.rows;
    if (n <= 0) return cudaSuccess;
    if (bf16) proc_kernel<__nv_bfloat16><<<(unsigned)n, PT, 0, s>>>(p);
    else proc_kernel<float><<<(unsigned)n, PT, 0, s>>>(p);
    return cudaGetLastError();
}

}  // namespace msd
