// msd_rollback.cu -- row a7: batched paged-KV rollback (§4.4).
//
// Step 1 of the paper (logical rollback, Eq. 8) becomes `seq_len -= r` plus the
// optional clearing of cache_mask[b, new:old); step 2 (physical truncation, Eq. 9)
// becomes the release of every whole 16-token block past the new length, per
// sequence (strictly more reclaiming than the batch-common r_min tail).  One CTA
// per model; the release order (request-major, ascending block) comes from a
// block-wide exclusive scan, so the free stack is deterministic.
#include "msd_common.cuh"
#include "msd_internal.h"

namespace msd {

constexpr int RT = 1024;

__global__ void __launch_bounds__(RT) rollback_kernel(RollbackParams p) {
    const msd_paged_kv kv = p.kv[blockIdx.x];
    const int32_t* r = p.rollback + (size_t)blockIdx.x * p.B;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int bs = kv.block_size;
    __shared__ int32_t wsum[RT / 32];
    __shared__ int32_t s_carry, s_total;
    if (tid == 0) s_total = 0;
    __syncthreads();

    // a request is left untouched (ROLLBACK_OVF) when r is negative, exceeds its length, or its
    // length claims more blocks than its block-table row holds (an inconsistent caller state)
    const int64_t cap_tokens = (int64_t)kv.max_blocks * bs;
    // pass A: total number of blocks released by this model
    int32_t tot = 0;
    for (int b = tid; b < p.B; b += RT) {
        const int32_t old = kv.seq_len[b], rb = r[b];
        if (rb < 0 || rb > old || old > cap_tokens) continue;
        const int32_t nw = old - rb;
        tot += (old + bs - 1) / bs - (nw + bs - 1) / bs;
    }
    atomicAdd(&s_total, tot);
    __syncthreads();
    const int32_t fc0 = *kv.free_count;
    const bool can_free = (int64_t)fc0 + s_total <= (int64_t)kv.free_cap;

    // pass B: chunks of RT requests, exclusive scan of released-block counts
    if (tid == 0) s_carry = 0;
    __syncthreads();
    for (int c0 = 0; c0 < p.B; c0 += RT) {
        const int b = c0 + tid;
        int32_t old = 0, nw = 0, n = 0;
        bool valid = false;
        if (b < p.B) {
            old = kv.seq_len[b];
            const int32_t rb = r[b];
            valid = rb >= 0 && rb <= old && old <= cap_tokens;
            if (valid) {
                nw = old - rb;
                n = (old + bs - 1) / bs - (nw + bs - 1) / bs;
            }
        }
        int32_t incl = n;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int32_t t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += t;
        }
        if (lane == 31) wsum[warp] = incl;
        __syncthreads();
        int32_t woff = 0;
        for (int wi = 0; wi < warp; ++wi) woff += wsum[wi];
        const int32_t off = s_carry + woff + incl - n;
        if (b < p.B) {
            if (!valid) {
                atomicOr(&p.flags[b], (uint32_t)MSD_F_ROLLBACK_OVF);
            } else if (nw != old) {
                if (kv.cache_mask)
                    for (int32_t j = nw; j < old && j < kv.mask_ld; ++j)
                        kv.cache_mask[(size_t)b * kv.mask_ld + j] = 0;
                const int32_t j0 = (nw + bs - 1) / bs;
                if (n > 0) {
                    if (can_free) {
                        for (int32_t k = 0; k < n; ++k) {
                            int32_t* slot = kv.block_table + (size_t)b * kv.max_blocks + j0 + k;
                            kv.free_ids[fc0 + off + k] = *slot;
                            *slot = -1;
                        }
                    } else {
                        atomicOr(&p.flags[b], (uint32_t)MSD_F_FREELIST_OVF);
                    }
                }
                kv.seq_len[b] = nw;
            }
        }
        __syncthreads();
        if (tid == RT - 1) s_carry += woff + incl;
        __syncthreads();
    }
    if (tid == 0 && can_free) *kv.free_count = fc0 + s_total;
}

cudaError_t launch_rollback(const RollbackParams& p, cudaStream_t s) {
    if (p.B <= 0 || p.n_models <= 0) return cudaSuccess;
    rollback_kernel<<<p.n_models, RT, 0, s>>>(p);
    return cudaGetLastError();
}

}  // namespace msd
