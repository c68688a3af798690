// msd_internal.h -- host-side launch interfaces between the C ABI (msd_api.cpp)
// and the kernels.  Not part of the public ABI.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/msd.h"

namespace msd {

struct Partial;
struct RowStat;
struct JobBoard;

struct LevelDesc {
    const void* ptr[4];
    int64_t ld[4];
    int64_t bs[4];
    int32_t rows[4];
};

struct CoreParams {
    LevelDesc lv;
    int32_t L, B, K, C, U, VSe;
    uint32_t kinv;      // ceil(2^32 / K): u / K == umulhi(u, kinv) for u < 2^24
    int64_t V;
    int64_t n_items;
    int32_t stages;     // TMA ring stages (host-computed from the shared-memory budget)
    int32_t rs;         // ring row stride in entries (active pass-1 warps x 512)
    int32_t pat_p, pat_t;   // item pattern: of every pat_p items the first pat_t park e in TMEM
    int32_t pf_dist;        // items requested into L2 ahead of their ring copies (0: none)
    Partial* partials;
    float2* partms;     // compact (slice max, slice sum) for the pass-2 exchange
    RowStat* rowstat;
    double* kl;
    double* resid;
    uint32_t* cnt;
    uint32_t* ready;
    uint32_t* flags;
    uint32_t* err;
    JobBoard* board;             // reset by CTA 0 before the roles start (the tail's exact-draw jobs)
    unsigned long long* trace;   // debug: 16 globaltimer stamps per item, or NULL
    int32_t dbg;                 // debug isolation mode (msd_debug_set_knobs): 0 = normal
    float inv_temp;              // 1 / temperature of the logits processor (1 = none)
    const double* lse;           // [L][B][K] producer-supplied row normalisers, or NULL (exchange)
};

// exp of every bf16 value in float64 (65536 entries), filled once per device by msd_init (or
// lazily by the first verify call): `init` = 1 fills it on a private stream and waits for it
cudaError_t exp_table(const double** out, int init);

struct TailParams {
    LevelDesc lv;
    int32_t L, B, K, C, VSe;
    int64_t V;
    const int32_t* cand0;
    const int32_t* m0;
    const float* u_acc;
    const float* u_emit;
    int64_t ua_l, ua_b, ue_l, ue_b;
    int32_t greedy, ibonus, fbonus, draft_fed;
    int32_t* n_acc;
    int32_t* m_cand;
    int32_t* out_tok;
    int32_t out_ld;
    int32_t* out_len;
    int32_t* rollback;
    float* pos_dtv;
    float* pos_kl;
    msd_pair_stats* stats;
    uint32_t* flags;
    const Partial* partials;
    float2* partms;
    const double* resid;
    uint32_t* cnt;
    double z_safe;
    int32_t exact_all;
    int32_t prefetch;   // set by launch_tail: partials + residuals of a request fit in shared memory
    const double* exptab;   // exp of every bf16 value (exact-draw path), from exp_table()
    JobBoard* board;        // exact-draw work sharing (reset by the core kernel)
    float inv_temp;         // 1 / temperature: the tail works on z / T (1 = none)
};

struct PoolParams {          // SimScore bootstrap (msd_pool.cu)
    LevelDesc lv;
    int32_t N, B, K;
    int64_t V;
    float* pos_dtv;
    float* pos_kl;
    msd_pair_stats* stats;
    uint32_t* flags;
};

struct DraftParams {         // draft-side sampling step (msd_draft.cu)
    const void* z;
    int64_t ld, bs;
    int32_t row, B, greedy;
    int64_t V;
    const float* u;
    int32_t* token;
    float* lse;
    float* q_tok;
    uint32_t* flags;
};

struct ProcParams {           // top-k / top-p logits processors (msd_proc.cu)
    const void* in;
    void* out;                // may equal in (in place)
    int64_t in_ld, in_bs, out_ld, out_bs;
    int32_t B, rows;
    int64_t V;
    float inv_temp;           // 1 / T (top-p masses are those of softmax(z / T))
    int32_t top_k;            // 0 = off
    float top_p;              // outside (0, 1) = off
    float* tau;               // [B][rows] or NULL
    uint32_t* flags;          // [B] or NULL
};

struct RollbackParams {
    msd_paged_kv kv[8];
    int32_t n_models, B;
    const int32_t* rollback;
    uint32_t* flags;
};

struct LmHeadParams {        // fused lm_head GEMM + row normaliser (msd_lmhead.cu)
    const void* H;           // [M][D] bf16
    const void* W;           // [V][D] bf16
    int32_t M, D;
    int64_t V;
    const int32_t* cand;     // [M] or NULL
    float* lse;              // [M] or NULL
    float* z_cand;           // [M] or NULL
    void* ws;
    size_t ws_bytes;
    void* logits;            // [M][ldz] bf16 output (msd_lmhead_logits) or NULL (never written)
    int64_t ldz;
    double* lse64;           // [M] float64 LSE of the written (bf16-rounded) logits, or NULL
};

// Test / diagnostic overrides (msd_debug_set_knobs); the defaults are the release behaviour.
struct DebugKnobs {
    int32_t pat_t = -1, pat_r = -1, stages = -1, core_dbg = 0, exact_draws = 0;
    double z_safe = 0.01;
};
extern DebugKnobs g_knobs;

// Returns cudaSuccess or the launch error.  bf16 = 1 for bf16 logits, 0 for f32.
cudaError_t launch_core(const CoreParams& p, int bf16, int greedy, cudaStream_t s);
cudaError_t launch_tail(const TailParams& p, int bf16, cudaStream_t s);
cudaError_t launch_rollback(const RollbackParams& p, cudaStream_t s);
cudaError_t launch_pool(const PoolParams& p, int bf16, cudaStream_t s);
cudaError_t launch_draft(const DraftParams& p, int bf16, cudaStream_t s);
cudaError_t launch_proc(const ProcParams& p, int bf16, cudaStream_t s);
cudaError_t launch_lmhead(const LmHeadParams& p, cudaStream_t s);
size_t lmhead_workspace(int32_t M, int64_t V, int nsm);

}  // namespace msd
