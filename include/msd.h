/*
 * msd.h -- C ABI of libmsd, the B200-native (sm_100a) hot path of multi-level
 * speculative decoding from arxiv 2505.07680 ("SpecRouter"):
 *   batched verification of draft tokens at every level of a model chain,
 *   token-distribution divergence for the chain scheduler, and paged-KV rollback.
 *
 * Citations: "P:n" = the paper's PAPER.md line n; "S:n" = SPEC.md line n.
 *
 * Conventions (all entry points)
 * ------------------------------
 *  - Plain C types only.  Device arrays are raw device pointers owned by the caller
 *    (libmsd never allocates on the hot path).  `stream` is a cudaStream_t passed
 *    as void* (NULL = the legacy default stream).
 *  - Device entry points only ENQUEUE work on `stream` and return; no host sync.
 *  - Host-detectable argument errors return a non-OK msd_status synchronously,
 *    set msd_last_error() and enqueue nothing.
 *  - Data-dependent problems never abort a launch: they are OR-ed into the
 *    caller's per-request `flags[b]` (MSD_F_* bits); check after synchronising.
 *  - Determinism: identical inputs give bit-identical outputs (fixed reduction
 *    trees; the only atomics are integer adds), independent of how requests are
 *    sharded across GPUs.
 *  - Logits: row-major [B][rows][ld] with the vocabulary contiguous, V <= ld (a
 *    padded lm_head stride is allowed).  For the bulk-copy path every row start
 *    must be 16-byte aligned: ptr % 16 == 0, (ld * elem) % 16 == 0 and
 *    (batch_stride * elem) % 16 == 0, else MSD_E_ALIGN.  Logits <= -1e30 are
 *    treated as -inf (probability 0); NaN or +inf make the row invalid
 *    (MSD_F_NONFINITE).
 *  - Requires an sm_100 device (B200); otherwise MSD_E_ARCH.
 */
#ifndef MSD_H
#define MSD_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MSD_ABI_VERSION 1

typedef enum {
    MSD_OK = 0,
    MSD_E_ARG = 1,        /* null pointer, bad size, K+L > 32, V > ld, L outside [2,4] ... */
    MSD_E_DTYPE = 2,      /* unknown msd_dtype or mixed dtypes across levels            */
    MSD_E_ARCH = 3,       /* current device is not sm_100                              */
    MSD_E_CUDA = 4,       /* a CUDA runtime call failed (message in msd_last_error)    */
    MSD_E_WORKSPACE = 5,  /* ws NULL or ws_bytes < required size                        */
    MSD_E_ALIGN = 6       /* a logit row start is not 16-byte aligned                  */
} msd_status;

typedef enum { MSD_F32 = 0, MSD_BF16 = 1 } msd_dtype;
typedef enum { MSD_STOCHASTIC = 0, MSD_GREEDY = 1 } msd_mode;

/* per-request flag bits, OR-ed into flags[b] by the kernels */
enum {
    MSD_F_NONFINITE = 1,     /* a row used by this request holds NaN/+inf, or is all -inf   */
    MSD_F_TOKEN_OOB = 2,     /* a candidate token is outside [0, V): rejected there         */
    MSD_F_RESID_SMALL = 4,   /* residual mass < 1e-12: drew from p instead           */
    MSD_F_ROLLBACK_OVF = 8,  /* rollback r_b > seq_len_b: request left unchanged    */
    MSD_F_FREELIST_OVF = 16, /* freed blocks would overflow the free stack: none freed      */
    MSD_F_KL_INF = 32,       /* some KL(p_l || p_{l-1}) is +inf (p > 0 where q = 0)         */
    MSD_F_NEAR_TIE = 64,     /* a decision had |u - threshold| < 1e-6 (R18)   */
    MSD_F_EXACT_DRAW = 128,  /* a draw took the exact float64 full-row path                 */
    MSD_F_TIMEOUT = 256      /* internal cross-CTA wait timed out (results invalid)         */
};

/* One chain level's logits.  Element (b, i, v) is at
 * ((const T*)ptr)[b * batch_stride + i * ld + v], T = float or bf16. */
typedef struct {
    const void* ptr;
    int32_t dtype;          /* msd_dtype */
    int32_t rows;           /* rows supplied per request */
    int64_t ld;             /* row stride in elements, >= V */
    int64_t batch_stride;   /* request stride in elements, >= rows * ld */
} msd_logits;

/* Per adjacent model pair (M_{l-1}, M_l) statistics, accumulated (+=) by the
 * kernels with integer atomics: exact, order-independent, so an int64 sum
 * all-reduce across ranks gives bit-identical totals on every rank (P:292
 * "token acceptance counts"; Eq. 5 / Eq. 6 inputs). */
#define MSD_DTV_SCALE 4294967296.0      /* dtv_fx = sum_i llrint(DTV_i * 2^32)            */
#define MSD_KL_SCALE 268435456.0        /* kl_fx  = sum_i llrint(min(KL_i, 2^20) * 2^28)  */
typedef struct {
    int64_t dtv_fx;      /* sum over draft positions of DTV(p_l, p_{l-1}) (Eq. 5), fixed point */
    int64_t kl_fx;       /* sum over draft positions of KL(p_l || p_{l-1}), fixed point         */
    int64_t positions;   /* number of draft positions summed                                    */
    int64_t proposed;    /* candidate tokens offered to level l (sum of m_l)                    */
    int64_t accepted;    /* candidate tokens accepted by level l (sum of n_l)                   */
    int64_t near_ties;   /* decisions with |u - threshold| < 1e-6                               */
    int64_t exact_draws; /* draws that took the exact float64 path                              */
    int64_t kl_inf;      /* positions whose KL was +inf (excluded from kl_fx)                   */
} msd_pair_stats;

/* ---------------------------------------------------------------------------
 * msd_verify_level -- one verification level (P:247 VerifyProcessor).
 *
 * q: proposal rows [B][>=K] (the previous level's distribution at each candidate
 *    position); p: verifier rows [B][>=K+1] (row K = bonus distribution).
 * cand[B][K] (device int32): candidate tokens; m[B] (device, or NULL = K): number
 *    of candidates of request b (0 <= m_b <= K).
 * u_acc[B][K], u_emit[B][K+1] (device float32 in [0,1)): acceptance uniforms and
 *    draw uniforms (slot n for a residual draw after rejecting position n, slot m
 *    for the bonus draw).  Ignored (may be NULL) in MSD_GREEDY mode.
 * Acceptance: token t at position i is accepted iff u_acc < min(1, p_i(t)/q_i(t))
 *    (q(t)=0 -> accept iff p(t)>0); greedy: iff t == argmax p_i
 *    (lowest id on ties).  Verification stops at the first rejection.
 * Emission: rejection at n -> y ~ norm(max(p_n - q_n, 0)) (mass < 1e-12 ->
 *    y ~ p_n); all accepted and emit_bonus -> y ~ p_m.  Greedy: y = argmax.
 *    Draws use the inverse CDF in ascending token order: min{t : C_t > u * Z}.
 * Outputs (device): n_acc[B] accepted prefix length; out_tok[B][K+1] emitted tokens
 *    c[0:n] ++ [y] (pad -1); out_len[B]; pos_dtv/pos_kl[B][K] (or NULL): DTV(p_i,q_i)
 *    (Eq. 5) and KL(p_i || q_i) in nats at every position i < K; stats (or NULL):
 *    one msd_pair_stats, +=; flags[B]: OR-ed MSD_F_* bits (required).
 * ws: device workspace of >= msd_verify_level_workspace(B, K, V) bytes (256-byte aligned), not
 *    modified by the caller between calls.  Its layout depends on (B, K, V): the library zeroes
 *    the exchange-record region (on `stream`) whenever a workspace is used with a shape other
 *    than its previous one, or for the first time, so one maximal workspace may serve calls of
 *    different shapes; calls sharing a workspace must not run concurrently.
 * ------------------------------------------------------------------------- */
msd_status msd_verify_level(msd_logits q, msd_logits p, int32_t B, int32_t K, int64_t V,
                            const int32_t* cand, const int32_t* m,
                            const float* u_acc, const float* u_emit,
                            int32_t mode, int32_t emit_bonus,
                            int32_t* n_acc, int32_t* out_tok, int32_t* out_len,
                            float* pos_dtv, float* pos_kl, msd_pair_stats* stats,
                            uint32_t* flags, void* ws, size_t ws_bytes, void* stream);
size_t msd_verify_level_workspace(int32_t B, int32_t K, int64_t V);

/* ---------------------------------------------------------------------------
 * msd_chain_verify -- collaborative multi-level verification of one speculative
 * cycle for a batch (§4.3; Listing 1 Execute_Speculative_Step).
 *
 * levels[0..L-1]: level 0 = drafter M_1 (rows >= K), level l >= 1 = verifier M_{l+1}
 *    (rows >= K+l with intermediate_bonus, else >= K+1); level L-1 = target M_t.
 *    2 <= L <= 4, K+L <= 32, all levels share V (consistent tokenizer).
 * draft_tok[B][K]: the drafter's tokens x (candidates of level 1).
 * u_acc, u_emit: [L-1][B][K+L-1] float32 (device); level l uses row l-1.
 * Level l verifies its candidates c_l against level l-1's rows at the same
 *    positions, then emits c_{l+1} = c_l[0:n_l] ++ [y_l]; an intermediate
 *    level that accepts everything emits a bonus only if intermediate_bonus,
 *    the target always does.
 * draft_fed in {K-1, K}: speculative KV entries the drafter holds for this cycle.
 * Outputs (device; NULL allowed where marked):
 *    n_acc[L-1][B], m_cand[L-1][B] (NULL ok): accepted prefix / candidates per level;
 *    commit_tok[B][K+L-1] (pad -1), commit_len[B]: the target's emission;
 *    rollback[L][B] (NULL ok): r_b per model = |fed_l| - lcp(fed_l, commit)
 *      ("rollback length for each model based on consensus");
 *    pos_dtv, pos_kl [L-1][B][K] (NULL ok): Eq. 5 DTV and KL(p_l || p_{l-1}) at
 *      every draft position, for every adjacent pair (SimScore input, Eq. 6);
 *    stats[L-1] (NULL ok): per-pair msd_pair_stats, +=;  flags[B]: required.
 * ws: >= msd_chain_verify_workspace(L, B, K, V) bytes; same contract as msd_verify_level's.
 * Equivalence: identical to L-1 sequential msd_verify_level calls where level l's q
 *    rows are level l-1's p rows (tokens, lengths, per-position divergence at i < K).
 * ------------------------------------------------------------------------- */
msd_status msd_chain_verify(const msd_logits* levels, int32_t L, int32_t B, int32_t K, int64_t V,
                            const int32_t* draft_tok, const float* u_acc, const float* u_emit,
                            int32_t mode, int32_t intermediate_bonus, int32_t draft_fed,
                            int32_t* n_acc, int32_t* m_cand, int32_t* commit_tok,
                            int32_t* commit_len, int32_t* rollback, float* pos_dtv, float* pos_kl,
                            msd_pair_stats* stats, uint32_t* flags, void* ws, size_t ws_bytes,
                            void* stream);
size_t msd_chain_verify_workspace(int32_t L, int32_t B, int32_t K, int64_t V);

/* ---------------------------------------------------------------------------
 * msd_chain_verify_proc -- msd_chain_verify with a logits processor (
 * P:150 "LogitsProcessorList"): every level's distribution is softmax(z / T) instead of
 * softmax(z) -- the acceptance ratios, residual / bonus draws, DTV, KL and stats are those of the
 * temperature-scaled distributions; greedy mode is unchanged (argmax z / T = argmax z).  The
 * logits are read once as before (the scale is applied inside the kernels, never written back).
 * proc (host pointer, NULL = msd_chain_verify): temperature in (1e-6, 1e6]; top_k must be 0 and
 * top_p 1 (or <= 0) here (MSD_E_ARG otherwise): top-k / top-p are applied beforehand by
 * msd_logits_process on every level (they remove entries; the temperature stays fused here).  All
 * other arguments as msd_chain_verify.
 * ------------------------------------------------------------------------- */
typedef struct {
    float temperature;   /* T > 0; 1 = no scaling */
    int32_t top_k;       /* 0 = off (msd_chain_verify_proc: only value accepted) */
    float top_p;         /* 1 = off (<= 0 also means off; msd_chain_verify_proc: only value accepted) */
} msd_processors;
msd_status msd_chain_verify_proc(const msd_logits* levels, int32_t L, int32_t B, int32_t K, int64_t V,
                                 const int32_t* draft_tok, const float* u_acc, const float* u_emit,
                                 int32_t mode, int32_t intermediate_bonus, int32_t draft_fed,
                                 int32_t* n_acc, int32_t* m_cand, int32_t* commit_tok,
                                 int32_t* commit_len, int32_t* rollback, float* pos_dtv, float* pos_kl,
                                 msd_pair_stats* stats, uint32_t* flags, void* ws, size_t ws_bytes,
                                 const msd_processors* proc, void* stream);

/* ---------------------------------------------------------------------------
 * msd_chain_verify_lse -- msd_chain_verify when the producer of the logits already knows every
 * draft-position row's normaliser (the lm_head epilogue reduces each row to
 * LSE_r = log sum_v exp z_rv on the fly, Eq. 1).  lse (device float64, [L][B][K]): the
 * natural-log normaliser of rows i < K of every level, of the logits exactly as supplied (T = 1).
 * The core kernel then needs no cross-CTA exchange of slice records: pass 2 (DTV, residual masses)
 * starts as soon as this CTA's pass 1 is done.  Outputs, workspace and every other argument as
 * msd_chain_verify; acceptance, KL and the draws still use the kernels' own float64 normalisers,
 * so a wrong lse changes only DTV and the residual slice masses (caller contract: lse must be the
 * normaliser of the supplied rows to float64 precision).
 * ------------------------------------------------------------------------- */
msd_status msd_chain_verify_lse(const msd_logits* levels, int32_t L, int32_t B, int32_t K, int64_t V,
                                const int32_t* draft_tok, const float* u_acc, const float* u_emit,
                                int32_t mode, int32_t intermediate_bonus, int32_t draft_fed,
                                int32_t* n_acc, int32_t* m_cand, int32_t* commit_tok,
                                int32_t* commit_len, int32_t* rollback, float* pos_dtv, float* pos_kl,
                                msd_pair_stats* stats, uint32_t* flags, void* ws, size_t ws_bytes,
                                const double* lse, void* stream);

/* ---------------------------------------------------------------------------
 * msd_kv_rollback -- batched rollback of each model's paged KV state
 * (§4.4: logical rollback of the last r_b entries, Eq. 8; physical
 * reclamation, Eq. 9, generalised to per-sequence release of whole blocks).
 *
 * kv[n_models] (HOST array of descriptors holding DEVICE pointers):
 *    seq_len[B] (in/out), block_table[B][max_blocks] (in/out; -1 = no block),
 *    free_ids[free_cap] + free_count[1] (in/out free stack), block_size (e.g. 16),
 *    cache_mask[B][mask_ld] (uint8, NULL ok; entries [new, old) are cleared).
 * rollback[n_models][B] (device int32): r_b per model (msd_chain_verify output).
 * Per model and request: new = seq_len - r; blocks j in [ceil(new/bs), ceil(old/bs))
 *    are pushed on the free stack in request-major, ascending-j order and their
 *    table entries set to -1.  r < 0, r > seq_len, or seq_len > max_blocks * block_size
 *    (the request's block-table row cannot hold it): request untouched, MSD_F_ROLLBACK_OVF.  If a model's released blocks would overflow free_cap,
 *    none of its blocks are released (seq_len still shrinks), MSD_F_FREELIST_OVF.
 * flags[B] (device): OR-ed.
 * ------------------------------------------------------------------------- */
typedef struct {
    int32_t* seq_len;
    int32_t* block_table;
    int32_t max_blocks;
    int32_t block_size;
    int32_t* free_ids;
    int32_t* free_count;
    int32_t free_cap;
    int32_t mask_ld;
    uint8_t* cache_mask;
} msd_paged_kv;

msd_status msd_kv_rollback(const msd_paged_kv* kv, int32_t n_models, int32_t B,
                           const int32_t* rollback, uint32_t* flags, void* stream);

/* ---------------------------------------------------------------------------
 * Scheduler feed (host, synchronous, pure).  §4.2 P:170-236.
 *
 * msd_predict_chain_latency: Eq. 7 for chain [M_1..M_N]:
 *    L_1 = W; fed_j = W (j=2) or L_{j-1} (+1 if intermediate_bonus);
 *    L_j = a_j (1 - a_j^fed_j) / (1 - a_j) (= fed_j at a_j = 1);
 *    T_eff = (W T_1 + sum_{j>=2} cost_j) / (L_N + 1), cost_j = T_j (verify_cost 0,
 *    one pass, Eq. 4 convention) or W T_j (verify_cost 1).  N = 1: T_eff = T_1.
 *    T[N] per-token times, alpha[N-1] pair acceptance (alpha[j-1] for (M_j, M_{j+1})).
 * msd_select_chain: Alg. 1 over every capability-ordered subsequence of
 *    the pool 0..P-1 ending at the target P-1 with length <= max_len; alpha_ij =
 *    clamp(sim[i*P+j], 0, 1) (Eq. 2 justifies the identity map); argmin T_eff,
 *    ties -> shorter, then lexicographic; default [M_t].  Writes chain_out (<= 32 ids),
 *    returns its length in *chain_len and its T_eff in *t_eff.
 * msd_simscore_update: Eq. 6 with the EMA of P:175/P:182 from one step's pair stats:
 *    mean DTV = dtv_fx / (positions * 2^32); sim <- w (1 - meanDTV) + (1 - w) sim
 *    (first = 1 initialises).  Returns the new SimScore.
 * ------------------------------------------------------------------------- */
msd_status msd_predict_chain_latency(int32_t N, const double* T, const double* alpha, int32_t W,
                                     int32_t verify_cost, int32_t intermediate_bonus,
                                     double* t_eff);
msd_status msd_select_chain(int32_t P, const double* T, const double* sim, int32_t W,
                            int32_t max_len, int32_t verify_cost, int32_t intermediate_bonus,
                            int32_t* chain_out, int32_t* chain_len, double* t_eff);
double msd_simscore_update(double sim, const msd_pair_stats* step_stats, double weight,
                           int32_t first);

/* ---------------------------------------------------------------------------
 * msd_pool_divergence -- SimScore bootstrap of an N-model pool (
 *    S:472-480 "bootstrap(prefill dists per model) -> initialized pairwise SimScores",
 *    P:152 "initial logits used by the scheduler for baseline similarity calculations").
 *
 * models[N] (HOST array, 2 <= N <= 4, capability order): logits [B][rows >= K][ld] of every
 *    pool model at the same K positions (same dtype, V <= ld, 16-byte aligned rows).
 * For every position (b, k) and pair (i < j), in lexicographic pair order q:
 *    pos_dtv[q][b][k] = DTV(p_i, p_j)  (Eq. 5)    (device f32, NULL ok)
 *    pos_kl[q][b][k]  = KL(p_j || p_i) in nats (reading R9)  (device f32, NULL ok)
 *    stats[q] += int64 fixed-point sums as in msd_chain_verify (device, NULL ok):
 *       SimScore_ij = 1 - dtv_fx / (positions * 2^32) initialises every pair.
 * flags[B] (device, NULL ok): NONFINITE for a row without finite maximum, KL_INF.
 * Asynchronous on `stream`; no workspace.  Not on the per-step path: reads every row twice.
 * ------------------------------------------------------------------------- */
msd_status msd_pool_divergence(const msd_logits* models, int32_t N, int32_t B, int32_t K, int64_t V,
                               float* pos_dtv, float* pos_kl, msd_pair_stats* stats, uint32_t* flags,
                               void* stream);

/* ---------------------------------------------------------------------------
 * msd_draft_sample -- one draft-side sampling step for B sequences (
 *    P:62 "the draft model ... autoregressively generates ... gamma candidate tokens",
 *    P:245 DraftProcessor; "W sequential next_dist+sample (or argmax in greedy
 *    mode)").  Called once per draft step k (the drafter's forward is the caller's).
 *
 * drafter (HOST pointer to one descriptor): logits [B][rows][ld]; row `row` (0 <= row <
 *    rows) of every request is sampled; V <= ld, 16-byte aligned rows, V <= 2^18.
 * u[B] (device f32 in [0,1)): the uniforms, ignored when greedy.
 * token[B] (device int32, required): min{t : C_t > u Z}, C_t = sum_{v<=t} exp(z_v - M),
 *    Z = C_{V-1} (inverse CDF of softmax, reading R5; tokens with p = 0 are never drawn);
 *    greedy: the first argmax.  -1 for a row without a finite LSE (NONFINITE flag).
 * lse[B] (device f32, NULL ok): log sum_v exp z_v (Eq. 1).
 * q_tok[B] (device f32, NULL ok): softmax(z)[token] -- the q(x) of the acceptance ratio.
 * flags[B] (device, NULL ok): |= NONFINITE; NEAR_TIE when u Z is within 1e-6 Z of the drawn
 *    token's CDF boundaries (float64 rescan; the decision can differ from exact arithmetic
 *    only there).  Asynchronous on `stream`; no workspace; one read of each row.
 * ------------------------------------------------------------------------- */
msd_status msd_draft_sample(const msd_logits* drafter, int32_t row, int32_t B, int64_t V,
                            const float* u, int32_t greedy, int32_t* token, float* lse,
                            float* q_tok, uint32_t* flags, void* stream);

/* ---------------------------------------------------------------------------
 * msd_logits_process -- top-k / top-p logits processors ("sets up
 *    sampling parameters (LogitsProcessorList)"; R19 / R23: Hugging Face's
 *    Temperature -> TopK -> TopP warper order, whole tie groups kept).  Per row of one level:
 *    tau_k = the top_k-th largest logit (0 < top_k < V; else -inf); over softmax(z / T) of the
 *    entries z >= tau_k, tau_p = the value at which the cumulative mass of the groups of equal
 *    values, largest first, reaches top_p (0 < top_p < 1; else -inf); tau = max(tau_k, tau_p).
 *    out = z where z >= tau, -inf elsewhere.  Call once per chain level, then
 *    msd_chain_verify_proc with the same temperature (top_k 0, top_p 1) on the outputs.
 * in, out (HOST pointers to one descriptor each; same dtype; out->ptr may equal in->ptr: in
 *    place): rows [0, rows) of every request b < B are processed; V <= ld; 16-byte aligned rows.
 * proc: temperature (the top-p masses), top_k >= 0, top_p.
 * tau[B][rows] (device f32, NULL ok): the threshold (-inf when nothing is removed; NaN for a row
 *    holding NaN or +inf, which is passed through unchanged and flagged NONFINITE).
 * flags[B] (device, NULL ok): |= NONFINITE; NEAR_TIE when the top-p boundary decision lies within
 *    3e-7 Z of top_p Z (the masses are float32 exponentials summed exactly in 2^-40 fixed point,
 *    so the decision can differ from exact arithmetic only there).
 * One CTA per row: radix selection on the order-preserving integer key of the values (2 passes
 *    per selection for bf16, 4 for f32) plus a maximum and a write pass -- every pass after the
 *    first reads the row from L2.  Asynchronous on `stream`; no workspace.
 * ------------------------------------------------------------------------- */
msd_status msd_logits_process(const msd_logits* in, const msd_logits* out, int32_t B, int32_t rows, int64_t V,
                              const msd_processors* proc, float* tau, uint32_t* flags, void* stream);

/* ---------------------------------------------------------------------------
 * msd_lmhead_lse -- the step before the path, fused (Eq. 1
 * "softmax(h_t W)"): for every row r of H the normaliser LSE_r = log sum_v exp(z_rv) of the
 * logits z = H W^T and the candidate's logit z_r,cand[r], computed by a tcgen05 GEMM whose
 * epilogue reduces each accumulator tile on the fly -- the M x V logits are never written.
 * H [M][D] bf16 row-major (hidden states), W [V][D] bf16 row-major (the lm_head weight, nn.Linear
 * layout); D a multiple of 64; 16-byte aligned.  cand [M] int32 (NULL ok; -1 / out of range ->
 * z_cand NaN); outputs lse [M] f32, z_cand [M] f32 (NULL ok).  Arithmetic: bf16 products with
 * fp32 tensor-core accumulation (the logits a bf16 lm_head produces before rounding), online
 * (max, sum) in fp32 per 32 columns and float64 across them.  ws: >= msd_lmhead_workspace(M, V)
 * bytes (per-row partial records).  Asynchronous on `stream`.
 * ------------------------------------------------------------------------- */
size_t msd_lmhead_workspace(int32_t M, int64_t V);
/* msd_lmhead_logits -- the same GEMM when the verify needs the full distributions (DTV, residual
 * draws): the epilogue also writes the logits, rounded to bf16, to logits [M][ldz] (16-byte
 * aligned rows, ldz >= V), and reduces the *written* values, so lse64 [M] (device float64) is the
 * normaliser of exactly the tensor msd_chain_verify_lse then reads (its `lse` input) -- the verify
 * core needs no exchange.  z_cand as msd_lmhead_lse (of the rounded logits); ws as msd_lmhead_lse. */
msd_status msd_lmhead_logits(const void* H, const void* W, int32_t M, int32_t D, int64_t V, const int32_t* cand,
                             void* logits, int64_t ldz, double* lse64, float* z_cand, void* ws, size_t ws_bytes,
                             void* stream);
msd_status msd_lmhead_lse(const void* H, const void* W, int32_t M, int32_t D, int64_t V, const int32_t* cand,
                          float* lse, float* z_cand, void* ws, size_t ws_bytes, void* stream);

/* ---------------------------------------------------------------------------
 * Diagnostics.
 * msd_last_error: thread-local message for the last non-OK status of this thread.
 * msd_prof_enable(1): record CUDA events around every msd_core launch (the
 *    dominant kernel); msd_prof_read: after the stream is synchronised, total
 *    milliseconds and launch count since the last read (then resets).
 * ------------------------------------------------------------------------- */
const char* msd_last_error(void);
int32_t msd_abi_version(void);
/* msd_init: one-time setup of the current device (the float64 exp table of the exact draws,
 * filled on a private stream that is waited for).  Called lazily by the first verify call;
 * call it explicitly before capturing verify calls into a CUDA graph.  Host-synchronous. */
msd_status msd_init(void);
msd_status msd_prof_enable(int32_t on);
msd_status msd_prof_read(double* core_ms, int32_t* core_launches, int32_t* total_launches);
/* msd_debug_set_trace: device buffer of 128 bytes per core item (unit x slice) receiving 16
 * globaltimer stamps of the pipeline stages of each item (NULL disables).  Debug only. */
msd_status msd_debug_set_trace(void* dev_buf, size_t bytes);
/* msd_debug_set_knobs: process-wide test / diagnostic overrides of internal choices (the library
 * reads no environment variables).  pat_t / pat_r: core item pattern (TMEM-parked items, ring-
 * kept items per period; -1 = default); stages: TMA ring depth (-1 = default); core_dbg: core
 * isolation mode (0 = normal; 1 = pass 1 + ring only, results invalid; 4|1 = ring only; bits
 * 8..11 = L2 prefetch distance in items + 1, 0 = the default 2);
 * exact_draws: 1 = every residual / bonus draw takes the float64 exact path; z_safe: residual
 * mass below which a draw takes the exact path (default 0.01, R4; < 0 = default).
 * The outputs are identical for every pattern / stage choice and for exact_draws 0 / 1 outside
 * the documented near-tie bands.  Not thread-safe against concurrent calls. */
msd_status msd_debug_set_knobs(int32_t pat_t, int32_t pat_r, int32_t stages, int32_t core_dbg,
                               int32_t exact_draws, double z_safe);

#ifdef __cplusplus
}
#endif
#endif /* MSD_H */
