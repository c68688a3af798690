/*
 * msd_oracle.h -- float64 CPU oracle for the multi-level speculative-decoding
 * verify / divergence / KV-rollback path of arxiv 2505.07680 ("SpecRouter").
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no source with the CUDA product (paper_2505_07680_b200/csrc).
 *
 * Citations: "P:n" = PAPER.md line n, "S:n" = SPEC.md line n.
 * Every function follows the paper's definition literally, in float64, one
 * request at a time (OpenMP only across independent requests).
 *
 * Parity pins: see tests/test_oracle_*.py.  Functions marked "parity
 * unpinned" below are definitional choices with no closed form to pin to.
 */
#ifndef MSD_ORACLE_H
#define MSD_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* One chain level's logits: z[b*bstride + i*ld + v], v < V <= ld, i < rows. */
typedef struct {
    const double* z;
    int64_t ld;
    int64_t bstride;
    int32_t rows;
} or_level;

/* per-request flag bits (same meaning as the product's; values restated here) */
#define OR_F_NONFINITE   1u
#define OR_F_TOKEN_OOB   2u
#define OR_F_RESID_SMALL 4u
#define OR_F_ROLLBACK_OVF 8u
#define OR_F_FREELIST_OVF 16u
#define OR_F_KL_INF      32u

/* ---- primitives (Eq. 1, Eq. 5) ---- */
double  or_lse(const double* z, int64_t V);
int64_t or_argmax(const double* z, int64_t V);
double  or_dtv(const double* za, double A, const double* zb, double B, int64_t V);
double  or_kl(const double* za, double A, const double* zb, double B, int64_t V);
int     or_accept(double za_t, double A, double zb_t, double B, double u, int* near_tie);
int64_t or_sample(const double* z, double A, int64_t V, double u, int* near_tie);
int64_t or_sample_residual(const double* za, double A, const double* zb, double B,
                           int64_t V, double u, int* near_tie, int* small);

/* ---- whole cascade ----
 * lv[0] = drafter rows (i < K), lv[l] = level-l verifier rows.
 * cand0[B,K]: candidates fed to level 1 (the draft tokens); m0[B] or NULL (=K).
 * u_acc / u_emit: element (l-1, b, i) at [(l-1)*u_lstride + b*u_bstride + i].
 * Outputs (any may be NULL):
 *   n_acc[(l-1)*B+b], m_cand[(l-1)*B+b]      accepted prefix / candidate count at level l
 *   out_tok[b*out_ld + j], out_len[b]         committed emission of the last level (pad -1)
 *   rollback[l*B+b]                          per-model KV rollback r_b (model l = level l)
 *   pos_dtv/pos_kl[((l-1)*B+b)*K + i]        divergence of pair (l-1,l) at draft position i < K
 *   near_tie[b]                              first level (1-based verifier index l) whose decision
 *                                            was a near tie, else 0: acceptance |u - min(1,p/q)| <
 *                                            tie_eps, draws |u - C/Z| < tie_eps_draw (C = a CDF
 *                                            boundary adjacent to the drawn token)
 *   flags[b]                                 OR_F_* bits
 * Returns 0 on success, nonzero on argument error.
 */
int or_chain_verify(const or_level* lv, int32_t L, int32_t B, int32_t K, int64_t V,
                    const int32_t* cand0, const int32_t* m0,
                    const float* u_acc, const float* u_emit, int64_t u_lstride, int64_t u_bstride,
                    int32_t greedy, int32_t intermediate_bonus, int32_t final_bonus,
                    int32_t draft_fed, double tie_eps, double tie_eps_draw,
                    int32_t* n_acc, int32_t* m_cand, int32_t* out_tok, int32_t out_ld,
                    int32_t* out_len, int32_t* rollback, double* pos_dtv, double* pos_kl,
                    int32_t* near_tie, uint32_t* flags, int32_t nthreads);

/* ---- KV-state rollback, two views (Eq. 8-9) ---- */
/* Paper view: cache_mask[B][cap] (1 = valid), one physical length *L_phys shared by the batch.
 * Clears the last r_b valid entries of row b, then physically truncates the longest
 * all-zero tail.  Returns 0, or sets flags[b] |= OR_F_ROLLBACK_OVF when r_b > L'_b. */
void or_rollback_mask(uint8_t* cache_mask, int32_t B, int32_t cap, int32_t* L_phys,
                      const int32_t* r, uint32_t* flags);
/* Paged view: seq_len[B], block_table[B][max_blocks] (-1 = none), free stack. */
void or_rollback_paged(int32_t* seq_len, int32_t* block_table, int32_t B, int32_t max_blocks,
                       int32_t block_size, int32_t* free_ids, int32_t* free_count, int32_t free_cap,
                       uint8_t* cache_mask, int32_t mask_ld, const int32_t* r, uint32_t* flags);

/* ---- scheduler cost model (Eq. 3, Eq. 4, Eq. 7, Alg. 1) ---- */
double or_expected_accepted(double alpha, int32_t gamma);                 /* Eq. 3 */
double or_theoretical_speedup(double alpha, int32_t gamma, double c);     /* Eq. 4 */
double or_ema(double old_value, double measured, double weight, int32_t first);
double or_predict_chain_latency(int32_t N, const double* T, const double* alpha, int32_t W,
                                int32_t verify_linear, int32_t intermediate_bonus); /* Eq. 7 */
/* Alg. 1: pool models 0..P-1 sorted by capability (ascending), target = P-1.
 * sim[i*P+j] = SimScore(M_i, M_j).  Writes the chosen chain into chain_out (model ids),
 * returns its length.  Ties -> shorter chain, then lexicographic ids. */
int32_t or_select_chain(int32_t P, const double* T, const double* sim, int32_t W, int32_t max_len,
                        int32_t verify_linear, int32_t intermediate_bonus,
                        int32_t* chain_out, double* t_eff_out);

/* SimScore bootstrap: per pool pair (i < j, lexicographic) and position,
 * DTV(p_i, p_j) (Eq. 5) and KL(p_j || p_i); outputs [N(N-1)/2][B][K].  Pinned by
 * tests/test_oracle_pool.py (identical models, hand-computed pair, mixture closed form,
 * adjacent pairs equal or_chain_verify's divergences, scipy KL). */
void or_pool_divergence(const or_level* lv, int32_t N, int32_t B, int32_t K, int64_t V,
                        double* dtv, double* kl);

/* Draft-side sampling: one draft step for B
 * rows z[b * ld + v]: token = inverse-CDF draw from softmax (u[b]) or argmax (greedy), lse,
 * q_tok = softmax(z_b)[token], near_tie = |u - C/Z| < tie_eps_draw at the drawn token's CDF
 * boundaries.  Non-finite LSE -> token -1.  Pinned by tests/test_oracle_draft.py. */
void or_draft_sample(const double* z, int64_t ld, int32_t B, int64_t V, const float* u,
                     int32_t greedy, double tie_eps_draw, int32_t* token, double* lse,
                     double* q_tok, int32_t* near_tie);

/* Logits processors top-k / top-p (R19 / R23): the row's
 * threshold tau (entries z < tau are removed; ties at tau kept), NaN for a row holding NaN / +inf;
 * near = the top-p boundary decision lies within eps * Z of p * Z.  Pinned by
 * tests/test_oracle_proc.py (brute-force subsets, Hugging Face's warpers, closed forms). */
double or_logits_threshold(const double* z, int64_t V, double T, int32_t top_k, double top_p,
                           double eps, int32_t* near);

#ifdef __cplusplus
}
#endif
#endif
