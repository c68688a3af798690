/*
 * msd_oracle.c -- plain, slow, obviously-correct float64 CPU oracle.
 *
 * TEST INFRASTRUCTURE ONLY (see msd_oracle.h).  It follows the paper step by
 * step: no blocking, no fusion, no reordering beyond what the cited
 * definition states.  Shares no code with the CUDA product.
 *
 * Notation: level 0 = drafter M_1, level L-1 = target M_t.
 * p_l[i] = softmax(Z_l[i]) (Eq. 1).
 */
#include "msd_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* Neumaier-compensated running sum (so the oracle's sums are ~exact in f64). */
typedef struct { double s, c; } nsum;
static void ns_add(nsum* a, double x) {
    double t = a->s + x;
    if (fabs(a->s) >= fabs(x)) a->c += (a->s - t) + x;
    else                        a->c += (x - t) + a->s;
    a->s = t;
}
static double ns_get(const nsum* a) { return a->s + a->c; }

/* Eq. 1: the softmax normaliser  LSE = log sum_v exp(z_v), computed as
 * max + log(sum exp(z - max)).  Returns -inf for an all -inf row and NaN when the
 * row holds NaN or +inf (not a distribution). */
double or_lse(const double* z, int64_t V) {
    double m = -INFINITY;
    for (int64_t v = 0; v < V; ++v) {
        if (isnan(z[v]) || z[v] == INFINITY) return NAN;
        if (z[v] > m) m = z[v];
    }
    if (m == -INFINITY) return -INFINITY;
    nsum s = {0.0, 0.0};
    for (int64_t v = 0; v < V; ++v) ns_add(&s, exp(z[v] - m));
    return m + log(ns_get(&s));
}

/* Greedy rule ("greedy"): index of the maximum, ties -> lowest id. */
int64_t or_argmax(const double* z, int64_t V) {
    int64_t best = 0;
    for (int64_t v = 1; v < V; ++v)
        if (z[v] > z[best]) best = v;
    return best;
}

/* Eq. 5 literally: DTV(p,q) = 1/2 sum_v |p(v) - q(v)|. */
double or_dtv(const double* za, double A, const double* zb, double B, int64_t V) {
    nsum s = {0.0, 0.0};
    for (int64_t v = 0; v < V; ++v) ns_add(&s, fabs(exp(za[v] - A) - exp(zb[v] - B)));
    return 0.5 * ns_get(&s);
}

/* KL(p_a || p_b) in nats (BASELINE.json north_star "KL and total variation";
 * DESIGN.md reading R9: verifier || proposer).  Terms with p_a(v) = 0 contribute 0
 * (0 log 0 = 0); p_a(v) > 0 with p_b(v) = 0 gives +inf. */
double or_kl(const double* za, double A, const double* zb, double B, int64_t V) {
    nsum s = {0.0, 0.0};
    for (int64_t v = 0; v < V; ++v) {
        double p = exp(za[v] - A);
        if (p == 0.0) continue;
        if (zb[v] == -INFINITY) return INFINITY;
        ns_add(&s, p * ((za[v] - A) - (zb[v] - B)));
    }
    return ns_get(&s);
}

/* Probabilistic acceptance (cites [leviathan2023fast]; rule as in S:349-350):
 * accept the drafted token t iff u < min(1, p(t)/q(t)).  p(t)/q(t) is evaluated as
 * exp(log p(t) - log q(t)).  q(t) = 0: accept iff p(t) > 0.
 * near_tie is set when |u - min(1,p/q)| < tie_eps (caller passes the eps via the
 * global below; reading R18). */
static double g_tie_eps = 1e-6;       /* acceptance band (north star: |u - p/q| < 1e-6) */
static double g_tie_eps_draw = 1e-6;  /* inverse-CDF band |u - C/Z| (reading R18) */
int or_accept(double za_t, double A, double zb_t, double B, double u, int* near_tie) {
    if (za_t == -INFINITY) {               /* p(t) = 0: never accepted (u >= 0) */
        if (near_tie && u < g_tie_eps) *near_tie = 1;
        return 0;
    }
    if (zb_t == -INFINITY) return 1;       /* q(t) = 0 < p(t): ratio +inf */
    double lr = (za_t - A) - (zb_t - B);
    double r = lr >= 0.0 ? 1.0 : exp(lr);  /* min(1, p/q) */
    if (near_tie && fabs(u - r) < g_tie_eps) *near_tie = 1;
    return u < r;
}

/* Inverse-CDF draw over an (unnormalised) non-negative weight vector w (S:79
 * "inverse-CDF over the vector"; reading R5): with C_t = sum_{v<=t} w_v and
 * Z = C_{V-1}, return min{t : C_t > u*Z}; if no such t (rounding) return the last t
 * with w_t > 0.  near_tie when u is within tie_eps of C_{t-1}/Z or C_t/Z. */
static int64_t inv_cdf(const double* w, int64_t V, double Z, double u, int* near_tie) {
    double target = u * Z;
    nsum c = {0.0, 0.0};
    int64_t last_pos = -1;
    double prev = 0.0;
    for (int64_t t = 0; t < V; ++t) {
        if (w[t] > 0.0) last_pos = t;
        ns_add(&c, w[t]);
        double ct = ns_get(&c);
        if (ct > target && w[t] > 0.0) {
            if (near_tie && (fabs(u - prev / Z) < g_tie_eps_draw || fabs(u - ct / Z) < g_tie_eps_draw))
                *near_tie = 1;
            return t;
        }
        prev = ct;
    }
    if (near_tie) *near_tie = 1;   /* fell off the end: u*Z >= computed total */
    return last_pos < 0 ? 0 : last_pos;
}

/* Draw from p = softmax(z) (bonus token P:65). */
int64_t or_sample(const double* z, double A, int64_t V, double u, int* near_tie) {
    double* w = (double*)malloc(sizeof(double) * (size_t)V);
    nsum s = {0.0, 0.0};
    for (int64_t v = 0; v < V; ++v) { w[v] = exp(z[v] - A); ns_add(&s, w[v]); }
    int64_t t = inv_cdf(w, V, ns_get(&s), u, near_tie);
    free(w);
    return t;
}

/* Residual draw after a rejection ("probabilistic acceptance", rule S:94-102):
 * sample from normalize(max(p - q, 0)); if the residual mass is < 1e-12, sample
 * from p instead (S:97 degenerate fallback) and set *small. */
int64_t or_sample_residual(const double* za, double A, const double* zb, double B,
                           int64_t V, double u, int* near_tie, int* small) {
    double* w = (double*)malloc(sizeof(double) * (size_t)V);
    nsum s = {0.0, 0.0};
    for (int64_t v = 0; v < V; ++v) {
        double r = exp(za[v] - A) - exp(zb[v] - B);
        w[v] = r > 0.0 ? r : 0.0;
        ns_add(&s, w[v]);
    }
    double Z = ns_get(&s);
    int64_t t;
    if (Z < 1e-12) {
        if (small) *small = 1;
        t = or_sample(za, A, V, u, near_tie);
    } else {
        t = inv_cdf(w, V, Z, u, near_tie);
    }
    free(w);
    return t;
}

/* ------------------------------------------------------------------ */
/* The cascade for one request: S:346-363 (verify_level / run_cycle)
 * (SD steps 3-4), P:247 (VerifyProcessor "repeats for each verification level"),
 * P:249 (rollback "based on consensus").  Level l >= 1 verifies candidates c_l
 * against the proposal density p_{l-1} at the same row (reading R7). */

typedef struct {
    const or_level* lv; int32_t L, K; int64_t V; int64_t b;
    double* lse;      /* [L][K+L] cache, NaN = not yet computed */
    int32_t rows_max;
    uint32_t flags;
} req_ctx;

static const double* row(const req_ctx* c, int32_t l, int32_t i) {
    return c->lv[l].z + c->b * c->lv[l].bstride + (int64_t)i * c->lv[l].ld;
}
static double row_lse(req_ctx* c, int32_t l, int32_t i) {
    double* slot = &c->lse[(int64_t)l * c->rows_max + i];
    if (isnan(*slot)) {
        double A = or_lse(row(c, l, i), c->V);
        if (!isfinite(A)) {                 /* NaN/+inf row or all -inf row */
            c->flags |= OR_F_NONFINITE;
            if (isnan(A)) A = -INFINITY;    /* keep the cache slot marked as computed */
        }
        *slot = A;
    }
    return *slot;
}

static int32_t lcp(const int32_t* a, int32_t na, const int32_t* b, int32_t nb) {
    int32_t n = 0;
    while (n < na && n < nb && a[n] == b[n]) ++n;
    return n;
}

static void chain_one(const or_level* lv, int32_t L, int32_t B, int32_t K, int64_t V, int64_t b,
                      const int32_t* cand0, const int32_t* m0,
                      const float* u_acc, const float* u_emit, int64_t u_lstride, int64_t u_bstride,
                      int32_t greedy, int32_t intermediate_bonus, int32_t final_bonus, int32_t draft_fed,
                      int32_t* n_acc, int32_t* m_cand, int32_t* out_tok, int32_t out_ld,
                      int32_t* out_len, int32_t* rollback, double* pos_dtv, double* pos_kl,
                      int32_t* near_tie, uint32_t* flags) {
    const int32_t cap = K + L;
    req_ctx ctx;
    ctx.lv = lv; ctx.L = L; ctx.K = K; ctx.V = V; ctx.b = b; ctx.flags = 0;
    ctx.rows_max = cap;
    ctx.lse = (double*)malloc(sizeof(double) * (size_t)L * (size_t)cap);
    for (int64_t j = 0; j < (int64_t)L * cap; ++j) ctx.lse[j] = NAN;

    int32_t* c = (int32_t*)malloc(sizeof(int32_t) * (size_t)cap * (size_t)(L + 1));
    int32_t* cl = c;            /* c_l lists: level l's candidates at cl + l*cap */
    int32_t* m = (int32_t*)calloc((size_t)(L + 1), sizeof(int32_t));
    int32_t first_tie = 0;

    /* c_1 = draft tokens x ("draft on M_1 -> verify_level through M_2..M_N") */
    m[1] = m0 ? m0[b] : K;
    for (int32_t i = 0; i < m[1]; ++i) cl[1 * cap + i] = cand0[b * K + i];

    for (int32_t l = 1; l < L; ++l) {
        /* Divergence of the adjacent pair (l-1, l) at every draft position i < K
         * (Eq. 5, Eq. 6 input; reading R10: path-independent, all i < K). */
        for (int32_t i = 0; i < K; ++i) {
            double A = row_lse(&ctx, l, i), Bq = row_lse(&ctx, l - 1, i);
            double d = or_dtv(row(&ctx, l, i), A, row(&ctx, l - 1, i), Bq, V);
            double kl = or_kl(row(&ctx, l, i), A, row(&ctx, l - 1, i), Bq, V);
            if (isinf(kl)) ctx.flags |= OR_F_KL_INF;
            if (pos_dtv) pos_dtv[((int64_t)(l - 1) * B + b) * K + i] = d;
            if (pos_kl)  pos_kl[((int64_t)(l - 1) * B + b) * K + i] = kl;
        }

        /* Sequential verification; stop at the first rejection. */
        const int32_t* cc = cl + l * cap;
        int32_t mm = m[l], n = mm;
        int tie = 0;
        for (int32_t i = 0; i < mm; ++i) {
            int32_t t = cc[i];
            int acc;
            if (t < 0 || t >= V) { ctx.flags |= OR_F_TOKEN_OOB; acc = 0; }
            else if (greedy) {
                /* greedy: accepted iff it equals the verifier's argmax */
                acc = (or_argmax(row(&ctx, l, i), V) == t);
            } else {
                double A = row_lse(&ctx, l, i), Bq = row_lse(&ctx, l - 1, i);
                double u = (double)u_acc[(int64_t)(l - 1) * u_lstride + b * u_bstride + i];
                acc = or_accept(row(&ctx, l, i)[t], A, row(&ctx, l - 1, i)[t], Bq, u, &tie);
            }
            if (!acc) { n = i; break; }
        }
        if (n_acc) n_acc[(int64_t)(l - 1) * B + b] = n;
        if (m_cand) m_cand[(int64_t)(l - 1) * B + b] = mm;

        /* Emission: replacement on rejection (S:349 residual), else bonus (
         * intermediate levels per reading R8). */
        int32_t* nxt = cl + (l + 1) * cap;
        for (int32_t i = 0; i < n; ++i) nxt[i] = cc[i];
        int emit = 0;
        int32_t y = -1;
        int32_t at = n;
        const int is_final = (l == L - 1);
        if (n < mm) {
            emit = 1;
            if (greedy) y = (int32_t)or_argmax(row(&ctx, l, n), V);
            else {
                double A = row_lse(&ctx, l, n), Bq = row_lse(&ctx, l - 1, n);
                double u = (double)u_emit[(int64_t)(l - 1) * u_lstride + b * u_bstride + n];
                int small = 0;
                y = (int32_t)or_sample_residual(row(&ctx, l, n), A, row(&ctx, l - 1, n), Bq, V, u,
                                                &tie, &small);
                if (small) ctx.flags |= OR_F_RESID_SMALL;
            }
        } else if (is_final ? final_bonus : intermediate_bonus) {
            emit = 1;
            if (greedy) y = (int32_t)or_argmax(row(&ctx, l, mm), V);
            else {
                double A = row_lse(&ctx, l, mm);
                double u = (double)u_emit[(int64_t)(l - 1) * u_lstride + b * u_bstride + mm];
                y = (int32_t)or_sample(row(&ctx, l, mm), A, V, u, &tie);
            }
        }
        if (emit) { nxt[at] = y; m[l + 1] = n + 1; }
        else      { m[l + 1] = mm; for (int32_t i = n; i < mm; ++i) nxt[i] = cc[i]; }
        if (tie && !first_tie) first_tie = l;
    }

    /* Commit = the target's emission. */
    const int32_t* commit = cl + L * cap;
    const int32_t clen = m[L];
    if (out_len) out_len[b] = clen;
    if (out_tok) {
        for (int32_t j = 0; j < out_ld; ++j) out_tok[b * out_ld + j] = j < clen ? commit[j] : -1;
    }
    /* Per-model rollback: r = tokens appended this cycle minus those
     * that stay a prefix of the committed emission.  Drafter: its first draft_fed
     * draft tokens; verifier l: the candidates c_l it was fed. */
    if (rollback) {
        int32_t d = draft_fed;
        rollback[b] = d - lcp(cand0 + b * K, d, commit, clen);
        for (int32_t l = 1; l < L; ++l)
            rollback[(int64_t)l * B + b] = m[l] - lcp(cl + l * cap, m[l], commit, clen);
    }
    if (near_tie) near_tie[b] = first_tie;
    if (flags) flags[b] = ctx.flags;
    free(ctx.lse); free(c); free(m);
}

int or_chain_verify(const or_level* lv, int32_t L, int32_t B, int32_t K, int64_t V,
                    const int32_t* cand0, const int32_t* m0,
                    const float* u_acc, const float* u_emit, int64_t u_lstride, int64_t u_bstride,
                    int32_t greedy, int32_t intermediate_bonus, int32_t final_bonus,
                    int32_t draft_fed, double tie_eps, double tie_eps_draw,
                    int32_t* n_acc, int32_t* m_cand, int32_t* out_tok, int32_t out_ld,
                    int32_t* out_len, int32_t* rollback, double* pos_dtv, double* pos_kl,
                    int32_t* near_tie, uint32_t* flags, int32_t nthreads) {
    if (L < 2 || B < 0 || K < 1 || V < 1 || !lv || !cand0) return 1;
    if (!greedy && (!u_acc || !u_emit)) return 1;
    g_tie_eps = tie_eps > 0 ? tie_eps : 1e-6;
    g_tie_eps_draw = tie_eps_draw > 0 ? tie_eps_draw : g_tie_eps;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 1)
#endif
    for (int64_t b = 0; b < B; ++b)
        chain_one(lv, L, B, K, V, b, cand0, m0, u_acc, u_emit, u_lstride, u_bstride, greedy,
                  intermediate_bonus, final_bonus, draft_fed, n_acc, m_cand, out_tok, out_ld,
                  out_len, rollback, pos_dtv, pos_kl, near_tie, flags);
    return 0;
}

/* ------------------------------------------------------------------ */
/* Rollback, paper view: step 1 logical rollback clears the last r_b
 * valid mask entries of row b (Eq. 8 uses the mask); step 2 physical truncation
 * drops the trailing columns that are 0 in every row (Eq. 9 with r_min read as the
 * longest all-zero tail, S:261 / reading R14). */
void or_rollback_mask(uint8_t* mask, int32_t B, int32_t cap, int32_t* L_phys,
                      const int32_t* r, uint32_t* flags) {
    for (int32_t b = 0; b < B; ++b) {
        uint8_t* rowm = mask + (int64_t)b * cap;
        int32_t valid = 0;
        for (int32_t j = 0; j < *L_phys; ++j) valid += rowm[j] ? 1 : 0;
        if (r[b] > valid) { if (flags) flags[b] |= OR_F_ROLLBACK_OVF; continue; }
        int32_t cleared = 0;
        for (int32_t j = *L_phys - 1; j >= 0 && cleared < r[b]; --j)
            if (rowm[j]) { rowm[j] = 0; ++cleared; }
    }
    int32_t Lp = *L_phys;
    while (Lp > 0) {
        int all_zero = 1;
        for (int32_t b = 0; b < B; ++b) if (mask[(int64_t)b * cap + Lp - 1]) { all_zero = 0; break; }
        if (!all_zero) break;
        --Lp;
    }
    *L_phys = Lp;
}

/* Rollback, paged view (reading R14/R16: prefix mask == seq_len): new = seq_len - r;
 * blocks j in [ceil(new/bs), ceil(old/bs)) are released in request-major, ascending-j
 * order onto the free stack and their table entries set to -1; the optional mask
 * row is cleared on [new, old).  If the batch's released blocks would exceed the
 * free stack, no block is released and every releasing request is flagged. */
void or_rollback_paged(int32_t* seq_len, int32_t* block_table, int32_t B, int32_t max_blocks,
                       int32_t bs, int32_t* free_ids, int32_t* free_count, int32_t free_cap,
                       uint8_t* cache_mask, int32_t mask_ld, const int32_t* r, uint32_t* flags) {
    int64_t total = 0;
    int32_t* newlen = (int32_t*)malloc(sizeof(int32_t) * (size_t)(B > 0 ? B : 1));
    for (int32_t b = 0; b < B; ++b) {
        int32_t old = seq_len[b];
        /* DESIGN.md R22: r < 0, r > seq_len, or seq_len beyond the block-table row (an
         * inconsistent caller state) -> request untouched + ROLLBACK_OVF */
        if (r[b] < 0 || r[b] > old || (int64_t)old > (int64_t)max_blocks * bs) {
            if (flags) flags[b] |= OR_F_ROLLBACK_OVF;
            newlen[b] = old;
            continue;
        }
        newlen[b] = old - r[b];
        int32_t j0 = (newlen[b] + bs - 1) / bs, j1 = (old + bs - 1) / bs;
        total += (j1 - j0);
    }
    int can_free = (*free_count + total <= free_cap);
    for (int32_t b = 0; b < B; ++b) {
        int32_t old = seq_len[b], nw = newlen[b];
        if (nw == old) continue;
        if (cache_mask) for (int32_t j = nw; j < old && j < mask_ld; ++j) cache_mask[(int64_t)b * mask_ld + j] = 0;
        int32_t j0 = (nw + bs - 1) / bs, j1 = (old + bs - 1) / bs;
        if (j1 > j0) {
            if (can_free) {
                for (int32_t j = j0; j < j1; ++j) {
                    free_ids[(*free_count)++] = block_table[(int64_t)b * max_blocks + j];
                    block_table[(int64_t)b * max_blocks + j] = -1;
                }
            } else if (flags) flags[b] |= OR_F_FREELIST_OVF;
        }
        seq_len[b] = nw;
    }
    free(newlen);
}

/* ------------------------------------------------------------------ */
/* Eq. 3 as printed: (1 - alpha^{gamma+1}) / (1 - alpha); alpha = 1 -> gamma+1. */
double or_expected_accepted(double alpha, int32_t gamma) {
    if (alpha >= 1.0) return (double)gamma + 1.0;
    return (1.0 - pow(alpha, gamma + 1)) / (1.0 - alpha);
}
/* Eq. 4: (1 - alpha^{gamma+1}) / ((1 - alpha)(gamma c + 1)). */
double or_theoretical_speedup(double alpha, int32_t gamma, double c) {
    return or_expected_accepted(alpha, gamma) / ((double)gamma * c + 1.0);
}
/* EMA of P:175: T_new = a T_meas + (1 - a) T_old; first observation initialises. */
double or_ema(double old_value, double measured, double weight, int32_t first) {
    if (first) return measured;
    return weight * measured + (1.0 - weight) * old_value;
}

/* Eq. 7 with the continuous acceptance composition of S:457:
 * L_1 = W (the drafter proposes W tokens) and fed_2 = W;
 * L_j = alpha_j (1 - alpha_j^{fed_j}) / (1 - alpha_j)  (= fed_j at alpha_j = 1), the expected
 *       number of the fed_j candidates that level j accepts (a run of Bernoulli(alpha_j) tests
 *       that stops at the first rejection);
 * fed_{j+1} = L_j + 1 with the intermediate bonus: level j always emits one token, the
 *       correction on a rejection or the bonus after a full acceptance;
 * fed_{j+1} = L_j + (1 - alpha_j^{fed_j}) without it: the correction token is still emitted on
 *       a rejection, whose probability is 1 - alpha_j^{fed_j} (continuous extension);
 * tokens per cycle = L_N + 1 (the target's correction or bonus); latency = W T_1 +
 * sum_{j>=2} cost_j with cost_j = T_j (one verify pass, Eq. 4 convention) or W T_j (P:189
 * "W x T_j").  Chain [M_t] alone: T_eff = T_t. */
double or_predict_chain_latency(int32_t N, const double* T, const double* alpha, int32_t W,
                                int32_t verify_linear, int32_t intermediate_bonus) {
    if (N <= 1) return T[0];
    double fed = (double)W;
    double Lj = 0.0;
    double latency = (double)W * T[0];
    for (int32_t j = 1; j < N; ++j) {
        double a = alpha[j - 1];
        double p_all = (a >= 1.0) ? 1.0 : pow(a, fed);       /* all fed candidates accepted */
        Lj = (a >= 1.0) ? fed : a * (1.0 - p_all) / (1.0 - a);
        latency += verify_linear ? (double)W * T[j] : T[j];
        fed = Lj + (intermediate_bonus ? 1.0 : (1.0 - p_all));
    }
    return latency / (Lj + 1.0);
}

/* Alg. 1 by exhaustive enumeration: every strictly increasing
 * subsequence of the capability-sorted pool that ends at the target (P-1), length
 * <= max_len; alpha_{ij} = clamp(SimScore, 0, 1) (S:439 identity mapping, reading
 * R11).  Ties -> shorter chain, then lexicographic ids. */
int32_t or_select_chain(int32_t P, const double* T, const double* sim, int32_t W, int32_t max_len,
                        int32_t verify_linear, int32_t intermediate_bonus,
                        int32_t* chain_out, double* t_eff_out) {
    double best = INFINITY;
    int32_t best_len = 1;
    int32_t best_chain[32];
    best_chain[0] = P - 1;
    best = T[P - 1];                                    /* default [M_t] */
    int32_t nsub = P - 1;                               /* models that may precede the target */
    for (uint32_t mask = 1; mask < (1u << nsub); ++mask) {
        int32_t ch[32], n = 0;
        for (int32_t i = 0; i < nsub; ++i) if (mask & (1u << i)) ch[n++] = i;
        ch[n++] = P - 1;
        if (n > max_len) continue;
        double Tc[32], ac[32];
        for (int32_t j = 0; j < n; ++j) Tc[j] = T[ch[j]];
        for (int32_t j = 1; j < n; ++j) {
            double s = sim[ch[j - 1] * P + ch[j]];
            ac[j - 1] = s < 0 ? 0 : (s > 1 ? 1 : s);
        }
        double t = or_predict_chain_latency(n, Tc, ac, W, verify_linear, intermediate_bonus);
        int better = t < best;
        if (!better && t == best) {
            if (n < best_len) better = 1;
            else if (n == best_len) {
                for (int32_t j = 0; j < n; ++j) {
                    if (ch[j] != best_chain[j]) { better = ch[j] < best_chain[j]; break; }
                }
            }
        }
        if (better) { best = t; best_len = n; memcpy(best_chain, ch, sizeof(int32_t) * (size_t)n); }
    }
    memcpy(chain_out, best_chain, sizeof(int32_t) * (size_t)best_len);
    if (t_eff_out) *t_eff_out = best;
    return best_len;
}

/* SimScore bootstrap ("bootstrap(prefill dists per model) ->
 * initialized pairwise SimScores"; "initial logits used by the scheduler for baseline
 * similarity calculations").  For every pair (i < j) of the N pool models, in lexicographic
 * pair order, and every position k < K of every request b: DTV(p_i, p_j) by Eq. 5 literally
 * (or_dtv) and KL(p_j || p_i) (the later / larger model against the earlier one, the
 * verifier || proposer direction of reading R9, or_kl).  Outputs [npairs][B][K]. */
void or_pool_divergence(const or_level* lv, int32_t N, int32_t B, int32_t K, int64_t V,
                        double* dtv, double* kl) {
    const int32_t np = N * (N - 1) / 2;
#pragma omp parallel for schedule(dynamic)
    for (int64_t bk = 0; bk < (int64_t)B * K; ++bk) {
        const int64_t b = bk / K, k = bk % K;
        double lse[32];
        for (int32_t l = 0; l < N; ++l) lse[l] = or_lse(lv[l].z + b * lv[l].bstride + k * lv[l].ld, V);
        int32_t pi = 0;
        for (int32_t i = 0; i < N; ++i) {
            for (int32_t j = i + 1; j < N; ++j, ++pi) {
                const double* zi = lv[i].z + b * lv[i].bstride + k * lv[i].ld;
                const double* zj = lv[j].z + b * lv[j].bstride + k * lv[j].ld;
                dtv[((int64_t)pi * B + b) * K + k] = or_dtv(zj, lse[j], zi, lse[i], V);
                kl[((int64_t)pi * B + b) * K + k] = or_kl(zj, lse[j], zi, lse[i], V);
            }
        }
        (void)np;
    }
}

/* Draft-side sampling, one draft step for B sequences ("the draft
 * model ... autoregressively generates a sequence of gamma candidate tokens"
 * DraftProcessor; "W sequential next_dist+sample (or argmax in greedy mode)"):
 * row b of z is the drafter's logits for the next token.  token[b] = or_sample (inverse CDF
 * of softmax(z_b) with u[b], reading R5) or or_argmax in greedy mode; lse[b] = log sum exp
 * z_b (Eq. 1); q_tok[b] = softmax(z_b)[token[b]] (the q(x) the verifier's ratio needs).
 * A row whose LSE is not finite (every entry -inf, a NaN, or +inf) gives token -1. */
void or_draft_sample(const double* z, int64_t ld, int32_t B, int64_t V, const float* u,
                     int32_t greedy, double tie_eps_draw, int32_t* token, double* lse,
                     double* q_tok, int32_t* near_tie) {
    g_tie_eps_draw = tie_eps_draw;
#pragma omp parallel for schedule(dynamic)
    for (int32_t b = 0; b < B; ++b) {
        const double* zb = z + (int64_t)b * ld;
        const double A = or_lse(zb, V);
        int nt = 0;
        int64_t t = -1;
        if (isfinite(A)) t = greedy ? or_argmax(zb, V) : or_sample(zb, A, V, (double)u[b], &nt);
        token[b] = (int32_t)t;
        lse[b] = A;
        q_tok[b] = t >= 0 ? exp(zb[t] - A) : NAN;
        near_tie[b] = nt;
    }
}

/* Logits processors top-k / top-p ("sets up sampling parameters
 * (LogitsProcessorList)"; R19 / R23).  The paper names the processor list only; the
 * reading is Hugging Face's TemperatureLogitsWarper -> TopKLogitsWarper -> TopPLogitsWarper order
 * with whole tie groups kept: sort the row's values in descending order;
 *   top-k (0 < k < V): tau_k = the k-th largest value (every entry equal to it is kept);
 *   top-p (0 < p < 1): over softmax(z / T) restricted to the entries z >= tau_k, walk the groups of
 *     equal values from the largest; tau_p = the value of the first group at which the cumulative
 *     mass reaches p * Z (Z = the kept mass), i.e. the smallest top set of mass >= p;
 *   tau = max(tau_k, tau_p); entries z < tau are removed (-inf).  Off: tau = -inf.
 * near = the cumulative mass before or after the chosen group lies within eps * Z of p * Z (the
 * decision is a floating-point tie).  A row holding a NaN or +inf returns NaN (not processed). */
static int cmp_desc(const void* a, const void* b) {
    const double x = *(const double*)a, y = *(const double*)b;
    return (x < y) - (x > y);
}
double or_logits_threshold(const double* z, int64_t V, double T, int32_t top_k, double top_p,
                           double eps, int32_t* near) {
    *near = 0;
    double* s = (double*)malloc(sizeof(double) * (size_t)V);
    for (int64_t v = 0; v < V; ++v) {
        if (isnan(z[v]) || z[v] == INFINITY) { free(s); return NAN; }
        s[v] = z[v];
    }
    qsort(s, (size_t)V, sizeof(double), cmp_desc);
    double tau_k = -INFINITY, tau_p = -INFINITY;
    if (top_k > 0 && top_k < V) tau_k = s[top_k - 1];
    if (top_p > 0.0 && top_p < 1.0 && s[0] > -INFINITY) {
        const double M = s[0];
        double Z = 0.0;
        for (int64_t v = 0; v < V && s[v] >= tau_k; ++v) Z += exp((s[v] - M) / T);
        const double target = top_p * Z;
        double cum = 0.0;
        for (int64_t v = 0; v < V && s[v] >= tau_k;) {
            int64_t e = v;
            while (e < V && s[e] == s[v]) ++e;          /* group of equal values [v, e) */
            const double before = cum;
            cum += (double)(e - v) * exp((s[v] - M) / T);
            if (cum >= target) {
                tau_p = s[v];
                *near = (fabs(cum - target) < eps * Z || fabs(before - target) < eps * Z) ? 1 : 0;
                break;
            }
            v = e;
        }
    }
    free(s);
    return tau_k > tau_p ? tau_k : tau_p;
}
