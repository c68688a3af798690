// msd_host.cpp -- row a8 on the host: the scheduler feed (§4.2).
// Pure, synchronous functions; see include/msd.h for the contract.
#include <algorithm>
#include <cmath>
#include <cstring>

#include "../../include/msd.h"

namespace {

// Expected length of the accepted run when `fed` candidates meet independent acceptance
// tests of probability a that stop at the first rejection: sum_{i=1..fed} a^i,
// continued to real `fed`.  Written as a (1 - a^fed) / (1 - a) via expm1/log.
double accepted_run(double a, double fed) {
    if (a <= 0.0) return 0.0;
    if (a >= 1.0) return fed;
    return a * -std::expm1(fed * std::log(a)) / (1.0 - a);
}

// Eq. 7: expected latency of one cycle over the expected number of target tokens
// it commits.  Level j >= 2 receives `fed` candidates: W from the drafter; from level j-1 its
// accepted run plus the token it emits -- always one with the intermediate bonus, otherwise
// the correction token, emitted only when a candidate was rejected (R12).
double t_eff(int32_t N, const double* T, const double* alpha, int32_t W, int32_t verify_cost,
             int32_t ibonus) {
    if (N <= 1) return T[0];
    double cycle = 0.0, fed = (double)W, run = 0.0;
    for (int32_t j = 0; j < N; ++j) {
        if (j == 0) {                               // drafting: W autoregressive steps of M_1
            cycle += (double)W * T[0];
            continue;
        }
        cycle += verify_cost ? (double)W * T[j] : T[j];
        const double a = alpha[j - 1];
        run = accepted_run(a, fed);
        const double p_reject = (a >= 1.0) ? 0.0 : -std::expm1(fed * std::log(a > 0.0 ? a : 1e-300));
        fed = run + (ibonus ? 1.0 : p_reject);
    }
    return cycle / (run + 1.0);
}

struct Search {                 // Alg. 1 by depth-first enumeration of candidate chains
    int32_t P, W, max_len, verify_cost, ibonus;
    const double* T;
    const double* sim;
    int32_t cur[32];
    int32_t best[32];
    int32_t best_n;
    double best_t;

    // is chain (ch, n) preferred over the incumbent at equal predicted time?  shorter, then
    // lexicographically smaller model ids (SPEC tie rule)
    bool tie_wins(const int32_t* ch, int32_t n) const {
        if (n != best_n) return n < best_n;
        return std::lexicographical_compare(ch, ch + n, best, best + best_n);
    }
    void consider(int32_t n) {
        double Tc[32], ac[32];
        for (int32_t j = 0; j < n; ++j) Tc[j] = T[cur[j]];
        for (int32_t j = 0; j + 1 < n; ++j)
            ac[j] = std::min(1.0, std::max(0.0, sim[cur[j] * P + cur[j + 1]]));   // alpha = clamp(SimScore)
        const double t = t_eff(n, Tc, ac, W, verify_cost, ibonus);
        if (t < best_t || (t == best_t && tie_wins(cur, n))) {
            best_t = t;
            best_n = n;
            std::copy(cur, cur + n, best);
        }
    }
    // models [next, P-1) may still be inserted before the target, in capability order
    void dfs(int32_t depth, int32_t next) {
        cur[depth] = P - 1;
        if (depth + 1 <= max_len) consider(depth + 1);
        if (depth + 2 > max_len) return;
        for (int32_t m = next; m < P - 1; ++m) {
            cur[depth] = m;
            dfs(depth + 1, m + 1);
        }
    }
};

}  // namespace

extern "C" {

msd_status msd_predict_chain_latency(int32_t N, const double* T, const double* alpha, int32_t W,
                                     int32_t verify_cost, int32_t intermediate_bonus,
                                     double* out) {
    if (N < 1 || N > 32 || !T || !out || (N > 1 && !alpha) || W < 1) return MSD_E_ARG;
    for (int32_t j = 0; j < N; ++j)
        if (!(T[j] > 0.0)) return MSD_E_ARG;
    for (int32_t j = 0; j + 1 < N; ++j)
        if (!(alpha[j] >= 0.0 && alpha[j] <= 1.0)) return MSD_E_ARG;
    *out = t_eff(N, T, alpha, W, verify_cost, intermediate_bonus);
    return MSD_OK;
}

// Alg. 1: candidates = capability-ordered subsequences of the pool ending at M_t
// (GenerateCandidateChains), alpha from SimScore (EstimateAcceptanceProb, identity clamp),
// Predict_Effective_Time, argmin; [M_t] alone is the default and always a candidate.
msd_status msd_select_chain(int32_t P, const double* T, const double* sim, int32_t W,
                            int32_t max_len, int32_t verify_cost, int32_t intermediate_bonus,
                            int32_t* chain_out, int32_t* chain_len, double* t_best) {
    if (P < 1 || P > 20 || !T || !sim || !chain_out || !chain_len || W < 1 || max_len < 1)
        return MSD_E_ARG;
    Search s;
    s.P = P; s.W = W; s.max_len = std::min(max_len, 32);
    s.verify_cost = verify_cost; s.ibonus = intermediate_bonus;
    s.T = T; s.sim = sim;
    s.best_n = 1;
    s.best[0] = P - 1;
    s.best_t = T[P - 1];
    s.dfs(0, 0);
    std::copy(s.best, s.best + s.best_n, chain_out);
    *chain_len = s.best_n;
    if (t_best) *t_best = s.best_t;
    return MSD_OK;
}

// Eq. 6: SimScore = 1 - E_EMA[DTV], the EMA weight of P:182.
double msd_simscore_update(double sim, const msd_pair_stats* s, double weight, int32_t first) {
    if (!s || s->positions <= 0) return sim;
    const double mean_dtv = (double)s->dtv_fx / (MSD_DTV_SCALE * (double)s->positions);
    const double obs = 1.0 - mean_dtv;
    return first ? obs : weight * obs + (1.0 - weight) * sim;
}

}  // extern "C"
