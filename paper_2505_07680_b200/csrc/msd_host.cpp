// msd_host.cpp -- row a8 on the host: the scheduler feed (§4.2).
// Pure, synchronous functions; see include/msd.h for the contract.
#include <cmath>
#include <cstring>

#include "../../include/msd.h"

namespace {

// Eq. 7 with the cascade composition read as in DESIGN.md R12.
double t_eff(int32_t N, const double* T, const double* alpha, int32_t W, int32_t verify_cost,
             int32_t ibonus) {
    if (N <= 1) return T[0];
    double accepted = (double)W;             // L_1 = W
    double latency = (double)W * T[0];       // W x T_1 (drafting)
    for (int32_t j = 1; j < N; ++j) {
        const double fed = (j == 1) ? (double)W : accepted + (ibonus ? 1.0 : 0.0);
        const double a = alpha[j - 1];
        accepted = (a >= 1.0) ? fed : a * (1.0 - std::pow(a, fed)) / (1.0 - a);
        latency += verify_cost ? (double)W * T[j] : T[j];
    }
    return latency / (accepted + 1.0);       // expected target tokens per cycle
}

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

// Alg. 1: candidates = capability-ordered subsequences ending at M_t
// (GenerateCandidateChains), alpha from SimScore (EstimateAcceptanceProb, identity
// clamp), Predict_Effective_Time, argmin with the default [M_t].
msd_status msd_select_chain(int32_t P, const double* T, const double* sim, int32_t W,
                            int32_t max_len, int32_t verify_cost, int32_t intermediate_bonus,
                            int32_t* chain_out, int32_t* chain_len, double* t_best) {
    if (P < 1 || P > 20 || !T || !sim || !chain_out || !chain_len || W < 1 || max_len < 1)
        return MSD_E_ARG;
    int32_t best[32];
    int32_t best_n = 1;
    best[0] = P - 1;
    double best_t = T[P - 1];
    const uint32_t nsub = (uint32_t)(P - 1);
    for (uint32_t mask = 1; mask < (1u << nsub); ++mask) {
        int32_t ch[32], n = 0;
        for (uint32_t i = 0; i < nsub; ++i)
            if (mask & (1u << i)) ch[n++] = (int32_t)i;
        ch[n++] = P - 1;
        if (n > max_len) continue;
        double Tc[32], ac[32];
        for (int32_t j = 0; j < n; ++j) Tc[j] = T[ch[j]];
        for (int32_t j = 1; j < n; ++j) {
            double s = sim[ch[j - 1] * P + ch[j]];
            ac[j - 1] = s < 0.0 ? 0.0 : (s > 1.0 ? 1.0 : s);
        }
        const double t = t_eff(n, Tc, ac, W, verify_cost, intermediate_bonus);
        bool better = t < best_t;
        if (!better && t == best_t) {
            if (n < best_n) better = true;
            else if (n == best_n) {
                for (int32_t j = 0; j < n; ++j)
                    if (ch[j] != best[j]) { better = ch[j] < best[j]; break; }
            }
        }
        if (better) {
            best_t = t;
            best_n = n;
            std::memcpy(best, ch, sizeof(int32_t) * (size_t)n);
        }
    }
    std::memcpy(chain_out, best, sizeof(int32_t) * (size_t)best_n);
    *chain_len = best_n;
    if (t_best) *t_best = best_t;
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
