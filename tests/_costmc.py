"""Monte-Carlo cascade for pinning Eq. 7 -- test infrastructure.

A cycle of the chain [M_1, ..., M_N]: the drafter proposes W tokens; level j tests the
candidates it is fed in order with independent Bernoulli(alpha_j) acceptances and stops at
the first rejection; an intermediate level then feeds its accepted run plus one
emitted token to the next level (the correction token on a rejection; after a full
acceptance the bonus token only with the intermediate bonus); the target commits its
accepted run + 1 token.  The latency of a cycle is W T_1 + sum_j cost_j (cost_j = T_j, or
W T_j for the linear verify cost of P:189), so T_eff = total latency / total committed tokens.
"""
import numpy as np


def simulate_t_eff(T, alpha, W, verify_linear=False, intermediate_bonus=True, cycles=10_000, seed=0):
    rng = np.random.default_rng(seed)
    N = len(T)
    if N == 1:
        return float(T[0])
    lat = W * T[0] + sum((W * T[j] if verify_linear else T[j]) for j in range(1, N))
    fed = np.full(cycles, W, dtype=np.int64)
    for j in range(1, N):
        a = alpha[j - 1]
        # successes before the first failure of a Bernoulli(a) sequence
        run = rng.geometric(1.0 - a, cycles) - 1 if a < 1.0 else np.full(cycles, 1 << 30)
        acc = np.minimum(run, fed)
        if j < N - 1:
            rejected = acc < fed
            fed = acc + np.where(rejected | bool(intermediate_bonus), 1, 0)
        else:
            committed = acc + 1
    return lat * cycles / float(committed.sum())
