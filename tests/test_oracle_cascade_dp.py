"""Exact law of a 3-level cascade's commit, by dynamic programming over probabilities, against
the oracle's sampled cascade (SURVEY 8(c) "Multi-level cascade" pin; P:60-67, P:247,
S:349-358).

The DP propagates probability mass, not samples: the drafter's tokens x_i ~ q_i; level 2
accepts candidate i with probability min(1, p2_i(x)/q_i(x)) and stops at the first rejection
(P:64), emitting a token from the normalised residual max(p2_n - q_n, 0), or after a
full acceptance a bonus from p2_K (intermediate bonus) or nothing; level 3 repeats this
on level 2's candidates with proposal rows p2 (reading R7) and target rows p3 and always
ends with a correction or bonus token.  Rows are context-free (fixed per position), so the law
of the committed sequence is a finite sum.  The DP itself is pinned by losslessness: the first
committed token is distributed exactly as p3_0 (the target's own first-position law).
"""
import collections
import itertools

import numpy as np
import pytest
import scipy.stats

import oracle as O


def _residual(p, q):
    r = np.maximum(p - q, 0.0)
    z = r.sum()
    return p if z < 1e-12 else r / z          # S:97 fallback (never hit with these rows)


def _level(cands, weight, prop, tgt, bonus, out):
    """Push the law of one level: cands = candidate tuple with probability `weight`; prop /
    tgt = proposal / target rows (by position); adds (emitted tuple -> prob) into out."""
    alive = weight
    for n, t in enumerate(cands):
        a = 1.0 if prop[n][t] == 0 else min(1.0, tgt[n][t] / prop[n][t])
        rej = alive * (1.0 - a)
        if rej > 0:
            for y, py in enumerate(_residual(tgt[n], prop[n])):
                if py > 0:
                    out[cands[:n] + (y,)] += rej * py
        alive *= a
    if alive > 0:
        if bonus:
            for y, py in enumerate(tgt[len(cands)]):
                if py > 0:
                    out[cands + (y,)] += alive * py
        else:
            out[cands] += alive


def exact_commit_law(q, p2, p3, ibonus):
    K, V = q.shape
    lvl3 = collections.defaultdict(float)
    for x in itertools.product(range(V), repeat=K):
        w = float(np.prod([q[i][x[i]] for i in range(K)]))
        if w > 0:
            _level(x, w, q, p2, ibonus, lvl3)
    commit = collections.defaultdict(float)
    for c, w in lvl3.items():
        _level(c, w, p2, p3, True, commit)
    return commit


def _rows(rng, R, V):
    return rng.dirichlet(np.full(V, 0.8), size=R)


@pytest.mark.parametrize("K,V,ibonus,seed", [(2, 4, True, 0), (2, 4, False, 1), (3, 3, True, 2),
                                             (3, 3, False, 3)])
def test_three_level_commit_law_matches_exact_dp(K, V, ibonus, seed):
    rng = np.random.default_rng(seed)
    q = _rows(rng, K, V)
    p2 = _rows(rng, K + 1, V)
    p3 = _rows(rng, K + 2, V)
    law = exact_commit_law(q, p2, p3, ibonus)
    assert sum(law.values()) == pytest.approx(1.0, abs=1e-12)
    # losslessness pins the DP: commit[0] ~ p3_0 exactly
    first = np.zeros(V)
    for c, w in law.items():
        first[c[0]] += w
    assert np.allclose(first, p3[0], atol=1e-12)

    # the oracle's sampled cascade on N independent requests with the same rows
    N = 200_000
    with np.errstate(divide="ignore"):
        lq, l2, l3 = np.log(q), np.log(p2), np.log(p3 if ibonus else p3[:K + 1])
    levels = [np.ascontiguousarray(np.broadcast_to(z, (N,) + z.shape)) for z in (lq, l2, l3)]
    cdf = np.cumsum(q, axis=1)
    draft = np.stack([np.minimum(np.searchsorted(cdf[i], rng.random(N), side="right"), V - 1)
                      for i in range(K)], axis=1).astype(np.int32)
    u_acc = rng.random((2, N, K + 2)).astype(np.float32)
    u_emit = rng.random((2, N, K + 2)).astype(np.float32)
    o = O.chain_verify(levels, draft, u_acc, u_emit, intermediate_bonus=ibonus)
    emp = collections.Counter(tuple(int(t) for t in o["out_tok"][b, :o["out_len"][b]]) for b in range(N))
    assert set(emp) <= {c for c, w in law.items() if w > 0}
    # every commit sequence: |freq - law| within 5 sigma; then one chi-square over them
    for c, w in law.items():
        assert abs(emp[c] / N - w) <= 5 * np.sqrt(w * (1 - w) / N) + 1e-9, (c, emp[c] / N, w)
    keys = [c for c, w in law.items() if w * N >= 5]
    f_obs = np.array([emp[c] for c in keys] + [N - sum(emp[c] for c in keys)], float)
    f_exp = np.array([law[c] * N for c in keys] + [N * (1 - sum(law[c] for c in keys))])
    keep = f_exp > 0
    assert scipy.stats.chisquare(f_obs[keep], f_exp[keep] * f_obs[keep].sum() / f_exp[keep].sum()).pvalue > 1e-3
    # and the commit-length law
    lens = collections.Counter(int(x) for x in o["out_len"])
    for n in range(1, K + 3):
        w = sum(v for c, v in law.items() if len(c) == n)
        assert abs(lens[n] / N - w) <= 5 * np.sqrt(max(w * (1 - w), 1e-12) / N) + 1e-9, (n, lens[n] / N, w)


def test_dp_detects_a_wrong_proposal_row():
    # mutation check of the pin: a DP whose level 3 compares against the drafter's rows (not
    # level 2's, reading R7) gives a different law, so the test above can fail
    rng = np.random.default_rng(9)
    K, V = 2, 4
    q, p2, p3 = _rows(rng, K, V), _rows(rng, K + 1, V), _rows(rng, K + 2, V)
    good = exact_commit_law(q, p2, p3, True)
    lvl3 = collections.defaultdict(float)
    for x in itertools.product(range(V), repeat=K):
        w = float(np.prod([q[i][x[i]] for i in range(K)]))
        _level(x, w, q, p2, True, lvl3)
    bad = collections.defaultdict(float)
    qq = np.vstack([q, p2[K:]])
    for c, w in lvl3.items():
        _level(c, w, qq, p3, True, bad)
    assert max(abs(good[c] - bad[c]) for c in set(good) | set(bad)) > 1e-2
