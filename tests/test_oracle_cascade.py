"""Pins for the oracle's multi-level cascade.

The cascade is pinned by what the paper and the mathematics fix: losslessness of
rejection sampling (the emitted token's law equals the target's), Eq. 2 (acceptance
rate = overlap), Eq. 3 (expected tokens per cycle), greedy == argmax matching,
p == q => full acceptance and zero divergence, and hand-worked rollback counts.
"""
import numpy as np
import pytest
import scipy.stats

import oracle as O

NEG = -np.inf


def _logits(p):
    p = np.asarray(p, dtype=np.float64)
    out = np.full(p.shape, NEG)
    np.log(p, where=p > 0, out=out)
    return out


def _bcast(rows, B):
    """rows [R, V] -> [B, R, V] contiguous."""
    return np.ascontiguousarray(np.broadcast_to(rows, (B,) + rows.shape))


def _dirichlet(rng, R, V, conc=1.0):
    return rng.dirichlet(np.full(V, conc), size=R)


# ------------------------------------------------------------------ special cases
def test_identical_levels_accept_everything_zero_divergence():
    rng = np.random.default_rng(0)
    B, K, V, L = 6, 5, 300, 3
    Z = rng.normal(0, 4, (B, K + L, V))
    levels = [Z[:, :K], Z[:, :K + 1], Z[:, :K + 2]]
    draft = rng.integers(0, V, (B, K)).astype(np.int32)
    u = rng.random((L - 1, B, K + L - 1)).astype(np.float32)
    o = O.chain_verify(levels, draft, u, u)
    assert (o["n_acc"] == [[K] * B, [K + 1] * B]).all()     # every candidate accepted
    assert (o["out_len"] == K + 2).all()
    assert (o["out_tok"][:, :K] == draft).all()
    assert (o["pos_dtv"] == 0.0).all() and (o["pos_kl"] == 0.0).all()
    assert (o["rollback"] == 0).all()


def test_onehot_target_makes_stochastic_equal_greedy():
    rng = np.random.default_rng(1)
    B, K, V = 64, 4, 40
    draft_rows = rng.normal(0, 2, (B, K, V))
    tgt = np.full((B, K + 1, V), NEG)
    hot = rng.integers(0, V, (B, K + 1))
    tgt[np.arange(B)[:, None], np.arange(K + 1)[None, :], hot] = 0.0
    draft = np.where(rng.random((B, K)) < 0.7, hot[:, :K], rng.integers(0, V, (B, K))).astype(np.int32)
    u = rng.random((1, B, K + 1)).astype(np.float32)
    s = O.chain_verify([draft_rows, tgt], draft, u, u)
    g = O.chain_verify([draft_rows, tgt], draft, greedy=True)
    for key in ("n_acc", "out_tok", "out_len", "rollback"):
        assert (s[key] == g[key]).all(), key
    # and both equal plain argmax matching against the one-hot target
    mism = draft != hot[:, :K]
    n_ref = np.where(mism.any(1), mism.argmax(1), K)
    assert (g["n_acc"][0] == n_ref).all()


@pytest.mark.parametrize("L", [2, 3])
def test_greedy_commits_target_argmax(L):
    # P:361 output quality: under greedy decoding every committed token is the
    # target's argmax at its position; level 2 accepts exactly the matching prefix.
    rng = np.random.default_rng(2 + L)
    B, K, V = 200, 6, 25
    Zt = rng.normal(0, 2, (B, K + L, V))
    levels = [Zt[:, :K] + rng.normal(0, 1.0, (B, K, V))]
    for l in range(1, L):
        sig = 0.0 if l == L - 1 else 0.5
        levels.append(Zt[:, :K + l] + sig * rng.normal(0, 1, (B, K + l, V)))
    am = [np.argmax(z, axis=2) for z in levels]
    draft = np.where(rng.random((B, K)) < 0.8, am[1][:, :K], rng.integers(0, V, (B, K))).astype(np.int32)
    o = O.chain_verify(levels, draft, greedy=True)
    tgt_am = np.argmax(Zt, axis=2)
    for b in range(B):
        n = o["out_len"][b]
        assert (o["out_tok"][b, :n] == tgt_am[b, :n]).all()
    mism = draft != am[1][:, :K]
    n_ref = np.where(mism.any(1), mism.argmax(1), K)
    assert (o["n_acc"][0] == n_ref).all()


# ------------------------------------------------------------------ Eq. 2 and Eq. 3
def test_eq2_acceptance_rate_equals_overlap():
    rng = np.random.default_rng(7)
    V, B = 6, 200000
    q, p = _dirichlet(rng, 1, V)[0], _dirichlet(rng, 1, V)[0]
    x = rng.choice(V, size=B, p=q).astype(np.int32)[:, None]
    levels = [_bcast(_logits(q)[None], B), _bcast(_logits(np.stack([p, p])), B)]
    u = rng.random((1, B, 2)).astype(np.float32)
    o = O.chain_verify(levels, x, u, u)
    alpha = np.minimum(p, q).sum()                    # Eq. 2 overlap
    rate = (o["n_acc"][0] == 1).mean()
    assert abs(rate - alpha) < 4 * np.sqrt(alpha * (1 - alpha) / B) + 1e-3


@pytest.mark.parametrize("K", [2, 4, 8])
def test_eq3_expected_tokens_per_cycle(K):
    # i.i.d. positions with the same (q, p): E[n + 1] = (1 - a^{K+1}) / (1 - a),
    # a = sum_v min(p, q)  (Eq. 3 read as counting the bonus token, reading R1).
    rng = np.random.default_rng(100 + K)
    V, B = 8, 100000
    q, p = _dirichlet(rng, 1, V, 0.7)[0], _dirichlet(rng, 1, V, 0.7)[0]
    x = rng.choice(V, size=(B, K), p=q).astype(np.int32)
    levels = [_bcast(np.tile(_logits(q), (K, 1)), B), _bcast(np.tile(_logits(p), (K + 1, 1)), B)]
    u = rng.random((1, B, K + 1)).astype(np.float32)
    o = O.chain_verify(levels, x, u, u)
    a = np.minimum(p, q).sum()
    expect = (1 - a ** (K + 1)) / (1 - a)
    got = o["out_len"].astype(np.float64)
    assert abs(got.mean() - expect) < 4 * got.std() / np.sqrt(B)
    assert expect == pytest.approx(O.expected_accepted(a, K), rel=1e-12)


# ------------------------------------------------------------------ losslessness
@pytest.mark.parametrize("V", [4, 8])
def test_two_level_emitted_law_equals_target_exact_grid(V):
    # Enumerate the draft token x (weight q(x)) x a midpoint grid over (u_acc, u_emit):
    # the law of the first committed token equals p (rejection sampling is lossless,
    # P:64 [leviathan2023fast]) up to the grid resolution 1/Na + 1/Ne.
    rng = np.random.default_rng(10 + V)
    Na, Ne = 256, 128
    q, p, pb = _dirichlet(rng, 3, V, 0.8)
    xs, ua, ue = np.meshgrid(np.arange(V), (np.arange(Na) + 0.5) / Na, (np.arange(Ne) + 0.5) / Ne,
                             indexing="ij")
    B = xs.size
    x = xs.reshape(B, 1).astype(np.int32)
    u_acc = np.zeros((1, B, 2), np.float32)
    u_emit = np.zeros((1, B, 2), np.float32)
    u_acc[0, :, 0] = ua.reshape(B)
    u_emit[0, :, 0] = ue.reshape(B)
    u_emit[0, :, 1] = ue.reshape(B)
    levels = [_bcast(_logits(q)[None], B), _bcast(_logits(np.stack([p, pb])), B)]
    o = O.chain_verify(levels, x, u_acc, u_emit)
    w = q[xs.reshape(B)] / (Na * Ne)
    law = np.bincount(o["out_tok"][:, 0], weights=w, minlength=V)
    assert np.abs(law - p).max() <= 1.0 / Na + 1.0 / Ne
    assert law.sum() == pytest.approx(1.0)


@pytest.mark.parametrize("ibonus", [True, False])
def test_three_level_first_commit_follows_target_chi_square(ibonus):
    rng = np.random.default_rng(33 + ibonus)
    V, K, B = 5, 2, 60000
    p1 = _dirichlet(rng, K, V, 0.8)
    p2 = _dirichlet(rng, K + 1, V, 0.8)
    p3 = _dirichlet(rng, K + 2, V, 0.8)
    x = np.stack([rng.choice(V, size=B, p=p1[i]) for i in range(K)], 1).astype(np.int32)
    levels = [_bcast(_logits(p1), B), _bcast(_logits(p2), B), _bcast(_logits(p3), B)]
    ua = rng.random((2, B, K + 2)).astype(np.float32)
    ue = rng.random((2, B, K + 2)).astype(np.float32)
    o = O.chain_verify(levels, x, ua, ue, intermediate_bonus=ibonus)
    obs = np.bincount(o["out_tok"][:, 0], minlength=V)
    res = scipy.stats.chisquare(obs, p3[0] * B)
    assert res.pvalue > 1e-3, (obs / B, p3[0])
    # a wrong proposal density at level 3 (e.g. the drafter's) breaks it
    assert o["out_len"].min() >= 1 and o["out_len"].max() <= K + 2


def test_three_level_mutated_proposal_is_detected():
    # mutation check of the pin above: feeding level 3 the drafter's rows as its
    # proposal density (instead of level 2's, reading R7) is not lossless.
    rng = np.random.default_rng(5)
    V, K, B = 5, 1, 60000
    p1 = _dirichlet(rng, K, V, 0.5)
    p2 = _dirichlet(rng, K + 1, V, 0.5)
    p3 = _dirichlet(rng, K + 2, V, 0.5)
    x = rng.choice(V, size=(B, 1), p=p1[0]).astype(np.int32)
    ua = rng.random((2, B, K + 2)).astype(np.float32)
    ue = rng.random((2, B, K + 2)).astype(np.float32)
    # correct chain
    good = O.chain_verify([_bcast(_logits(p1), B), _bcast(_logits(p2), B), _bcast(_logits(p3), B)],
                          x, ua, ue)
    obs = np.bincount(good["out_tok"][:, 0], minlength=V)
    assert scipy.stats.chisquare(obs, p3[0] * B).pvalue > 1e-3
    # 2-level chain (drafter -> target) with level-2 emissions ignored is also lossless,
    # but a chain whose middle level is skipped while its tokens are kept is not:
    mid = O.chain_verify([_bcast(_logits(p1), B), _bcast(_logits(p2), B)], x, ua[:1], ue[:1])
    bad_levels = [_bcast(_logits(np.vstack([p1, p1[:1]])), B), _bcast(_logits(p3), B)]
    bad = O.chain_verify(bad_levels, mid["out_tok"][:, :1].astype(np.int32), ua[1:], ue[1:])
    obs_bad = np.bincount(bad["out_tok"][:, 0], minlength=V)
    assert scipy.stats.chisquare(obs_bad, p3[0] * B).pvalue < 1e-6


# ------------------------------------------------------------------ rollback counts
def test_rollback_counts_hand_example():
    # K=3 two-level greedy chain, draft = [a0, wrong, a2]: level 2 rejects at 1 and
    # emits a1 = argmax, commit = [a0, a1].  Drafter fed K-1=2 tokens [a0, wrong]:
    # keeps 1, rolls back 1.  Target fed [a0, wrong, a2]: keeps 1, rolls back 2.
    V, K = 10, 3
    Zd = np.zeros((1, K, V))
    Zt = np.full((1, K + 1, V), -1.0)
    a = [3, 7, 1, 5]
    for i, t in enumerate(a):
        Zt[0, i, t] = 2.0
    x = np.array([[3, 2, 1]], np.int32)
    o = O.chain_verify([Zd, Zt], x, greedy=True, draft_fed=K - 1)
    assert o["n_acc"][0, 0] == 1 and o["out_len"][0] == 2
    assert list(o["out_tok"][0, :2]) == [3, 7]
    assert list(o["rollback"][:, 0]) == [1, 2]
    o = O.chain_verify([Zd, Zt], x, greedy=True, draft_fed=K)
    assert list(o["rollback"][:, 0]) == [2, 2]
    # full acceptance: nothing to roll back (bonus token never entered any cache)
    x = np.array([[3, 7, 1]], np.int32)
    o = O.chain_verify([Zd, Zt], x, greedy=True, draft_fed=K)
    assert list(o["out_tok"][0, :4]) == [3, 7, 1, 5] and list(o["rollback"][:, 0]) == [0, 0]


def test_token_out_of_range_is_rejected_and_flagged():
    rng = np.random.default_rng(3)
    B, K, V = 2, 3, 16
    Z = rng.normal(0, 1, (B, K + 1, V))
    x = np.array([[1, 99, 2], [-1, 0, 0]], np.int32)
    u = np.zeros((1, B, K + 1), np.float32)
    o = O.chain_verify([Z[:, :K], Z], x, u, u)
    assert o["n_acc"][0, 0] <= 1 and o["n_acc"][0, 1] == 0
    assert (o["flags"] & 2).all()
