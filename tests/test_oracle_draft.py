"""Pins of the oracle's draft-side sampling step (P:62, P:245,
S:337-345): or_draft_sample against what the definition and the mathematics fix."""
import numpy as np
import pytest

import oracle


def test_uniform_grid_reproduces_the_distribution_exactly():
    """Brute force: n midpoints of [0,1) through the inverse CDF give each token a count
    within 1 of n * p(v) (p = softmax, Eq. 1) -- a wrong CDF, a dropped term or an
    off-by-one boundary breaks it."""
    rng = np.random.default_rng(0)
    V, n = 37, 20000
    z = rng.standard_normal(V) * 2
    p = np.exp(z - np.logaddexp.reduce(z))
    u = (np.arange(n) + 0.5) / n
    out = oracle.draft_sample(np.tile(z, (n, 1)), u)
    cnt = np.bincount(out["token"], minlength=V)
    assert np.all(np.abs(cnt - n * p) <= 1.0 + 1e-9)
    assert np.allclose(out["lse"], np.logaddexp.reduce(z), rtol=0, atol=1e-13)
    assert np.allclose(out["q_tok"], p[out["token"]], rtol=1e-13)


def test_matches_cumsum_searchsorted_away_from_ties():
    """Special case reducing to a library routine: token = searchsorted(cumsum(p), u, 'right')."""
    rng = np.random.default_rng(1)
    B, V = 64, 1000
    z = rng.standard_normal((B, V)) * 4
    u = rng.random(B).astype(np.float32)
    out = oracle.draft_sample(z, u)
    for b in range(B):
        c = np.cumsum(np.exp(z[b] - np.logaddexp.reduce(z[b])))
        want = int(np.searchsorted(c, float(u[b]) * c[-1], side="right"))
        if not out["near_tie"][b]:
            assert out["token"][b] == want


def test_greedy_is_first_argmax_and_masked_tokens_are_never_drawn():
    z = np.array([[0.0, 3.0, 3.0, -1.0], [-np.inf, -np.inf, 1.0, -np.inf]])
    g = oracle.draft_sample(z, np.zeros(2, np.float32), greedy=True)
    assert list(g["token"]) == [1, 2]
    s = oracle.draft_sample(z[[1, 1, 1]], np.array([0.0, 0.5, 0.9999], np.float32))
    assert list(s["token"]) == [2, 2, 2] and np.allclose(s["q_tok"], 1.0)


def test_one_hot_row_and_extreme_uniforms():
    """u -> 0 draws the first token with positive mass; u -> 1 the last one."""
    z = np.full((2, 50), -np.inf)
    z[:, [7, 30]] = 0.0
    out = oracle.draft_sample(z, np.array([0.0, np.nextafter(np.float32(1), np.float32(0))], np.float32))
    assert list(out["token"]) == [7, 30]
    assert np.allclose(out["q_tok"], 0.5) and np.allclose(out["lse"], np.log(2.0))


def test_non_finite_row_gives_minus_one():
    z = np.array([[-np.inf] * 4, [0.0, np.nan, 0.0, 0.0]])
    with np.errstate(invalid="ignore"):
        out = oracle.draft_sample(z, np.array([0.3, 0.3], np.float32))
    assert list(out["token"]) == [-1, -1]
