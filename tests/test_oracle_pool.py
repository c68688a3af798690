"""Pins of the oracle's SimScore bootstrap:
or_pool_divergence / bootstrap_sim against what the spec and the mathematics fix."""
import numpy as np
import pytest
from scipy.stats import entropy

import oracle



def _rows(N, B, K, V, seed=0, scale=2.0):
    rng = np.random.default_rng(seed)
    return [rng.standard_normal((B, K, V)) * scale for _ in range(N)]


def test_identical_models_give_zero_divergence_and_simscore_one():
    """identical models -> all SimScores 1 (and every DTV / KL exactly 0)."""
    z = _rows(1, 3, 4, 97)[0]
    d, k = oracle.pool_divergence([z, z.copy(), z.copy()])
    assert d.shape == (3, 3, 4)
    assert np.all(d == 0.0) and np.all(k == 0.0)
    assert np.array_equal(oracle.bootstrap_sim([z, z, z]), np.ones((3, 3)))


def test_hand_computed_pair_gives_one_minus_dtv():
    """one position, hand-computable distributions -> SimScore = 1 - dtv.
    p0 = (0.5, 0.5), p1 = (0.9, 0.1): DTV = 0.4, KL(p1 || p0) = 0.9 ln 1.8 + 0.1 ln 0.2."""
    z0 = np.log(np.array([0.5, 0.5]))[None, None, :]
    z1 = np.log(np.array([0.9, 0.1]))[None, None, :]
    d, k = oracle.pool_divergence([z0, z1])
    assert d[0, 0, 0] == pytest.approx(0.4, abs=1e-15)
    assert k[0, 0, 0] == pytest.approx(0.9 * np.log(1.8) + 0.1 * np.log(0.2), abs=1e-15)
    sim = oracle.bootstrap_sim([z0, z1])
    assert sim[0, 1] == pytest.approx(0.6, abs=1e-15) and sim[1, 0] == sim[0, 1]


def test_mixture_closed_form_for_every_pair():
    """Pool of mixtures q_e = (1 - e) p + e U: q_a - q_b = (e_b - e_a)(p - U), so every pair's
    DTV is |e_b - e_a| DTV(p, U) exactly (S:709's mixture family)."""
    rng = np.random.default_rng(3)
    V = 64
    p = rng.dirichlet(np.ones(V))
    U = np.full(V, 1.0 / V)
    eps = [0.0, 0.1, 0.3, 0.6]
    zs = [np.log((1 - e) * p + e * U)[None, None, :] for e in eps]
    d, _ = oracle.pool_divergence(zs)
    dpu = 0.5 * np.abs(p - U).sum()
    pi = 0
    for i in range(4):
        for j in range(i + 1, 4):
            assert d[pi, 0, 0] == pytest.approx(abs(eps[j] - eps[i]) * dpu, rel=1e-12, abs=1e-15)
            pi += 1


def test_kl_direction_matches_scipy_and_pair_order_is_lexicographic():
    z = _rows(4, 2, 3, 40, seed=5)
    d, k = oracle.pool_divergence(z)
    pi = 0
    for i in range(4):
        for j in range(i + 1, 4):
            for b in range(2):
                for t in range(3):
                    pj = np.exp(z[j][b, t] - np.logaddexp.reduce(z[j][b, t]))
                    pq = np.exp(z[i][b, t] - np.logaddexp.reduce(z[i][b, t]))
                    assert k[pi, b, t] == pytest.approx(entropy(pj, pq), rel=1e-10, abs=1e-14)
                    assert d[pi, b, t] == pytest.approx(0.5 * np.abs(pj - pq).sum(), rel=1e-10, abs=1e-15)
            pi += 1


def test_adjacent_pairs_equal_the_cascade_divergences():
    """The bootstrap of a pool equals the per-position divergences the verification cascade
    (or_chain_verify, pinned independently) reports for adjacent levels of the same rows."""
    B, K, V, N = 3, 4, 80, 3
    z = _rows(N, B, K + N, V, seed=9)
    levels = [z[0][:, :K]] + [z[l][:, :K + l] for l in range(1, N)]
    rng = np.random.default_rng(1)
    draft = rng.integers(0, V, (B, K)).astype(np.int32)
    W = K + N - 1
    ref = oracle.chain_verify(levels, draft, rng.random((N - 1, B, W)).astype(np.float32),
                              rng.random((N - 1, B, W)).astype(np.float32))
    d, k = oracle.pool_divergence([zz[:, :K] for zz in z])
    # adjacent pairs (0,1) and (1,2) are pair indices 0 and 2 in lexicographic order
    for l, pi in ((1, 0), (2, 2)):
        assert np.allclose(d[pi], ref["pos_dtv"][l - 1], rtol=1e-12, atol=1e-15)
        assert np.allclose(k[pi], ref["pos_kl"][l - 1], rtol=1e-12, atol=1e-15)


def test_masked_support_gives_infinite_kl_and_unit_dtv():
    """Disjoint supports: DTV = 1; KL(p_j || p_i) = +inf where p_j > 0 = p_i."""
    z0 = np.log(np.array([1.0, 0.0, 0.0, 0.0]) + 0.0)[None, None, :]
    z1 = np.log(np.array([0.0, 0.5, 0.5, 0.0]))[None, None, :]
    with np.errstate(divide="ignore"):
        d, k = oracle.pool_divergence([z0, z1])
    assert d[0, 0, 0] == pytest.approx(1.0, abs=1e-15)
    assert np.isinf(k[0, 0, 0])
