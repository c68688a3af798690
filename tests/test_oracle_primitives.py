"""Pins for the oracle's primitives (Eq. 1, Eq. 5, KL, acceptance, draws).

Each test pins the oracle to something other than itself: a library routine
(scipy), a closed form, a SPEC.md worked example, or a mathematical invariant.
"""
import math

import numpy as np
import pytest
import scipy.special
import scipy.stats

import oracle as O

RNG = np.random.default_rng(1234)


def _rand_p(V, rng=RNG, zeros=0):
    p = rng.dirichlet(np.ones(V))
    if zeros:
        idx = rng.choice(V, zeros, replace=False)
        p[idx] = 0.0
        p /= p.sum()
    return p


# ------------------------------------------------------------------ Eq. 1 normaliser
@pytest.mark.parametrize("V", [1, 2, 7, 1000, 32000])
def test_lse_matches_scipy_logsumexp(V):
    z = RNG.normal(0, 4, V)
    assert O.lse(z) == pytest.approx(scipy.special.logsumexp(z), rel=1e-14, abs=1e-13)


def test_lse_with_masked_entries_matches_scipy():
    z = RNG.normal(0, 4, 513)
    z[::3] = -np.inf
    assert O.lse(z) == pytest.approx(scipy.special.logsumexp(z), rel=1e-14)


@pytest.mark.parametrize("c,V", [(0.0, 5), (-3.25, 1000), (17.5, 128256)])
def test_lse_constant_logits_closed_form(c, V):
    # softmax of a constant row is uniform: LSE = c + log V exactly
    assert O.lse(np.full(V, c)) == pytest.approx(c + math.log(V), rel=0, abs=1e-12)


def test_lse_special_rows():
    assert O.lse(np.full(4, -np.inf)) == -np.inf
    assert math.isnan(O.lse(np.array([0.0, np.nan, 1.0])))
    assert math.isnan(O.lse(np.array([0.0, np.inf, 1.0])))


# ------------------------------------------------------------------ argmax
def test_argmax_spec_examples():
    assert O.argmax(np.log([0.1, 0.7, 0.2])) == 1
    assert O.argmax(np.log([0.5, 0.5])) == 0          # S:92 ties -> lowest id
    assert O.argmax(np.log([0, 0, 0, 1.0])) == 3      # S:93 one-hot
    z = np.array([1.0, 3.0, -2.0, 3.0, 3.0])
    assert O.argmax(z) == 1


# ------------------------------------------------------------------ Eq. 5 DTV
def test_dtv_spec_examples():
    assert O.dtv([0.5, 0.5], [0.5, 0.5]) == 0.0
    assert O.dtv([1.0, 0.0], [0.0, 1.0]) == pytest.approx(1.0)
    assert O.dtv([0.8, 0.2], [0.6, 0.4]) == pytest.approx(0.2, abs=1e-15)


@pytest.mark.parametrize("V", [2, 5, 64, 4096])
def test_overlap_plus_dtv_is_one(V):
    # Eq. 2 / S:105: sum_v min(p,q) + DTV(p,q) = 1
    p, q = _rand_p(V), _rand_p(V, zeros=V // 4)
    overlap = np.minimum(p, q).sum()
    assert overlap + O.dtv(p, q) == pytest.approx(1.0, abs=1e-12)


@pytest.mark.parametrize("eps", [0.1, 0.3, 0.6])
def test_dtv_mixture_family_closed_form(eps):
    # q = (1-eps) p + eps U  =>  DTV(p, q) = eps * DTV(p, U)   (S:709 family)
    V = 37
    p = _rand_p(V)
    U = np.full(V, 1.0 / V)
    q = (1 - eps) * p + eps * U
    assert O.dtv(p, q) == pytest.approx(eps * O.dtv(p, U), rel=1e-12)


def test_dtv_disjoint_support_is_one():
    p = np.array([0.3, 0.7, 0, 0, 0])
    q = np.array([0, 0, 0.2, 0.5, 0.3])
    assert O.dtv(p, q) == pytest.approx(1.0, abs=1e-15)


def test_dtv_is_shift_invariant_in_logits_and_symmetric():
    za, zb = RNG.normal(0, 3, 300), RNG.normal(0, 3, 300)
    d = O.dtv_logits(za, zb)
    assert O.dtv_logits(za + 11.0, zb - 4.0) == pytest.approx(d, rel=1e-12)
    assert O.dtv_logits(zb, za) == pytest.approx(d, rel=1e-12)


# ------------------------------------------------------------------ KL(p || q)
@pytest.mark.parametrize("V", [2, 9, 500])
def test_kl_matches_scipy_entropy(V):
    p, q = _rand_p(V, zeros=V // 3), _rand_p(V)
    assert O.kl(p, q) == pytest.approx(scipy.stats.entropy(p, q), rel=1e-12, abs=1e-14)


def test_kl_onehot_closed_form():
    q = _rand_p(11)
    for t in (0, 4, 10):
        p = np.zeros(11)
        p[t] = 1.0
        assert O.kl(p, q) == pytest.approx(-math.log(q[t]), rel=1e-13)


def test_kl_identical_is_exactly_zero_and_support_rules():
    p = _rand_p(20, zeros=5)
    assert O.kl(p, p) == 0.0
    q = p.copy()
    q[np.argmax(p)] = 0.0
    q /= q.sum()
    assert O.kl(p, q) == math.inf                    # p > 0 where q = 0
    assert math.isfinite(O.kl(q, p))                 # q = 0 terms are skipped


def test_pinsker_inequality():
    for _ in range(200):
        V = RNG.integers(2, 40)
        p, q = _rand_p(V), _rand_p(V)
        assert O.dtv(p, q) <= math.sqrt(O.kl(p, q) / 2) + 1e-12


# ------------------------------------------------------------------ acceptance
def test_accept_rule_cases():
    # p(t) >= q(t): every u in [0,1) accepts
    for u in (0.0, 0.5, 0.999999):
        assert O.accept(math.log(0.4), 0.0, math.log(0.3), 0.0, u)[0]
    # p(t)/q(t) = 0.25: accept iff u < 0.25 (strict; reading R2)
    za, zb = math.log(0.1), math.log(0.4)
    assert O.accept(za, 0.0, zb, 0.0, 0.2499)[0]
    assert not O.accept(za, 0.0, zb, 0.0, 0.2501)[0]
    # p(t) = 0: never;  q(t) = 0 < p(t): always
    assert not O.accept(-math.inf, 0.0, math.log(0.5), 0.0, 0.0)[0]
    assert O.accept(math.log(0.5), 0.0, -math.inf, 0.0, 0.999)[0]
    # near-tie flag when |u - p/q| < 1e-6
    assert O.accept(za, 0.0, zb, 0.0, 0.25 + 5e-7)[1]
    assert not O.accept(za, 0.0, zb, 0.0, 0.25 + 5e-6)[1]


# ------------------------------------------------------------------ draws
def test_sample_inverse_cdf_convention():
    z = np.log([0.2, 0.3, 0.5])
    assert O.sample(z, 0.1)[0] == 0
    assert O.sample(z, 0.2)[0] == 1      # strict crossing C_t > u
    assert O.sample(z, 0.49)[0] == 1
    assert O.sample(z, 0.5)[0] == 2
    assert O.sample(z, 0.999999)[0] == 2
    assert O.sample(np.log([0, 0, 0, 1.0, 0]), 0.7)[0] == 3     # S:82 one-hot


@pytest.mark.parametrize("V", [3, 8])
def test_sample_law_equals_p_on_uniform_grid(V):
    # The draw realises p: fraction of a midpoint u-grid mapped to t equals p_t.
    N = 20000
    p = _rand_p(V, zeros=1)
    z = np.log(p, where=p > 0, out=np.full(V, -np.inf))
    counts = np.zeros(V)
    for u in (np.arange(N) + 0.5) / N:
        counts[O.sample(z, u)[0]] += 1
    assert np.max(np.abs(counts / N - p)) <= 1.0 / N + 1e-12


def test_residual_spec_examples():
    # S:100 p=(.8,.2) q=(.6,.4) -> residual (1,0): every u draws 0
    for u in (0.0, 0.3, 0.99):
        t, _, small = O.sample_residual_logits(np.log([0.8, 0.2]), np.log([0.6, 0.4]), u)
        assert t == 0 and not small
    # S:101 p = q -> fallback to p
    p = np.array([0.25, 0.75])
    t, _, small = O.sample_residual_logits(np.log(p), np.log(p), 0.1)
    assert small and t == 0
    t, _, small = O.sample_residual_logits(np.log(p), np.log(p), 0.5)
    assert small and t == 1
    # S:102 p=(1,0) q=(0,1) -> (1,0)
    t, _, _ = O.sample_residual_logits(np.array([0.0, -np.inf]), np.array([-np.inf, 0.0]), 0.7)
    assert t == 0


def test_residual_never_draws_where_q_dominates():
    V = 50
    for _ in range(50):
        p, q = _rand_p(V), _rand_p(V)
        for u in RNG.random(20):
            t, _, _ = O.sample_residual_logits(np.log(p), np.log(q), u)
            assert p[t] > q[t]
