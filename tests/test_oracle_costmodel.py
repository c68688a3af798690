"""Pins for the oracle's scheduler cost model (Eq. 3, Eq. 4, Eq. 7, Alg. 1; S:58-75,
S:418-471)."""
import math

import numpy as np
import pytest

import oracle as O


def test_eq3_spec_examples():
    assert O.expected_accepted(0.0, 4) == 1.0
    assert O.expected_accepted(1.0, 4) == 5.0
    assert O.expected_accepted(0.8, 4) == pytest.approx(3.3616, abs=1e-12)


def test_eq4_spec_examples():
    assert O.theoretical_speedup(0.0, 1, 0.1) == pytest.approx(1 / 1.1, abs=1e-12)
    assert O.theoretical_speedup(0.8, 4, 0.1) == pytest.approx(3.3616 / 1.4, abs=1e-12)
    assert O.theoretical_speedup(1.0, 4, 1e-12) == pytest.approx(5.0, rel=1e-9)


def test_ema_spec_examples():
    assert O.ema(10.0, 20.0, 0.5) == 15.0
    assert O.ema(10.0, 20.0, 1.0) == 20.0
    assert O.ema(10.0, 20.0, 0.2, first=True) == 20.0


def test_predict_chain_latency_spec_examples():
    assert O.predict_chain_latency([100.0], [], 4) == 100.0            # S:460 [M_t]
    assert O.predict_chain_latency([10.0, 100.0], [1.0], 4) == pytest.approx(28.0)


@pytest.mark.parametrize("seed", range(20))
def test_two_level_constant_verify_equals_eq4(seed):
    # Eq. 7 model for [M_q, M_p] with one verify pass (Eq. 4 convention) must give
    # T_p / T_eff == Eq. 4's speedup for every alpha, gamma, c.
    rng = np.random.default_rng(seed)
    a, g, c = rng.random(), int(rng.integers(1, 12)), rng.random() * 0.5 + 0.01
    Tp = 40.0
    t_eff = O.predict_chain_latency([c * Tp, Tp], [a], g)
    assert Tp / t_eff == pytest.approx(O.theoretical_speedup(a, g, c), rel=1e-12)


def test_monotonicity_in_member_time():
    # raising a chain member's T_i never lowers that chain's T_eff
    base = O.predict_chain_latency([2.0, 5.0, 40.0], [0.7, 0.8], 6)
    assert O.predict_chain_latency([3.0, 5.0, 40.0], [0.7, 0.8], 6) > base
    assert O.predict_chain_latency([2.0, 6.0, 40.0], [0.7, 0.8], 6) > base


def test_select_chain_defaults_and_simple_wins():
    T = np.array([1.0, 5.0, 40.0])
    # all similarities 0 -> speculation never pays -> [M_t]
    ch, te = O.select_chain(T, np.zeros((3, 3)), 4)
    assert ch == [2] and te == 40.0
    # a perfect, cheap drafter: [A, T] costs (4*1 + 40)/5 = 8.8 < 40
    sim = np.zeros((3, 3))
    sim[0, 2] = 1.0
    ch, te = O.select_chain(T, sim, 4)
    assert ch == [0, 2] and te == pytest.approx(8.8)
    # perfect everywhere, no intermediate bonus: [A, T] (8.8) beats [A, B, T]
    # ((4 + 5 + 40) / 5 = 9.8): an extra verify pass for the same tokens
    ch, te = O.select_chain(T, np.ones((3, 3)), 4, intermediate_bonus=False)
    assert ch == [0, 2] and te == pytest.approx(8.8)
    # with the intermediate bonus B's extra token makes [A, B, T] worth it: 49 / 6
    ch, te = O.select_chain(T, np.ones((3, 3)), 4, intermediate_bonus=True)
    assert ch == [0, 1, 2] and te == pytest.approx(49.0 / 6.0)


def test_select_chain_tie_prefers_shorter_then_lexicographic():
    T = np.array([1.0, 1.0, 10.0])
    sim = np.zeros((3, 3))
    sim[0, 2] = sim[1, 2] = 0.5                      # [A,T] and [B,T] tie exactly
    ch, _ = O.select_chain(T, sim, 3)
    assert ch == [0, 2]


def test_select_chain_respects_max_len():
    T = np.array([0.1, 0.2, 0.3, 50.0])
    sim = np.full((4, 4), 0.95)
    ch, _ = O.select_chain(T, sim, 8, max_len=2)
    assert len(ch) <= 2 and ch[-1] == 3


# ------------------------------------------------------------------ Eq. 7 for N >= 3
import itertools

from tests._costmc import simulate_t_eff


@pytest.mark.parametrize("ibonus", [True, False])
@pytest.mark.parametrize("linear", [False, True])
def test_eq7_three_level_monte_carlo(ibonus, linear):
    # [M_1, M_2, M_t] predicted T_eff vs the simulated latency per committed
    # token over 10^4 cycles agree within 10% (the continuous composition pushes the
    # expectation through a nonlinear map, so it is not exact)
    T = [1.0, 5.0, 40.0]
    for a2, a3 in itertools.product((0.3, 0.6, 0.85, 0.97), repeat=2):
        for W in (2, 4, 8):
            pred = O.predict_chain_latency(T, [a2, a3], W, linear, ibonus)
            mc = simulate_t_eff(T, [a2, a3], W, linear, ibonus, cycles=10_000, seed=W)
            assert pred == pytest.approx(mc, rel=0.10), (a2, a3, W)


def _run_mean(a, fed):
    """E[min(G, fed)] for G = successes before the first failure of Bernoulli(a): sum over
    the law P(acc = i) = a^i (1 - a) (i < fed), P(acc = fed) = a^fed."""
    return sum(i * a ** i * (1 - a) for i in range(fed)) + fed * a ** fed


@pytest.mark.parametrize("ibonus", [True, False])
def test_eq7_exact_when_the_middle_level_is_deterministic(ibonus):
    # alpha_2 in {0, 1} makes the number fed to the target deterministic, so Eq. 7's
    # composition is exact: alpha_2 = 0 -> level 2 rejects the first draft and emits its
    # correction token (fed_3 = 1, with or without the bonus: P:64); alpha_2 = 1 -> all W
    # accepted, plus the bonus token only with the intermediate bonus
    T = [1.0, 5.0, 40.0]
    for W in (1, 3, 7):
        for a3 in (0.2, 0.5, 0.9):
            lat = W * T[0] + T[1] + T[2]
            t0 = O.predict_chain_latency(T, [0.0, a3], W, False, ibonus)
            assert t0 == pytest.approx(lat / (1 + _run_mean(a3, 1)), rel=1e-12)
            fed = W + 1 if ibonus else W
            t1 = O.predict_chain_latency(T, [1.0, a3], W, False, ibonus)
            assert t1 == pytest.approx(lat / (1 + _run_mean(a3, fed)), rel=1e-12)
            mc = simulate_t_eff(T, [0.0, a3], W, False, ibonus, cycles=100_000, seed=3)
            assert t0 == pytest.approx(mc, rel=0.02)


def test_eq7_four_level_monte_carlo():
    T = [1.0, 3.0, 10.0, 40.0]
    for a in ((0.4, 0.8, 0.95), (0.9, 0.6, 0.8), (0.95, 0.95, 0.95)):
        for ib in (True, False):
            pred = O.predict_chain_latency(T, list(a), 6, False, ib)
            assert pred == pytest.approx(simulate_t_eff(T, list(a), 6, False, ib, 20_000, 5), rel=0.10)
