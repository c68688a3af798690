"""Pins of the oracle's top-k / top-p logits processors (P:150
"LogitsProcessorList"; R19 / R23) against things other than itself: a brute-force search
over candidate thresholds, Hugging Face's own warpers, and closed forms."""
import numpy as np
import pytest

import oracle


def brute_tau(z, T=1.0, k=0, p=1.0):
    """Largest threshold c among the row's values such that {z >= c} satisfies the rule: for top-k,
    at least k entries; for top-p, mass >= p of the (top-k-kept) distribution.  Scans every
    candidate value; no sorting walk, no groups."""
    z = np.asarray(z, dtype=np.float64)
    vals = np.unique(z)
    tk = -np.inf
    if 0 < k < z.size:
        tk = max(c for c in vals if np.count_nonzero(z >= c) >= k)
    tp = -np.inf
    if 0 < p < 1 and np.isfinite(z.max()):
        kept = z >= tk
        w = np.where(kept, np.exp((z - z.max()) / T), 0.0)
        Z = w.sum()
        tp = max(c for c in vals if w[z >= c].sum() >= p * Z)
    return max(tk, tp)


@pytest.mark.parametrize("seed", range(40))
def test_threshold_matches_brute_force(seed):
    rng = np.random.default_rng(seed)
    V = int(rng.integers(2, 40))
    # a coarse grid makes ties frequent (whole tie groups must be kept)
    z = np.round(rng.normal(0, 2, V) * 2) / 2 if seed % 2 else rng.normal(0, 2, V)
    if seed % 5 == 0:
        z[rng.integers(0, V)] = -np.inf
    T = [1.0, 0.7, 1.8][seed % 3]
    k = int(rng.integers(0, V + 2))
    p = float(rng.choice([0.0, 0.3, 0.5, 0.9, 0.97, 1.0]))
    tau, near = oracle.logits_threshold(z, T, k, p)
    if near:
        return
    assert tau == brute_tau(z, T, k, p)


def _hf(z, T, k, p):
    torch = pytest.importorskip("torch")
    lp = pytest.importorskip("transformers.generation.logits_process")
    x = torch.tensor(z[None, :], dtype=torch.float64) / T
    if k:
        x = lp.TopKLogitsWarper(top_k=k)(None, x)
    if p < 1:
        x = lp.TopPLogitsWarper(top_p=p)(None, x)
    return np.isfinite(x[0].numpy())


@pytest.mark.parametrize("seed", range(12))
def test_kept_set_matches_hugging_face_warpers(seed):
    # continuous values (no ties): Hugging Face's sort-based warpers and the oracle's group walk
    # must keep exactly the same entries
    rng = np.random.default_rng(100 + seed)
    V = 64
    z = rng.normal(0, 3, V)
    T = [1.0, 0.5, 2.0][seed % 3]
    k = [0, 5, 20, 63][seed % 4]
    p = [0.9, 0.5, 1.0, 0.75][(seed // 4) % 4]
    tau, near = oracle.logits_threshold(z, T, k, p)
    assert not near
    ours = z >= tau
    assert np.array_equal(ours, _hf(z, T, k, p))


def test_closed_forms():
    z = np.array([0.5, 2.0, -1.0, 2.0, 1.0])
    assert oracle.logits_threshold(z, top_k=1)[0] == 2.0          # ties at the maximum kept
    assert oracle.logits_threshold(z, top_k=5)[0] == -np.inf       # k >= V: off
    assert oracle.logits_threshold(z, top_k=0)[0] == -np.inf       # 0: off
    assert oracle.logits_threshold(z, top_p=1e-9)[0] == 2.0        # tiny p: the top group
    assert oracle.logits_threshold(z, top_p=1.0)[0] == -np.inf     # off
    u = np.full(7, 0.25)                                          # one tie group: all kept
    assert oracle.logits_threshold(u, top_p=0.1)[0] == 0.25
    # two-point distribution: p(a) = 0.8 -> p < 0.8 keeps a only, p > 0.8 keeps both
    z2 = np.log([0.8, 0.2])
    assert oracle.logits_threshold(z2, top_p=0.79)[0] == z2[0]
    assert oracle.logits_threshold(z2, top_p=0.81)[0] == z2[1]
    # the boundary within eps of p is a tie
    assert oracle.logits_threshold(z2, top_p=0.8 + 1e-9)[1] == 1
    # top-k then top-p: p applies to the renormalised top-k distribution
    z3 = np.log([0.4, 0.3, 0.2, 0.1])
    tau, _ = oracle.logits_threshold(z3, top_k=2, top_p=0.5)      # 0.4/0.7 = 0.571 >= 0.5
    assert tau == z3[0]
    tau, _ = oracle.logits_threshold(z3, top_k=2, top_p=0.6)      # needs both of the two
    assert tau == z3[1]
    # temperature sharpens: at T = 0.25, p(0.4-token) = 0.4^4 / sum = 0.653 >= 0.6
    assert oracle.logits_threshold(z3, temperature=0.25, top_p=0.6)[0] == z3[0]
    assert oracle.logits_threshold(z3, temperature=1.0, top_p=0.6)[0] == z3[1]


def test_nonfinite_rows_and_masked_entries():
    assert np.isnan(oracle.logits_threshold(np.array([0.0, np.nan, 1.0]), top_k=1)[0])
    assert np.isnan(oracle.logits_threshold(np.array([0.0, np.inf]), top_p=0.5)[0])
    z = np.array([-np.inf, 0.0, -np.inf, 1.0])
    assert oracle.logits_threshold(z, top_k=3)[0] == -np.inf      # the 3rd largest is -inf
    assert oracle.logits_threshold(z, top_p=0.99)[0] == 0.0       # -inf entries carry no mass
    zp, tau, near = oracle.logits_process(np.array([[3.0, 1.0, 2.0], [0.0, 0.0, 5.0]]), top_k=2)
    assert np.array_equal(zp, np.array([[3.0, -np.inf, 2.0], [0.0, 0.0, 5.0]]))
