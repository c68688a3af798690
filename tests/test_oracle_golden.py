"""The oracle reproduces every worked example in tests/golden/spec_examples.json."""
import json
import os

import numpy as np
import pytest

import oracle as O

G = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def _lg(p):
    p = np.asarray(p, float)
    out = np.full(p.shape, -np.inf)
    np.log(p, where=p > 0, out=out)
    return out


@pytest.mark.parametrize("ex", G["dtv"], ids=lambda e: e["cite"])
def test_dtv(ex):
    assert O.dtv(ex["p"], ex["q"]) == pytest.approx(ex["expect"], abs=1e-15)


@pytest.mark.parametrize("ex", G["overlap"], ids=lambda e: e["cite"])
def test_overlap(ex):
    assert 1.0 - O.dtv(ex["p"], ex["q"]) == pytest.approx(ex["expect"], abs=1e-15)


@pytest.mark.parametrize("ex", G["expected_accepted"], ids=lambda e: e["cite"])
def test_expected_accepted(ex):
    assert O.expected_accepted(ex["alpha"], ex["gamma"]) == pytest.approx(ex["expect"], abs=1e-12)


@pytest.mark.parametrize("ex", G["speedup"], ids=lambda e: e["cite"])
def test_speedup(ex):
    assert O.theoretical_speedup(ex["alpha"], ex["gamma"], ex["c"]) == pytest.approx(ex["expect"], abs=1e-12)


@pytest.mark.parametrize("ex", G["argmax"], ids=lambda e: e["cite"])
def test_argmax(ex):
    assert O.argmax(_lg(ex["p"])) == ex["expect"]


@pytest.mark.parametrize("ex", G["residual"], ids=lambda e: e["cite"])
def test_residual(ex):
    N = 1000
    law = np.zeros(len(ex["p"]))
    for u in (np.arange(N) + 0.5) / N:
        law[O.sample_residual_logits(_lg(ex["p"]), _lg(ex["q"]), u)[0]] += 1.0 / N
    assert np.allclose(law, ex["law"], atol=1e-12)


@pytest.mark.parametrize("ex", G["predict_effective_time"], ids=lambda e: e["cite"])
def test_predict(ex):
    assert O.predict_chain_latency(ex["T"], ex["alpha"], ex["W"]) == pytest.approx(ex["expect"], rel=1e-14)


@pytest.mark.parametrize("ex", G["ema"], ids=lambda e: e["cite"])
def test_ema(ex):
    assert O.ema(ex["old"], ex["measured"], ex["weight"]) == ex["expect"]


@pytest.mark.parametrize("ex", G["logical_rollback"], ids=lambda e: e["cite"])
def test_logical_rollback(ex):
    n = len(ex["lengths"])
    cap = max(ex["lengths"])
    m = np.zeros((n, cap), np.uint8)
    for b, k in enumerate(ex["lengths"]):
        m[b, :k] = 1
    m2, _, _ = O.rollback_mask(m, cap, ex["r"])
    assert list(m2.sum(1)) == ex["expect"]


@pytest.mark.parametrize("ex", G["fix_kv_cache"], ids=lambda e: e["cite"])
def test_fix(ex):
    n = len(ex["lengths"])
    m = np.zeros((n, ex["L"]), np.uint8)
    for b, k in enumerate(ex["lengths"]):
        m[b, :k] = 1
    _, L, _ = O.rollback_mask(m, ex["L"], [0] * n)
    assert L == ex["expect_L"]
