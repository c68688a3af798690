"""The C ABI library builds, loads without a GPU, and exports every function declared
in include/msd.h; host-side (non-GPU) entry points behave per the header."""
import ctypes
import os
import re

import pytest

from paper_2505_07680_b200 import api

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "msd.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(msd_[a-z_0-9]+)\s*\(", src)))


def test_header_declares_the_four_boundary_calls():
    names = _declared()
    for n in ("msd_verify_level", "msd_chain_verify", "msd_kv_rollback", "msd_predict_chain_latency"):
        assert n in names


def test_library_exports_every_declared_symbol():
    lib = api.lib()
    missing = [n for n in _declared() if not hasattr(lib, n)]
    assert not missing, missing


def test_library_is_sm100a_only():
    so = api.LIB_PATH
    out = os.popen(f"/usr/local/cuda/bin/cuobjdump -lelf {so} 2>&1").read()
    assert "sm_100a" in out and "sm_90" not in out


def test_workspace_size_and_argument_errors_without_gpu():
    assert api.chain_workspace_bytes(3, 512, 8, 128256) > 0
    assert api.lib().msd_chain_verify_workspace(1, 4, 4, 100) == 0      # L < 2
    st = api.lib().msd_chain_verify(None, 3, 1, 1, 10, None, None, None, 0, 1, 0, None, None, None,
                                    None, None, None, None, None, None, None, 0, None)
    assert st == 1 and b"levels" in api.lib().msd_last_error()


def test_host_cost_model_spec_examples():
    assert api.predict_chain_latency([100.0], [], 4) == 100.0
    assert api.predict_chain_latency([10.0, 100.0], [1.0], 4) == pytest.approx(28.0)
    ch, te = api.select_chain([1.0, 5.0, 40.0], [[0.0] * 3] * 3, 4)
    assert ch == [2] and te == 40.0
    with pytest.raises(api.MsdError):
        api.predict_chain_latency([1.0, 2.0], [1.5], 4)                          # alpha > 1


def test_host_cost_model_matches_oracle_eq7_and_alg1():
    import numpy as np
    import oracle
    rng = np.random.default_rng(0)
    for _ in range(200):
        N = int(rng.integers(1, 5))
        T = list(rng.random(N) * 10 + 0.1)
        a = list(rng.random(N - 1))
        W = int(rng.integers(1, 9))
        for vc in (0, 1):
            for ib in (0, 1):
                assert api.predict_chain_latency(T, a, W, vc, ib) == pytest.approx(
                    oracle.predict_chain_latency(T, a, W, vc, ib), rel=1e-12)
    for _ in range(100):
        P = int(rng.integers(1, 6))
        T = np.sort(rng.random(P) * 10 + 0.1)
        sim = rng.random((P, P))
        W = int(rng.integers(1, 9))
        assert api.select_chain(T, sim, W, 4)[0] == oracle.select_chain(T, sim, W, 4)[0]


def test_simscore_update_ema():
    row = [int(0.25 * api.DTV_SCALE) * 10, 0, 10, 0, 0, 0, 0, 0]   # mean DTV 0.25
    assert api.simscore_update(0.0, row, 0.1, first=True) == pytest.approx(0.75)
    assert api.simscore_update(0.5, row, 0.5) == pytest.approx(0.625)           # P:182 EMA
