"""GPU parity of the top-k / top-p logits processors (msd_logits_process, SURVEY 8(f) NEXT-4;
P:150 "LogitsProcessorList"; R19 / R23) against the float64 oracle: the per-row threshold
and the processed rows bit-exact (except rows whose top-p boundary is a floating-point tie, flagged
by either side), and the chain verification on processed rows equal to the oracle's on the same
processed (and temperature-scaled) logits."""
import numpy as np
import pytest
import torch

import oracle
from paper_2505_07680_b200 import api, synth
from tests._parity import ACCEPT_BAND, DRAW_BAND, assert_parity

pytestmark = [pytest.mark.gpu]
DEV = "cuda"


def _rows(B, R, V, dtype, seed, ties=False, ld=None):
    g = torch.Generator().manual_seed(seed)
    z = torch.randn((B, R, V), generator=g, dtype=torch.float64) * 2.5
    z[:, :, :: 97] += 6.0                        # a few dominant tokens (peaked rows)
    if ties:
        z = torch.round(z * 2) / 2                # coarse grid: large tie groups
    ld = ld or (V + 7) // 8 * 8                  # 16-byte aligned rows (ABI)
    full = torch.full((B, R, ld), -7.0, dtype=torch.float64)
    full[:, :, :V] = z
    return full.to(dtype).to(DEV)


def _check(x, V, k, p, T, rows=None):
    out, tau, flags = api.logits_process(x, rows=rows, V=V, top_k=k, top_p=p, temperature=T)
    torch.cuda.synchronize()
    R = x.shape[1] if rows is None else rows
    z = x[:, :R, :V].double().cpu().numpy()
    # the GPU flags a top-p boundary within 3e-7 Z of p Z (its masses' worst-case error); so does the oracle here
    zp_ref, tau_ref, near_ref = oracle.logits_process(z, temperature=T, top_k=k, top_p=p, eps=3e-7)
    g_tau = tau.cpu().numpy().astype(np.float64)
    g_out = out[:, :R, :V].double().cpu().numpy()
    fl = flags.cpu().numpy()
    n_checked = 0
    for b in range(x.shape[0]):
        if (fl[b] & api.FLAG["NEAR_TIE"]) or near_ref[b].any():
            continue
        n_checked += 1
        assert np.array_equal(g_tau[b], tau_ref[b]), (b, g_tau[b], tau_ref[b])
        assert np.array_equal(g_out[b], zp_ref[b]), b
    assert n_checked >= 1
    return out, tau, flags


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
@pytest.mark.parametrize("k,p,T", [(0, 0.9, 1.0), (50, 1.0, 1.0), (1, 1.0, 1.0), (40, 0.8, 0.7),
                                   (0, 0.5, 1.6), (0, 0.99, 1.0), (1000, 0.95, 1.0)])
def test_threshold_and_rows_match_oracle(dtype, k, p, T):
    _check(_rows(8, 3, 32003, dtype, seed=k + int(p * 100)), 32003, k, p, T)


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
def test_tie_groups_padded_rows_and_subset_of_rows(dtype):
    x = _rows(5, 4, 5000, dtype, seed=3, ties=True, ld=5008)
    _check(x, 5000, 7, 1.0, 1.0)
    _check(x, 5000, 0, 0.7, 1.0, rows=2)
    _check(x, 5000, 3, 0.6, 0.8)


def test_full_vocabulary_rows():
    x = _rows(2, 2, 151936, torch.bfloat16, seed=11)
    _check(x, 151936, 20, 0.9, 1.0)
    x = _rows(2, 2, 128256, torch.float32, seed=12)
    _check(x, 128256, 0, 0.95, 0.9)


def test_in_place_nonfinite_and_masked_rows():
    x = _rows(4, 2, 3000, torch.bfloat16, seed=5)
    x[1, 0, 17] = float("nan")
    x[2, 1, 5] = float("inf")
    x[3, 0, :2990] = float("-inf")               # 10 live entries
    ref, tau_r, fl_r = api.logits_process(x, V=3000, top_k=4, top_p=0.8)
    y = x.clone()
    out, tau, fl = api.logits_process(y, V=3000, top_k=4, top_p=0.8, out=y)
    torch.cuda.synchronize()
    assert out.data_ptr() == y.data_ptr()
    # bit patterns (NaN entries compare unequal as values)
    assert torch.equal(y.view(torch.int16), ref.view(torch.int16))
    assert torch.equal(tau.view(torch.int32), tau_r.view(torch.int32)) and torch.equal(fl, fl_r)
    assert torch.equal(y[1, 0].isnan(), x[1, 0].isnan())          # passed through unchanged
    assert torch.isnan(tau[1, 0]) and torch.isnan(tau[2, 1])
    assert (fl[1] & api.FLAG["NONFINITE"]) and (fl[2] & api.FLAG["NONFINITE"])
    assert 1 <= torch.isfinite(y[3, 0]).sum() <= 4                 # within the top-4 of the 10 live entries
    _check(x[3:], 3000, 4, 0.8, 1.0)


@pytest.mark.parametrize("k,p,T", [(20, 1.0, 1.0), (0, 0.9, 1.0), (50, 0.8, 0.7)])
def test_chain_verify_on_processed_levels_matches_oracle(k, p, T):
    c = synth.CONFIGS["llama3"]
    inp = synth.gauss_chain(8, 30000, c["K"], c["L"], c["sigmas"], s=c["s"], seed=c["seed"], device=DEV,
                            dtype=c["dtype"])
    levels = []
    for t in inp.levels:
        o, _, _ = api.logits_process(t, V=inp.V, top_k=k, top_p=p, temperature=T)
        levels.append(o)
    cv = api.ChainVerify(levels, inp.draft, inp.u_acc, inp.u_emit, V=inp.V, temperature=T)
    cv()
    torch.cuda.synchronize()
    ref_levels = [oracle.logits_process(t[:, :, :inp.V].double().cpu().numpy(), temperature=T, top_k=k,
                                        top_p=p)[0] / T for t in inp.levels]
    ref = oracle.chain_verify(ref_levels, inp.draft.cpu().numpy(), inp.u_acc.cpu().numpy(),
                              inp.u_emit.cpu().numpy(), tie_eps=ACCEPT_BAND, tie_eps_draw=DRAW_BAND)
    assert_parity(cv.outputs(), ref)
