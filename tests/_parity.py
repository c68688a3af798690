"""Shared helpers for GPU-vs-oracle parity tests (test infrastructure)."""
import numpy as np
import torch

import oracle

DIV_REL, DIV_ABS = 1e-4, 1e-7     # DESIGN.md R18
KL_ABS = 1e-7                     # DESIGN.md R18
ACCEPT_BAND = 1e-6                # north star: |u - p/q| < 1e-6
DRAW_BAND = 1e-7                  # inverse-CDF draws: |u - C/Z| < 1e-7 (tighter than R18's 1e-6)


def to_np(o):
    return {k: (v.cpu().numpy() if torch.is_tensor(v) else v) for k, v in o.items()}


def run_oracle(inp, *, greedy=False, intermediate_bonus=True, draft_fed=None, requests=None,
               nthreads=0, tie_eps_draw=DRAW_BAND):
    """Oracle on (a subset of) the requests of a synth.ChainInputs."""
    sel = slice(None) if requests is None else requests
    levels = [t[sel].float().cpu().numpy() if t.dtype != torch.float32 else t[sel].cpu().numpy()
              for t in inp.levels]
    levels = [z[:, :, :inp.V] for z in levels]
    draft = inp.draft[sel].cpu().numpy()
    ua = inp.u_acc[:, sel].cpu().numpy()
    ue = inp.u_emit[:, sel].cpu().numpy()
    return oracle.chain_verify(levels, draft, ua, ue, greedy=greedy,
                               intermediate_bonus=intermediate_bonus, draft_fed=draft_fed,
                               tie_eps=ACCEPT_BAND, tie_eps_draw=tie_eps_draw, nthreads=nthreads)


def compare(gpu, ref, requests=None, check_rollback=True):
    """Return a report dict; mismatches outside near-tie requests are listed."""
    g = to_np(gpu)
    idx = np.arange(ref["out_len"].shape[0]) if requests is None else np.asarray(requests)
    rep = dict(mismatch=[], near_tie=int((ref["near_tie"] != 0).sum()), dtv_err=0.0, kl_err=0.0,
               dtv_maxabs=0.0)
    for j, b in enumerate(idx):
        if ref["near_tie"][j]:
            continue
        ok = int(g["commit_len"][b]) == int(ref["out_len"][j])
        ok &= np.array_equal(g["commit_tok"][b], ref["out_tok"][j])
        ok &= np.array_equal(g["n_acc"][:, b], ref["n_acc"][:, j])
        if "m_cand" in g:
            ok &= np.array_equal(g["m_cand"][:, b], ref["m_cand"][:, j])
        if check_rollback and "rollback" in g:
            ok &= np.array_equal(g["rollback"][:, b], ref["rollback"][:, j])
        if not ok:
            rep["mismatch"].append(int(b))
    if "pos_dtv" in g:
        d = g["pos_dtv"][:, idx].astype(np.float64)
        dr = ref["pos_dtv"]
        rep["dtv_err"] = float((np.abs(d - dr) - (DIV_REL * np.abs(dr) + DIV_ABS)).max())
        rep["dtv_maxabs"] = float(np.abs(d - dr).max())
        k = g["pos_kl"][:, idx].astype(np.float64)
        kr = ref["pos_kl"]
        fin = np.isfinite(kr)
        assert np.array_equal(np.isfinite(k), fin), "KL +inf pattern differs"
        if fin.any():
            rep["kl_err"] = float((np.abs(k[fin] - kr[fin]) - (DIV_REL * np.abs(kr[fin]) + KL_ABS)).max())
    return rep


def assert_parity(gpu, ref, requests=None, check_rollback=True, max_near_tie_frac=0.1, check_divergence=True):
    rep = compare(gpu, ref, requests, check_rollback)
    assert not rep["mismatch"], f"token/length mismatch outside near ties: requests {rep['mismatch'][:20]}"
    if check_divergence:
        assert rep["dtv_err"] <= 0, f"DTV outside tolerance by {rep['dtv_err']}"
        assert rep["kl_err"] <= 0, f"KL outside tolerance by {rep['kl_err']}"
    n = ref["out_len"].shape[0]
    assert rep["near_tie"] <= max(2, max_near_tie_frac * n), rep
    return rep
