"""GPU parity: libmsd (through the C ABI) vs the float64 oracle on identical seeded inputs.

Tokens, accepted lengths, candidate counts, commit lengths and rollback lengths must be
bit-exact except for requests whose oracle path had a near tie (|u - threshold| < 1e-6);
divergences within 1e-4 relative + 1e-7 absolute (R18).
"""
import os

import numpy as np
import pytest
import torch

from paper_2505_07680_b200 import api, synth
from tests._parity import assert_parity, run_oracle, to_np

pytestmark = [pytest.mark.gpu]
DEV = "cuda"


def _gauss(name, **kw):
    c = dict(synth.CONFIGS[name])
    c.update(kw)
    return synth.gauss_chain(c["B"], c["V"], c["K"], c["L"], c["sigmas"], s=c["s"], seed=c["seed"],
                             device=DEV, dtype=c["dtype"], ld=c.get("ld"),
                             intermediate_bonus=c.get("ibonus", True))


def _run(inp, **kw):
    o = api.chain_verify(inp.levels, inp.draft, inp.u_acc, inp.u_emit, V=inp.V, **kw)
    torch.cuda.synchronize()
    return o


@pytest.mark.parametrize("name,kw", [
    ("tiny", {}),
    ("llama2", {}),
    ("qwen25", dict(B=8)),
    ("llama3", dict(B=16)),
    ("sweep", dict(B=8)),
])
def test_configs_match_oracle(name, kw):
    inp = _gauss(name, **kw)
    o = _run(inp)
    ref = run_oracle(inp)
    rep = assert_parity(o, ref)
    f = to_np(o)["flags"]
    assert not (f & (api.FLAG["TIMEOUT"] | api.FLAG["NONFINITE"])).any()
    print(name, rep)


@pytest.fixture
def knobs():
    """msd_debug_set_knobs overrides, restored to the release defaults afterwards."""
    yield api.debug_knobs
    api.debug_knobs()


@pytest.mark.parametrize("pat_t,pat_r,stages", [(2, 0, -1), (1, 3, -1), (2, 2, -1), (2, 1, 3)])
def test_item_patterns_agree(knobs, pat_t, pat_r, stages):
    """T items (exponentials parked in TMEM) and R items (ring stage kept, pass 2 recomputes)
    must give the same accept / emit decisions and divergences as the oracle, in any mix and
    ring depth."""
    inp = _gauss("llama3", B=24, V=30000)
    knobs(pat_t=pat_t, pat_r=pat_r, stages=stages)
    o = _run(inp)
    assert_parity(o, run_oracle(inp))


@pytest.mark.parametrize("name,kw", [("tiny", {}), ("llama3", dict(B=12, V=40000)),
                                      ("sweep", dict(B=6, V=9000))])
def test_greedy_matches_oracle(name, kw):
    inp = _gauss(name, **kw)
    o = _run(inp, greedy=True)
    ref = run_oracle(inp, greedy=True)
    rep = assert_parity(o, ref)
    assert rep["near_tie"] == 0


def test_no_intermediate_bonus_and_draft_fed_k():
    inp = _gauss("llama3", B=12, V=30000, ibonus=False)
    o = _run(inp, intermediate_bonus=False, draft_fed=inp.K)
    ref = run_oracle(inp, intermediate_bonus=False, draft_fed=inp.K)
    assert_parity(o, ref)


@pytest.mark.parametrize("V,ld", [(32001, 32008), (4097, 4104), (5, 8), (1000, 1000), (8191, 8200)])
def test_ragged_vocab_and_padded_stride(V, ld):
    inp = synth.gauss_chain(6, V, 3, 3, (0.9, 0.4, 0.0), seed=11, device=DEV, dtype="bf16", ld=ld)
    o = _run(inp)
    ref = run_oracle(inp)
    assert_parity(o, ref)


def test_identical_levels_accept_all_zero_divergence():
    inp = _gauss("llama3", B=8, V=20000)
    for l in range(1, inp.L):
        inp.levels[l][:, :inp.K] = inp.levels[0][:, :inp.K]
        inp.levels[l][:, inp.K:] = inp.levels[-1][:, inp.K:inp.levels[l].shape[1]]
    # every level now equals the drafter at draft positions: all candidates accepted
    o = to_np(_run(inp))
    assert (o["n_acc"][0] == inp.K).all()
    assert (o["pos_dtv"] == 0).all() and (o["pos_kl"] == 0).all()
    ref = run_oracle(inp)
    assert_parity(_run(inp), ref)


def test_onehot_target_stochastic_equals_greedy():
    B, K, V = 16, 5, 3000
    inp = synth.gauss_chain(B, V, K, 2, (0.8, 0.0), seed=5, device=DEV, dtype="bf16")
    tgt = inp.levels[1]
    hot = torch.randint(0, V, (B, K + 1), device=DEV)
    tgt.fill_(float("-inf"))
    tgt.scatter_(2, hot.unsqueeze(2), 0.0)
    keep = torch.rand((B, K), device=DEV) < 0.7
    inp.draft[:] = torch.where(keep, hot[:, :K].int(), inp.draft)
    s = to_np(_run(inp))
    g = to_np(_run(inp, greedy=True))
    for k in ("n_acc", "commit_tok", "commit_len", "rollback"):
        assert np.array_equal(s[k], g[k]), k
    assert_parity(_run(inp), run_oracle(inp))


def test_masked_entries_and_out_of_range_tokens():
    inp = _gauss("llama3", B=8, V=12000)
    g = torch.Generator(device=DEV).manual_seed(3)
    for t in inp.levels:
        mask = torch.rand(t.shape, generator=g, device=DEV) < 0.3
        t.masked_fill_(mask, float("-inf"))
    inp.draft[0, 2] = inp.V + 5
    inp.draft[1, 0] = -1
    o = _run(inp)
    f = to_np(o)["flags"]
    assert f[0] & api.FLAG["TOKEN_OOB"] and f[1] & api.FLAG["TOKEN_OOB"]
    ref = run_oracle(inp)
    assert_parity(o, ref)


def test_full_llama3_batch_sampled_requests():
    # the bench configuration (B=512, V=128256, K=8, L=3): every request is verified on
    # the GPU in one call; 8 requests spread over the batch are checked against the oracle.
    inp = _gauss("llama3")
    o = _run(inp)
    req = [0, 73, 130, 255, 256, 390, 451, 511]
    ref = run_oracle(inp, requests=req)
    assert_parity(o, ref, requests=req)
    f = to_np(o)["flags"]
    assert not (f & api.FLAG["TIMEOUT"]).any()


@pytest.mark.parametrize("name", ["qwen25", "llama2", "sweep"])
def test_full_batch_sampled_requests_other_configs(name):
    # the other BASELINE configurations at their full sizes in one call (Qwen B=256 V=151936 K=6;
    # Llama-2 B=64 V=32000 K=5; the 4-level sweep pool V=128256): sampled requests vs the oracle
    inp = _gauss(name)
    o = _run(inp)
    B = inp.B
    req = sorted({0, B // 7, B // 3, B // 2, (2 * B) // 3, B - 1})
    ref = run_oracle(inp, requests=req)
    assert_parity(o, ref, requests=req)
    assert not (to_np(o)["flags"] & api.FLAG["TIMEOUT"]).any()


def test_deterministic_bit_identical():
    inp = _gauss("qwen25", B=12, V=70000)
    a = {k: v.clone() for k, v in _run(inp).items()}
    b = _run(inp)
    for k in a:
        assert torch.equal(a[k], b[k]), k


def test_shard_invariance():
    # G-invariance: two shards of global requests reproduce the unsharded run exactly
    full = _gauss("llama3", B=16, V=20000)
    o = _run(full)
    parts = []
    for r0, n in ((0, 9), (9, 7)):
        c = synth.CONFIGS["llama3"]
        inp = synth.gauss_chain(n, 20000, c["K"], c["L"], c["sigmas"], seed=c["seed"], req0=r0,
                                device=DEV, dtype="bf16")
        parts.append(_run(inp))
    for k in ("commit_tok", "commit_len", "pos_dtv", "pos_kl", "flags"):
        cat = torch.cat([p[k] for p in parts], dim=0 if k in ("commit_tok", "commit_len", "flags") else 1)
        assert torch.equal(cat, o[k]), k
    for k in ("n_acc", "m_cand", "rollback"):
        assert torch.equal(torch.cat([p[k] for p in parts], dim=1), o[k]), k
    assert torch.equal(parts[0]["stats"] + parts[1]["stats"], o["stats"])


def test_stats_are_consistent_with_outputs():
    inp = _gauss("llama3", B=20, V=25000)
    o = to_np(_run(inp))
    st = o["stats"]
    F = api.STATS_FIELDS
    for l in range(inp.L - 1):
        assert st[l, F.index("positions")] == inp.B * inp.K
        assert st[l, F.index("accepted")] == o["n_acc"][l].sum()
        assert st[l, F.index("proposed")] == o["m_cand"][l].sum()
        dsum = o["pos_dtv"][l].astype(np.float64).sum()
        assert abs(st[l, F.index("dtv_fx")] / api.DTV_SCALE - dsum) < 1e-5 * max(1.0, dsum)


def test_verify_level_composes_to_chain_verify():
    # msd_chain_verify == sequential msd_verify_level calls, level l's q = level l-1's rows
    inp = _gauss("llama3", B=10, V=30000)
    o = to_np(_run(inp))
    K, B = inp.K, inp.B
    cand = inp.draft.clone()
    m = torch.full((B,), K, dtype=torch.int32, device=DEV)
    last = None
    for l in range(1, inp.L):
        Kl = cand.shape[1]
        ua = inp.u_acc[l - 1][:, :Kl].contiguous()
        ue = inp.u_emit[l - 1][:, :Kl + 1].contiguous()
        q = inp.levels[l - 1][:, :Kl]
        p = inp.levels[l][:, :Kl + 1]
        v = api.verify_level(q, p, cand, ua, ue, m=m, V=inp.V)
        torch.cuda.synchronize()
        vo = to_np(v)
        assert np.array_equal(vo["n_acc"], o["n_acc"][l - 1]), l
        assert np.allclose(vo["pos_dtv"][:, :K], o["pos_dtv"][l - 1], rtol=1e-5, atol=1e-7)
        last = vo
        cand = v["out_tok"].clamp(min=0).contiguous()     # slots >= m are never read
        m = v["out_len"].clone()
    assert np.array_equal(last["out_tok"], o["commit_tok"])
    assert np.array_equal(last["out_len"], o["commit_len"])


def test_exact_draw_mode_agrees_with_fast_path(knobs):
    inp = _gauss("qwen25", B=10, V=60000)
    fast = {k: v.clone() for k, v in _run(inp).items()}
    knobs(exact_draws=True)
    exact = _run(inp)
    ref = run_oracle(inp)
    assert_parity(exact, ref)
    assert_parity(fast, ref)


def test_empty_batch_and_argument_errors():
    inp = _gauss("tiny")
    with pytest.raises(api.MsdError):
        api.chain_verify(inp.levels[:1] * 1 + inp.levels[1:], inp.draft, None, None)  # no uniforms
    bad = [inp.levels[0], inp.levels[1][:, :inp.K]]          # too few target rows
    with pytest.raises(api.MsdError):
        api.chain_verify(bad, inp.draft, inp.u_acc, inp.u_emit)
    e = api.chain_verify([t[:0] for t in inp.levels], inp.draft[:0], inp.u_acc[:, :0], inp.u_emit[:, :0])
    assert e["commit_len"].numel() == 0


# ------------------------------------------------------------------ rollback
def test_kv_rollback_matches_oracle():
    import oracle
    B, nm = 300, 3
    kv = synth.paged_kv(B, nm, seed=9, block_size=16, min_len=1, max_len=700, device=DEV)
    g = torch.Generator().manual_seed(4)
    r = torch.stack([torch.minimum(torch.randint(0, 40, (B,), generator=g), kv[i]["seq_len"].cpu())
                     for i in range(nm)]).to(torch.int32)
    r[1, 7] = 10_000                                     # overflow -> flagged, untouched
    mb = kv[0]["block_table"].shape[1]
    kv[0]["seq_len"][11] = mb * 16 + 5                   # beyond its block-table row (R22)
    r[0, 11] = 3
    masks = []
    for i in range(nm):
        cm = torch.zeros((B, 760), dtype=torch.uint8)
        for b in range(B):
            cm[b, :int(kv[i]["seq_len"][b])] = 1
        kv[i]["cache_mask"] = cm.to(DEV)
        masks.append(cm.numpy())
    before = [{k: (v.cpu().numpy().copy() if torch.is_tensor(v) else v) for k, v in d.items()} for d in kv]
    flags = torch.zeros(B, dtype=torch.int32, device=DEV)
    api.kv_rollback(kv, r.to(DEV), flags)
    torch.cuda.synchronize()
    fl = flags.cpu().numpy()
    for i in range(nm):
        o = oracle.rollback_paged(before[i]["seq_len"], before[i]["block_table"], 16,
                                  before[i]["free_ids"], int(before[i]["free_count"][0]), r[i].numpy(),
                                  cache_mask=masks[i])
        assert np.array_equal(kv[i]["seq_len"].cpu().numpy(), o["seq_len"])
        assert np.array_equal(kv[i]["block_table"].cpu().numpy(), o["block_table"])
        assert int(kv[i]["free_count"][0]) == o["free_count"]
        assert np.array_equal(kv[i]["free_ids"].cpu().numpy(), o["free_ids"])
        assert np.array_equal(kv[i]["cache_mask"].cpu().numpy(), o["cache_mask"])
    assert fl[7] & api.FLAG["ROLLBACK_OVF"] and fl[11] & api.FLAG["ROLLBACK_OVF"]


def test_kv_rollback_freelist_overflow():
    B = 4
    kv = synth.paged_kv(B, 1, seed=1, min_len=100, max_len=200, device=DEV)
    kv[0]["free_count"][0] = kv[0]["free_ids"].numel()       # stack already full
    r = torch.full((1, B), 50, dtype=torch.int32, device=DEV)
    flags = torch.zeros(B, dtype=torch.int32, device=DEV)
    sl = kv[0]["seq_len"].clone()
    api.kv_rollback(kv, r, flags)
    torch.cuda.synchronize()
    assert (flags.cpu().numpy() & api.FLAG["FREELIST_OVF"]).any()
    assert torch.equal(kv[0]["seq_len"], sl - 50)
