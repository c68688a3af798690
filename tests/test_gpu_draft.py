"""GPU parity of the draft-side sampling step:
msd_draft_sample through the C ABI vs oracle.draft_sample (float64) on the same seeded rows.
Tokens bit-exact outside the oracle's near ties (|u - C/Z| < 1e-7); lse / q_tok within
fp32 rounding of the float64 values."""
import numpy as np
import pytest
import torch

import oracle
from paper_2505_07680_b200 import api, synth
from tests._parity import DRAW_BAND

pytestmark = [pytest.mark.gpu]
DEV = "cuda"


def _rows(B, V, K=4, dtype="bf16", ld=None, seed=21):
    inp = synth.gauss_chain(B, V, K, 2, (0.75, 0.0), seed=seed, device=DEV, dtype=dtype, ld=ld)
    return inp.levels[0]                                   # drafter logits [B][K][ld]


def _uniforms(B, seed):
    g = torch.Generator(device="cpu").manual_seed(seed)
    return torch.rand((B,), generator=g).to(DEV)


def _check(out, ref, greedy=False):
    tok = out["token"].cpu().numpy()
    ok = ref["near_tie"] == 0
    assert np.array_equal(tok[ok], ref["token"][ok]), np.nonzero(tok[ok] != ref["token"][ok])
    assert ok.mean() > 0.9
    lse = out["lse"].double().cpu().numpy()
    assert np.allclose(lse, ref["lse"], rtol=1e-6, atol=1e-5)
    q = out["q_tok"].double().cpu().numpy()
    assert np.allclose(q[ok], ref["q_tok"][ok], rtol=2e-5, atol=1e-30)


@pytest.mark.parametrize("B,V,dtype,ld", [
    (64, 128256, "bf16", None),
    (32, 151936, "bf16", None),
    (48, 32001, "bf16", 32008),
    (16, 1000, "f32", None),
    (16, 4097, "f32", 4104),
    (8, 5, "bf16", 8),
])
@pytest.mark.parametrize("greedy", [False, True])
def test_draft_sample_matches_oracle(B, V, dtype, ld, greedy):
    z = _rows(B, V, dtype=dtype, ld=ld)
    for k in range(z.shape[1]):                            # W sequential draft steps
        u = _uniforms(B, 100 + k)
        out = api.draft_sample(z, u, row=k, V=V, greedy=greedy)
        torch.cuda.synchronize()
        ref = oracle.draft_sample(z[:, k, :V].double().cpu().numpy(), u.cpu().numpy(),
                                  greedy=greedy, tie_eps_draw=DRAW_BAND)
        _check(out, ref, greedy)
        f = out["flags"].cpu().numpy()
        assert not (f & api.FLAG["NONFINITE"]).any()


def test_uniform_grid_reproduces_softmax():
    """Brute force on the GPU: n grid uniforms through one row give every token a count
    within 1 of n p(v) (p from the float64 oracle)."""
    V, n = 300, 30000
    z = _rows(1, V, dtype="f32")[0, 0]
    rows = z.expand(n, V).unsqueeze(1).contiguous()
    u = synth.uniform_grid(n, device=DEV).float()
    out = api.draft_sample(rows, u)
    cnt = np.bincount(out["token"].cpu().numpy(), minlength=V)
    zz = z.double().cpu().numpy()
    p = np.exp(zz - np.logaddexp.reduce(zz))
    assert np.all(np.abs(cnt - n * p) <= 1.0 + 1e-6)


def test_masked_tokens_never_drawn_and_nonfinite_rows():
    B, V = 64, 20000
    z = _rows(B, V, dtype="bf16").clone()
    g = torch.Generator(device=DEV).manual_seed(5)
    mask = torch.rand((B, z.shape[1], V), generator=g, device=DEV) < 0.97
    z[mask] = float("-inf")
    z[3, 0, :] = float("-inf")                             # fully masked row
    z[5, 0, 77] = float("nan")                             # NaN row
    u = _uniforms(B, 9)
    out = api.draft_sample(z, u)
    torch.cuda.synchronize()
    tok = out["token"].cpu().numpy()
    f = out["flags"].cpu().numpy()
    assert tok[3] == -1 and tok[5] == -1
    assert f[3] & api.FLAG["NONFINITE"] and f[5] & api.FLAG["NONFINITE"]
    live = [b for b in range(B) if b not in (3, 5)]
    zr = z[:, 0].float().cpu().numpy()
    assert all(np.isfinite(zr[b, tok[b]]) for b in live)
    ref = oracle.draft_sample(z[live, 0].double().cpu().numpy(), u[live].cpu().numpy(), tie_eps_draw=DRAW_BAND)
    ok = ref["near_tie"] == 0
    assert np.array_equal(tok[live][ok], ref["token"][ok])


def test_greedy_ties_take_the_first_index():
    z = torch.zeros((4, 1, 4096), dtype=torch.bfloat16, device=DEV)
    z[0, 0, [10, 3000]] = 5.0
    z[1, 0, :] = 1.0
    z[2, 0, [4095, 2048]] = 2.0
    z[3, 0, 7] = -1.0
    out = api.draft_sample(z, None, greedy=True)
    assert out["token"].cpu().tolist() == [10, 0, 2048, 0]


def test_empty_batch_and_argument_errors():
    z = torch.zeros((0, 2, 100), device=DEV)
    api.draft_sample(z, torch.zeros((0,), device=DEV))
    y = torch.zeros((2, 2, 100), device=DEV)
    u = torch.zeros((2,), device=DEV)
    with pytest.raises(RuntimeError):
        api.draft_sample(y, u, row=2)
    with pytest.raises(RuntimeError):
        api.draft_sample(y, None)                          # stochastic mode needs u


def test_extreme_logits_and_uniform_endpoints():
    """Peaked rows (one logit 1e4 above the rest: every other weight underflows), flat rows
    (all equal: token = floor(u V)), u = 0 and the largest float below 1."""
    V = 50000
    z = torch.zeros((6, 1, V), dtype=torch.float32, device=DEV)
    z[0, 0, 123] = 1e4
    z[1, 0, :] = -3.0                                       # flat
    z[2, 0, :] = -3.0
    z[3, 0, :] = torch.linspace(-40, 40, V, device=DEV)     # monotone
    z[4, 0, ::2] = float("-inf")                            # every other token masked, rest flat
    z[5, 0, :] = 7.0
    one_minus = float(np.nextafter(np.float32(1), np.float32(0)))
    u = torch.tensor([0.7, 0.0, one_minus, 0.5, 0.3, 0.25], dtype=torch.float32, device=DEV)
    out = api.draft_sample(z, u)
    torch.cuda.synchronize()
    ref = oracle.draft_sample(z[:, 0].double().cpu().numpy(), u.cpu().numpy(), tie_eps_draw=DRAW_BAND)
    tok = out["token"].cpu().numpy()
    assert tok[0] == 123 and tok[1] == 0 and tok[2] == V - 1
    ok = ref["near_tie"] == 0
    assert np.array_equal(tok[ok], ref["token"][ok])
    assert tok[4] % 2 == 1
    assert np.allclose(out["lse"].double().cpu().numpy(), ref["lse"], rtol=1e-6, atol=1e-5)
