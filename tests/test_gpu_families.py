"""GPU parity on the correctness families of SURVEY 8(d) that the gauss-noise throughput family does
not cover: mixture drafters q = (1 - eps) p + eps U, level-wise constant shifts (the same
distributions: everything accepted, zero divergence), and disjoint / partially masked supports
(KL = +inf, large DTV, q = 0 / p = 0 acceptance rules).  Every case against the float64 oracle."""
import numpy as np
import pytest
import torch

from paper_2505_07680_b200 import api, synth
from tests._parity import assert_parity, run_oracle, to_np

pytestmark = [pytest.mark.gpu]
DEV = "cuda"


def _inputs(levels, K, V, seed):
    draft = synth.draft_tokens(levels[0], K, V, seed=seed)
    L, B = len(levels), levels[0].shape[0]
    g = torch.Generator().manual_seed(seed + 1)
    ua = torch.rand((L - 1, B, K + L - 1), generator=g).to(DEV)
    ue = torch.rand((L - 1, B, K + L - 1), generator=g).to(DEV)
    return synth.ChainInputs(levels=levels, draft=draft, u_acc=ua, u_emit=ue, V=V, K=K)


def _run(inp, **kw):
    o = api.chain_verify(inp.levels, inp.draft, inp.u_acc, inp.u_emit, V=inp.V, **kw)
    torch.cuda.synchronize()
    return o


def _target(B, R, V, seed, s=4.0):
    g = torch.Generator().manual_seed(seed)
    return torch.randn((B, R, V), generator=g, dtype=torch.float64) * s


@pytest.mark.parametrize("eps", [0.1, 0.3, 0.6])
@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
def test_mixture_drafters(eps, dtype):
    # level 0 = (1 - eps) p_1 + eps U, level 1 = (1 - eps / 2) p_2 + eps / 2 U, level 2 = p_2 (target)
    B, K, V = 12, 6, 40000
    z = _target(B, K + 2, V, seed=int(eps * 100))
    p = torch.softmax(z, dim=-1)
    lv = [torch.log((1 - eps) * p + eps / V), torch.log((1 - eps / 2) * p + eps / 2 / V), z]
    levels = [t[:, :K + l].to(dtype).to(DEV).contiguous() for l, t in enumerate(lv)]
    inp = _inputs(levels, K, V, seed=5)
    assert_parity(_run(inp), run_oracle(inp))


def test_constant_shifts_are_the_same_distribution():
    # Z_l = Z + c_l: identical softmax at every level -> every candidate accepted, DTV = KL = 0
    # (logits on a 2^-12 grid, so z + c is exact in fp32: the levels are exactly shifted copies)
    B, K, V = 10, 8, 30000
    z = torch.round(_target(B, K + 2, V, seed=11) * 4096) / 4096
    levels = [(z[:, :K + l] + c).to(torch.float32).to(DEV).contiguous() for l, c in enumerate((0.0, 3.0, -7.5))]
    inp = _inputs(levels, K, V, seed=6)
    o = to_np(_run(inp))
    ref = run_oracle(inp)
    assert_parity(o, ref)
    assert (o["n_acc"] == o["m_cand"]).all()
    assert np.abs(o["pos_dtv"]).max() <= 1e-6 and np.abs(o["pos_kl"]).max() <= 1e-6


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
def test_disjoint_and_partially_masked_supports(dtype):
    # drafter: only the first half of the vocabulary; middle level: everything but a band the
    # drafter favours; target: full support.  KL(p_l || p_{l-1}) = +inf where p_l has mass outside
    # p_{l-1}'s support; p(x) = 0 rejects, q(x) = 0 accepts (R3)
    B, K, V = 10, 6, 20000
    z = _target(B, K + 2, V, seed=21)
    z0 = z[:, :K].clone()
    z0[:, :, V // 2:] = -float("inf")
    z1 = z[:, :K + 1].clone() + torch.randn_like(z[:, :K + 1]) * 0.5
    z1[:, :, 1000:3000] = -float("inf")
    levels = [t.to(dtype).to(DEV).contiguous() for t in (z0, z1, z[:, :K + 2])]
    inp = _inputs(levels, K, V, seed=7)
    o = _run(inp)
    assert_parity(o, run_oracle(inp))
    g = to_np(o)
    assert np.isinf(g["pos_kl"][0]).all()          # the middle level has mass outside the drafter's support
    assert (g["flags"] & api.FLAG["KL_INF"]).all()
