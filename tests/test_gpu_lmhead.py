"""GPU parity of the fused lm_head GEMM + row normaliser (msd_lmhead_lse, SURVEY 8(f) NEXT-2,
Eq. 1): LSE of z = H W^T and the candidate logits, against float64 logits formed from
the same bf16 H and W (the oracle's LSE definition).  Tolerance from the arithmetic: bf16 products
are exact in fp32 and the tensor cores accumulate D of them in fp32, so |dz_v| <= gamma_D sum_k
|h_k w_vk| with gamma_D = D 2^-24 (the standard summation bound), and |dLSE| <= max_v |dz_v|
plus the fp32/fp64 reduction error (1e-6 relative)."""
import numpy as np
import pytest
import torch

import oracle
from paper_2505_07680_b200 import api

pytestmark = [pytest.mark.gpu]


def _case(M, D, V, seed):
    g = torch.Generator().manual_seed(seed)
    H = torch.randn((M, D), generator=g).to(torch.bfloat16)
    W = (torch.randn((V, D), generator=g) * (4.0 / D ** 0.5)).to(torch.bfloat16)
    cand = torch.randint(0, V, (M,), generator=g, dtype=torch.int32)
    cand[0] = -1
    cand[min(1, M - 1)] = V + 3
    return H, W, cand


def _check(H, W, cand, rows):
    out = api.lmhead_lse(H.cuda(), W.cuda(), cand.cuda())
    torch.cuda.synchronize()
    lse = out["lse"].cpu().numpy()
    zc = out["z_cand"].cpu().numpy()
    Hd, Wd = H.double().numpy(), W.double().numpy()
    D = H.shape[1]
    gamma = D * 2.0 ** -24
    for r in rows:
        z = Wd @ Hd[r]                                     # float64 logits of row r
        bound = gamma * (np.abs(Wd) @ np.abs(Hd[r]))        # per-logit summation bound
        ref = oracle.lse(z)
        assert abs(lse[r] - ref) <= bound.max() + 1e-6 * abs(ref) + 1e-6, (r, lse[r], ref)
        c = int(cand[r])
        if 0 <= c < W.shape[0]:
            assert abs(zc[r] - z[c]) <= bound[c] + 1e-6, (r, zc[r], z[c])
        else:
            assert np.isnan(zc[r])
    return out


@pytest.mark.parametrize("M,D,V", [(200, 256, 5000), (128, 64, 256), (37, 128, 1000), (300, 512, 33000)])
def test_lmhead_lse_small_shapes(M, D, V):
    H, W, cand = _case(M, D, V, seed=M + D)
    _check(H, W, cand, range(M))


def test_lmhead_lse_llama3_shape_sampled_rows():
    # the Llama-3 verify batch: B = 512 requests x R = 8 rows, hidden 4096, vocabulary 128256
    H, W, cand = _case(4096, 4096, 128256, seed=3)
    _check(H, W, cand, [0, 1, 127, 128, 2049, 4095])


# ---------------------------------------------------------------- the fused pipeline (NEXT-2)
def test_lmhead_logits_feed_the_exchange_free_verify():
    # per level l: hidden states H_l [B * rows_l, D] and its own vocabulary projection W_l; the
    # lm_head kernel writes bf16 logits and the float64 LSE of exactly those logits, which
    # msd_chain_verify_lse consumes (no cross-CTA exchange in the verify core).  The verify result
    # must equal the oracle's on the same bf16 logits.
    from paper_2505_07680_b200 import synth
    from tests._parity import assert_parity, run_oracle
    B, K, L, D, V = 6, 5, 3, 256, 32003
    g = torch.Generator().manual_seed(7)
    Hb = torch.randn((B, K + L - 1, D), generator=g)
    W0 = torch.randn((V, D), generator=g) * (3.0 / D ** 0.5)
    levels, lses = [], []
    for l in range(L):
        rows = K + l
        # the levels share the target's projection up to a perturbation (a chain of related models)
        W = (W0 + torch.randn((V, D), generator=g) * ((0.35 * (L - 1 - l)) / D ** 0.5)).to(torch.bfloat16).cuda()
        H = Hb[:, :rows].reshape(B * rows, D).to(torch.bfloat16).cuda().contiguous()
        out = api.lmhead_logits(H, W)
        torch.cuda.synchronize()
        z = out["logits"].view(B, rows, -1)
        levels.append(z)
        lses.append(out["lse64"].view(B, rows)[:, :K])
        ref = torch.logsumexp(z[:, :, :V].double(), dim=-1)
        assert float((out["lse64"].view(B, rows) - ref).abs().max()) < 2e-6      # LSE of the written logits
    lse = torch.stack(lses).contiguous()
    draft = synth.draft_tokens(levels[0], K, V, seed=3)
    gu = torch.Generator().manual_seed(9)
    ua = torch.rand((L - 1, B, K + L - 1), generator=gu).cuda()
    ue = torch.rand((L - 1, B, K + L - 1), generator=gu).cuda()
    inp = synth.ChainInputs(levels=levels, draft=draft, u_acc=ua, u_emit=ue, V=V, K=K)
    cv = api.ChainVerify(levels, draft, ua, ue, V=V, lse=lse)
    cv()
    torch.cuda.synchronize()
    assert_parity(cv.outputs(), run_oracle(inp))
