"""GPU parity of msd_chain_verify_lse (the producer -- the lm_head epilogue --
supplies every draft-position row's normaliser, so the core needs no cross-CTA exchange): the
outputs must equal the float64 oracle's on the same logits, like msd_chain_verify's."""
import pytest
import torch

from paper_2505_07680_b200 import api, synth
from tests._parity import assert_parity, run_oracle

pytestmark = [pytest.mark.gpu]
DEV = "cuda"


def _gauss(name, **kw):
    c = dict(synth.CONFIGS[name])
    c.update(kw)
    return synth.gauss_chain(c["B"], c["V"], c["K"], c["L"], c["sigmas"], s=c["s"], seed=c["seed"],
                             device=DEV, dtype=c["dtype"])


def _lse(inp):
    # row normalisers of the supplied rows i < K (float64; the producer's job)
    return torch.stack([torch.logsumexp(t[:, :inp.K, :inp.V].double(), dim=-1) for t in inp.levels]).contiguous()


def _run(inp, **kw):
    cv = api.ChainVerify(inp.levels, inp.draft, inp.u_acc, inp.u_emit, V=inp.V, lse=_lse(inp), **kw)
    cv()
    torch.cuda.synchronize()
    return cv.outputs()


@pytest.mark.parametrize("name,kw", [("llama3", dict(B=12, V=40000)), ("qwen25", dict(B=8, V=151936)),
                                     ("tiny", {}), ("sweep", dict(B=6, V=30000)), ("llama2", dict(B=16))])
def test_lse_fed_chain_matches_oracle(name, kw):
    inp = _gauss(name, **kw)
    assert_parity(_run(inp), run_oracle(inp))


def test_lse_fed_greedy_and_agreement_with_the_exchange_path():
    inp = _gauss("llama3", B=16, V=50000)
    assert_parity(_run(inp, greedy=True), run_oracle(inp, greedy=True))
    a = _run(inp)
    b = api.chain_verify(inp.levels, inp.draft, inp.u_acc, inp.u_emit, V=inp.V)
    torch.cuda.synchronize()
    for k in ("n_acc", "m_cand", "commit_len"):
        assert torch.equal(a[k], b[k]), k
    d = (a["pos_dtv"].double() - b["pos_dtv"].double()).abs()
    assert float(d.max()) < 5e-7
