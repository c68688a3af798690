"""GPU parity on the cases round 1 left untested (VERDICT r1 "What's weak" #4): f32 logits over
many slices, non-finite rows through msd_chain_verify, a vanishing residual (RESID_SMALL,
S:97), residual draws whose u Z sits next to a slice boundary, and the per-pair stats against
fixed-point totals formed from the oracle's divergences and lengths.  Plus every sub-chain of
a 4-model pool (the adaptive sweep's chains)."""
import itertools

import numpy as np
import pytest
import torch

import oracle
from paper_2505_07680_b200 import api, synth
from tests._parity import DIV_ABS, DIV_REL, assert_parity, run_oracle, to_np

pytestmark = [pytest.mark.gpu]
DEV = "cuda"


def _gauss(name, **kw):
    c = dict(synth.CONFIGS[name])
    c.update(kw)
    return synth.gauss_chain(c["B"], c["V"], c["K"], c["L"], c["sigmas"], s=c["s"], seed=c["seed"],
                             device=DEV, dtype=c["dtype"])


def _run(inp, **kw):
    o = api.chain_verify(inp.levels, inp.draft, inp.u_acc, inp.u_emit, V=inp.V, **kw)
    torch.cuda.synchronize()
    return o


def slice_geometry(V, VS=4096, REF=148):
    """The tail's slice geometry (msd_common.cuh slice_geometry), for placing test uniforms."""
    used = lambda c: (REF // ((c + 1) // 2)) * ((c + 1) // 2)
    cmin = (V + VS - 1) // VS
    best, u0 = cmin, used(cmin)
    for c in range(cmin + 1, cmin + cmin // 4 + 1):
        if used(c) > u0 or (used(c) == u0 and best % 2 and not c % 2):
            best, u0 = c, used(c)
    return best, ((V + best - 1) // best + 7) // 8 * 8


@pytest.mark.parametrize("greedy", [False, True])
def test_f32_logits_full_vocabulary(greedy):
    # f32 items hold one tail slice each: 32 CTAs per unit at V = 128256 (multi-slice exchange)
    inp = _gauss("llama3", B=6, dtype="f32")
    o = _run(inp, greedy=greedy)
    assert_parity(o, run_oracle(inp, greedy=greedy))
    assert not (to_np(o)["flags"] & api.FLAG["TIMEOUT"]).any()


def test_nonfinite_rows_flagged_like_the_oracle():
    inp = _gauss("llama3", B=6, V=20000)
    inp.levels[1][0, 2, 777] = float("nan")            # NaN in a verifier row
    inp.levels[2][1, 0, 5] = float("inf")              # +inf in the target row
    inp.levels[0][2, 3, 19999] = float("nan")          # NaN in the drafter row (last entry)
    o = to_np(_run(inp))
    ref = run_oracle(inp)
    nf = api.FLAG["NONFINITE"]
    assert ((o["flags"] & nf) != 0).tolist() == ((ref["flags"] & nf) != 0).tolist()
    assert (o["flags"][:3] & nf).all()
    ok = [b for b in range(inp.B) if not (ref["flags"][b] & nf)]
    for b in ok:
        if ref["near_tie"][b]:
            continue
        assert o["commit_len"][b] == ref["out_len"][b] and (o["commit_tok"][b] == ref["out_tok"][b]).all()


def test_vanishing_residual_falls_back_to_the_target():
    # p and q equal except one tiny-probability candidate t whose logit is eps lower under the
    # verifier: p(t)/q(t) = e^-eps, and the residual mass Z = sum max(p - q, 0) ~ q(t) eps ~ 1e-13.
    # A rejection at t (u above the ratio) must draw from p -> RESID_SMALL, same token as
    # the oracle.
    V, K, B = 3000, 3, 2
    g = torch.Generator().manual_seed(11)
    base = torch.randn((B, K + 1, V), generator=g, dtype=torch.float64) * 2.0
    t = 1234
    base[:, :, t] = base.max() - 36.0                   # q(t) ~ 1e-15 .. 1e-13
    q = base[:, :K].clone()
    p = base.clone()
    eps = 1e-5
    p[:, :, t] -= eps
    levels = [q.float().to(DEV), p.float().to(DEV)]
    draft = torch.full((B, K), t, dtype=torch.int32)
    u_acc = torch.full((1, B, K + 1), 0.999995, dtype=torch.float32)   # ratio 1 - 1e-5 < u: reject
    u_emit = torch.rand((1, B, K + 1), generator=g).float()             # [L-1][B][K+L-1]
    o = to_np(api.chain_verify(levels, draft.to(DEV), u_acc.to(DEV), u_emit.to(DEV), V=V))
    torch.cuda.synchronize()
    ref = oracle.chain_verify([x.cpu().numpy() for x in levels], draft.numpy(), u_acc.numpy(), u_emit.numpy(),
                              tie_eps=1e-6, tie_eps_draw=1e-7)
    assert (o["n_acc"][0] == 0).all() and (ref["n_acc"][0] == 0).all()
    assert (o["flags"] & api.FLAG["RESID_SMALL"]).all()
    for b in range(B):
        if not ref["near_tie"][b]:
            assert o["commit_tok"][b, 0] == ref["out_tok"][b, 0]


@pytest.mark.parametrize("delta", [-1e-5, -1e-6, -2e-7, 2e-7, 1e-6, 1e-5])
def test_residual_draw_next_to_a_slice_boundary(delta):
    # 2-level chain; for requests that reject at position n, place u_emit so that u Z lies
    # delta Z from the exact float64 prefix C_s of a slice boundary s (the fp32-derived slice
    # prefix is off by ~1e-7 Z): the token must equal the oracle's (outside the oracle's band)
    V = 40000
    C, VSe = slice_geometry(V)
    inp = _gauss("llama2", B=24, V=V)
    first = run_oracle(inp)
    z = [t[:, :, :V].double().cpu().numpy() for t in inp.levels]
    ue = inp.u_emit.clone().cpu()
    placed = 0
    rng = np.random.default_rng(int(abs(delta) * 1e9) + (delta > 0))
    for b in range(inp.B):
        n = int(first["n_acc"][0, b])
        if n >= inp.K:
            continue
        lp = z[1][b, n] - np.logaddexp.reduce(z[1][b, n])
        lq = z[0][b, n] - np.logaddexp.reduce(z[0][b, n])
        w = np.maximum(np.exp(lp) - np.exp(lq), 0.0)
        Z = w.sum()
        s = int(rng.integers(1, C))
        Cs = w[: s * VSe].sum()
        u = (Cs + delta * Z) / Z
        if 0.0 < u < 1.0:
            ue[0, b, n] = float(np.float32(u))
            placed += 1
    assert placed >= 5
    inp.u_emit.copy_(ue.to(DEV))
    ref = run_oracle(inp)
    # many residual weights are tiny, so u often lands within the oracle's 1e-7 band of the
    # drawn token's own boundaries (excused); every other placed draw must match
    assert_parity(_run(inp), ref, max_near_tie_frac=1.0)
    assert (ref["near_tie"] == 0).sum() >= 8


def test_stats_match_oracle_fixed_point_totals():
    inp = _gauss("llama3", B=24, V=30000)
    o = to_np(_run(inp))
    ref = run_oracle(inp)
    F = api.STATS_FIELDS
    st = o["stats"]
    for l in range(inp.L - 1):
        d = ref["pos_dtv"][l]
        exp_fx = np.rint(d * api.DTV_SCALE).sum()
        tol = (DIV_REL * np.abs(d) + DIV_ABS).sum() * api.DTV_SCALE + d.size
        assert abs(st[l, F.index("dtv_fx")] - exp_fx) <= tol
        k = ref["pos_kl"][l]
        exp_kfx = np.rint(np.minimum(k, 2 ** 20) * api.KL_SCALE).sum()
        ktol = (DIV_REL * np.abs(k) + DIV_ABS).sum() * api.KL_SCALE + k.size
        assert abs(st[l, F.index("kl_fx")] - exp_kfx) <= ktol
        assert st[l, F.index("positions")] == inp.B * inp.K
        if not ref["near_tie"].any():
            assert st[l, F.index("accepted")] == ref["n_acc"][l].sum()
            assert st[l, F.index("proposed")] == ref["m_cand"][l].sum()


CHAINS = [c for n in range(1, 4) for c in itertools.combinations(range(3), n)]


@pytest.mark.parametrize("pre", CHAINS, ids=["-".join(map(str, c)) for c in CHAINS])
def test_every_subchain_of_a_four_model_pool(pre):
    # the adaptive sweep's 7 chains of 2-4 levels ending at the target (Alg. 1 candidates):
    # levels = the pool models' logits, draft tokens from the chain's first model
    pool = _gauss("sweep", B=6, V=20000)
    chain = list(pre) + [3]
    n, K = len(chain), pool.K
    levels = [pool.levels[m] for m in chain]
    draft = synth.draft_tokens(pool.levels[chain[0]], K, pool.V, seed=5, salt=chain[0])
    ua = pool.u_acc[:n - 1, :, :K + n - 1].contiguous()
    ue = pool.u_emit[:n - 1, :, :K + n - 1].contiguous()
    o = api.chain_verify(levels, draft, ua, ue, V=pool.V)
    torch.cuda.synchronize()
    ref = oracle.chain_verify([t[:, :, :pool.V].float().cpu().numpy() for t in levels], draft.cpu().numpy(),
                              ua.cpu().numpy(), ue.cpu().numpy(), tie_eps=1e-6, tie_eps_draw=1e-7)
    assert_parity(o, ref)


@pytest.fixture
def knobs():
    yield api.debug_knobs
    api.debug_knobs()


def test_exact_draws_shared_across_ctas_are_deterministic(knobs):
    # every draw exact: up to 2 jobs per request posted on the job board and split over the
    # CTAs that finished their own request; chunk sums are combined in a fixed order, so the
    # outputs must be bit-identical run to run and equal the oracle's
    inp = _gauss("qwen25", B=40, V=50000)
    knobs(exact_draws=True)
    a = {k: v.clone() for k, v in _run(inp).items()}
    b = _run(inp)
    for k in a:
        assert torch.equal(a[k], b[k]), k
    assert_parity(b, run_oracle(inp))
    assert (to_np(b)["flags"] & api.FLAG["EXACT_DRAW"]).sum() > 0


@pytest.mark.parametrize("sigmas,seed", [((0.12, 0.06, 0.0), 3), ((0.3, 0.05, 0.0), 4)])
def test_small_residual_masses_on_the_fast_path(sigmas, seed):
    # near-identical levels: residual masses Z mostly in [1e-3, 5e-2]; draws with Z >= 0.01 are
    # decided from the core's fp32-derived slice masses (R4) and must equal the oracle
    inp = _gauss("llama3", B=40, V=60000, sigmas=sigmas, seed=seed)
    o = _run(inp)
    assert float(o["pos_dtv"].median()) < 0.06
    ref = run_oracle(inp)
    assert_parity(o, ref, check_divergence=False)
    # DTV: the plain bound.  KL of near-identical rows (KL ~ 1e-4): the row normalisers carry the
    # fp32 exponent error of their dominant entries (ex2.approx 2^-22 plus the argument rounding,
    # ~2e-7 relative each), which enters KL as an absolute error -- DESIGN.md R18 (KL floor for
    # KL < 3e-3, measured p99 1.5e-7, max 3.1e-7: profiles/r02c_kl_err.txt)
    g = to_np(o)
    d, dr = g["pos_dtv"].astype(np.float64), ref["pos_dtv"]
    assert (np.abs(d - dr) <= DIV_REL * np.abs(dr) + DIV_ABS).all()
    k, kr = g["pos_kl"].astype(np.float64), ref["pos_kl"]
    fin = np.isfinite(kr)
    assert (np.abs(k - kr)[fin] <= (DIV_REL * np.abs(kr) + 5e-7)[fin]).all()
    assert np.percentile(np.abs(k - kr)[fin], 99) <= 2e-7
