"""N > 1 plumbing on CPU (world_size 2, gloo): request sharding, the int64 per-pair stats
all-reduce and the scheduler decision.

Per-request stats come from the float64 oracle (tests may call oracle/) and are encoded
with the fixed point include/msd.h defines (MSD_DTV_SCALE / MSD_KL_SCALE); the checks are
that sharded inputs equal the unsharded ones request by request, that the all-reduced
totals are bit-identical on every rank and equal to the single-process totals, and that
every rank takes the same chain decision.
"""
import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2505_07680_b200 import synth
from paper_2505_07680_b200 import dist as mdist

V, K, L, SIG = 512, 4, 3, (0.7, 0.35, 0.0)
B_LOCAL = 6
DTV_SCALE, KL_SCALE = 4294967296.0, 268435456.0   # include/msd.h


def _inputs(B, req0):
    return synth.gauss_chain(B, V, K, L, SIG, s=4.0, seed=11, req0=req0, device="cpu", dtype="f32")


def _pair_stats(inp):
    """[L-1, 8] int64 msd_pair_stats of a shard, via the oracle and the ABI fixed point."""
    levels = [t.numpy() for t in inp.levels]
    o = oracle.chain_verify(levels, inp.draft.numpy(), inp.u_acc.numpy(), inp.u_emit.numpy(), tie_eps_draw=1e-7)
    st = np.zeros((L - 1, 8), np.int64)
    for l in range(L - 1):
        d = np.clip(o["pos_dtv"][l], 0.0, 1.0)
        k = o["pos_kl"][l]
        fin = np.isfinite(k)
        st[l, 0] = int(sum(int(np.rint(x * DTV_SCALE)) for x in d.ravel()))
        st[l, 1] = int(sum(int(np.rint(min(max(x, 0.0), 1048576.0) * KL_SCALE)) for x in k[fin].ravel()))
        st[l, 2] = d.size
        st[l, 3] = int(o["m_cand"][l].sum())
        st[l, 4] = int(o["n_acc"][l].sum())
        st[l, 7] = int((~fin).sum())
    return st


def _pool_stats(inp):
    """[L(L-1)/2, 8] int64 bootstrap stats of a shard's draft rows, via the oracle."""
    dtv, _ = oracle.pool_divergence([t[:, :K].numpy() for t in inp.levels])
    st = np.zeros((dtv.shape[0], 8), np.int64)
    for q in range(dtv.shape[0]):
        st[q, 0] = int(sum(int(np.rint(min(max(x, 0.0), 1.0) * DTV_SCALE)) for x in dtv[q].ravel()))
        st[q, 2] = dtv[q].size
    return st


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), WORLD_SIZE=str(world), RANK=str(rank),
                      LOCAL_RANK=str(rank))
    try:
        ws, r, _ = mdist.init_from_env("gloo")
        req0, b = mdist.shard(B_LOCAL, ws, r, "weak")
        inp = _inputs(b, req0)
        stats = torch.from_numpy(_pair_stats(inp))
        mdist.allreduce_stats(stats)
        sch = mdist.ChainScheduler(T_ms=[1.0, 3.0, 10.0], W=K)
        chain = sch.update(stats.tolist())
        pool = torch.from_numpy(_pool_stats(inp))
        mdist.allreduce_stats(pool)
        boot = mdist.ChainScheduler(T_ms=[1.0, 3.0, 10.0], W=K)
        bchain = boot.bootstrap(pool.tolist())
        # numpy copies only: torch tensors would travel as shared-memory handles, which the parent
        # cannot open once this process has exited
        q.put((r, req0, b, stats.numpy().copy(), chain, sch.t_eff, [t[:, :, :8].numpy().copy() for t in inp.levels],
               pool.numpy().copy(), bchain, boot.sim))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # surface the failure in the parent
        q.put((rank, "error", repr(e)))


@pytest.fixture(scope="module")
def two_ranks():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    out = [q.get(timeout=240) for _ in ps]
    for p in ps:
        p.join(timeout=60)
    for o in out:
        assert o[1] != "error", o
    return sorted(out, key=lambda o: o[0])


def test_shards_are_disjoint_and_cover_the_batch():
    for world in (1, 2, 3, 8):
        Bg = 37
        got = []
        for r in range(world):
            r0, b = mdist.shard(Bg, world, r, "strong")
            got += list(range(r0, r0 + b))
        assert got == list(range(Bg))
        for r in range(world):
            assert mdist.shard(Bg, world, r, "weak") == (r * Bg, Bg)


def test_sharded_inputs_equal_unsharded(two_ranks):
    full = _inputs(2 * B_LOCAL, 0)
    for r, req0, b, _, _, _, lv in (o[:7] for o in two_ranks):
        for l in range(L):
            assert np.array_equal(lv[l], full.levels[l][req0:req0 + b, :, :8].numpy())


def test_allreduced_stats_identical_and_exact(two_ranks):
    (_, _, _, s0, c0, t0), (_, _, _, s1, c1, t1) = (o[:6] for o in two_ranks)
    assert np.array_equal(s0, s1)
    single = _pair_stats(_inputs(2 * B_LOCAL, 0))
    assert np.array_equal(s0, single)          # integer sums: G-invariant, bit-exact
    assert s0[0, 2] == 2 * B_LOCAL * K
    assert c0 == c1 and t0 == t1               # every rank takes the same decision


def test_scheduler_decision_matches_single_process(two_ranks):
    _, _, _, s0, c0, t0 = two_ranks[0][:6]
    single = _pair_stats(_inputs(2 * B_LOCAL, 0))
    sch = mdist.ChainScheduler(T_ms=[1.0, 3.0, 10.0], W=K)
    assert sch.update(single.tolist()) == c0
    assert math.isclose(sch.t_eff, t0, rel_tol=0, abs_tol=0)
    # SimScore = 1 - mean DTV of each adjacent pair (Eq. 6), first update takes the observation
    for l in range(L - 1):
        assert math.isclose(sch.sim[l][l + 1], 1.0 - single[l, 0] / (DTV_SCALE * single[l, 2]), rel_tol=1e-12)


def test_allreduce_rejects_non_integer_stats():
    with pytest.raises(TypeError):
        mdist.allreduce_stats(torch.zeros(2, 8))


def test_bootstrap_stats_and_decision_match_single_process(two_ranks):
    """SimScore bootstrap across ranks: the all-reduced pool stats are bit-identical
    on both ranks and equal to the single-process totals, so both ranks bootstrap the same
    P x P SimScore matrix and take the same Alg. 1 decision."""
    p0, b0, m0 = two_ranks[0][7:10]
    p1, b1, m1 = two_ranks[1][7:10]
    assert np.array_equal(p0, p1) and b0 == b1 and m0 == m1
    single = _pool_stats(_inputs(2 * B_LOCAL, 0))
    assert np.array_equal(p0, single)
    sch = mdist.ChainScheduler(T_ms=[1.0, 3.0, 10.0], W=K)
    assert sch.bootstrap(single.tolist()) == b0
    assert sch.sim == m0
