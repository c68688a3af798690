"""Host scheduler feed with the SimScore bootstrap (8(f) NEXT-1):
the bootstrap initialises every pool pair from the pool divergences (observation count 1,
S:475) and Alg. 1 then chooses over every chain of the pool.  Stats are built
from the float64 oracle with the ABI's fixed point (tests may call oracle/)."""
import math

import numpy as np

import oracle
from paper_2505_07680_b200 import api
from paper_2505_07680_b200 import dist as mdist

DTV_SCALE = 4294967296.0


def _pool_stats(levels):
    dtv, _ = oracle.pool_divergence(levels)
    st = np.zeros((dtv.shape[0], 8), np.int64)
    for q in range(dtv.shape[0]):
        st[q, 0] = int(sum(int(np.rint(min(max(x, 0.0), 1.0) * DTV_SCALE)) for x in dtv[q].ravel()))
        st[q, 2] = dtv[q].size
    return st


def _pool(P=4, B=3, K=5, V=300, seed=2):
    rng = np.random.default_rng(seed)
    target = rng.standard_normal((B, K, V)) * 4
    sig = [1.5, 1.0, 0.5, 0.0][-P:]
    return [target + s * rng.standard_normal((B, K, V)) for s in sig]


def test_bootstrap_sets_every_pair_to_one_minus_mean_dtv():
    levels = _pool()
    st = _pool_stats(levels)
    sch = mdist.ChainScheduler(T_ms=[1.0, 3.0, 10.0, 40.0], W=5)
    chain = sch.bootstrap(st.tolist())
    ref = oracle.bootstrap_sim(levels)
    for i in range(4):
        for j in range(4):
            if i != j:
                assert math.isclose(sch.sim[i][j], ref[i, j], rel_tol=0, abs_tol=1e-9)
    # Alg. 1 over the bootstrapped matrix (host C ABI) equals the oracle's brute force
    want, t_eff = oracle.select_chain([1.0, 3.0, 10.0, 40.0], ref, 5, max_len=4)
    assert chain == want and math.isclose(sch.t_eff, t_eff, rel_tol=1e-9)


def test_identical_pool_bootstraps_to_simscore_one():
    """identical models -> all SimScores 1."""
    z = _pool(P=1)[0]
    sch = mdist.ChainScheduler(T_ms=[1.0, 3.0, 10.0], W=5)
    sch.bootstrap(_pool_stats([z, z, z]).tolist())
    assert all(sch.sim[i][j] == 1.0 for i in range(3) for j in range(3))


def test_online_update_folds_only_the_pairs_that_ran():
    levels = _pool()
    sch = mdist.ChainScheduler(T_ms=[1.0, 3.0, 10.0, 40.0], W=5)
    sch.bootstrap(_pool_stats(levels).tolist())
    before = [row[:] for row in sch.sim]
    row = [2 * int(DTV_SCALE), 0, 10, 0, 0, 0, 0, 0]      # mean DTV 0.2 over 10 positions
    sch.update([row], chain=[1, 3])
    assert math.isclose(sch.sim[1][3], 0.1 * 0.8 + 0.9 * before[1][3], rel_tol=1e-12)   # Eq. 6 EMA
    assert sch.sim[3][1] == sch.sim[1][3]
    for i in range(4):
        for j in range(4):
            if {i, j} != {1, 3}:
                assert sch.sim[i][j] == before[i][j]
