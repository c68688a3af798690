"""Multi-GPU plumbing of the hot path: request sharding, the int64
per-pair stats all-reduce, and the host scheduler feed (EMA SimScore -> alpha -> Eq. 7 ->
Alg. 1).

The verification path shards by request: every request's rows, candidates and KV live on
one rank, so the data path has no collective (weak scaling).  The only exchange is the
[L-1] x 8 int64 ``msd_pair_stats`` vector (<= 192 B): integer sums are exact and
order-independent, so every rank holds bit-identical totals after a SUM all-reduce and
takes the same scheduling decision ("adaptive model chain scheduling", Alg. 1
P:206-236).  The backend is whatever ``torch.distributed`` was initialised with (NCCL on
the GPU box, gloo in the CPU tests).
"""
from __future__ import annotations

import os
from dataclasses import dataclass, field

import torch

from . import api


def init_from_env(backend: str | None = None):
    """(world_size, rank, local_rank); initialises the default process group when the
    launcher (torchrun) set WORLD_SIZE > 1.  Rendezvous address comes from MASTER_ADDR
    (use 127.0.0.1 on these boxes)."""
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1 and not torch.distributed.is_initialized():
        torch.distributed.init_process_group(backend or ("nccl" if torch.cuda.is_available() else "gloo"))
    return ws, rank, local


def shard(B_global: int, world: int, rank: int, scaling: str = "weak") -> tuple[int, int]:
    """(first global request id, local batch) of `rank`.  Weak scaling: every rank owns
    B_global requests (ids rank*B_global ...); strong: B_global is split in contiguous
    blocks, the first B_global % world ranks taking one extra request."""
    if scaling == "weak":
        return rank * B_global, B_global
    base, extra = divmod(B_global, world)
    b = base + (1 if rank < extra else 0)
    r0 = rank * base + min(rank, extra)
    return r0, b


def allreduce_stats(stats: torch.Tensor) -> torch.Tensor:
    """In-place SUM all-reduce of an int64 [L-1, 8] msd_pair_stats tensor (no-op at N=1)."""
    if stats.dtype != torch.int64:
        raise TypeError("msd_pair_stats is int64")
    if torch.distributed.is_available() and torch.distributed.is_initialized() and \
            torch.distributed.get_world_size() > 1:
        torch.distributed.all_reduce(stats, op=torch.distributed.ReduceOp.SUM)
    return stats


@dataclass
class ChainScheduler:
    """Host scheduler fed by the reduced per-pair stats (row a8) over a pool of P models.

    sim: P x P SimScores (EMA of 1 - mean DTV, Eq. 6, weight `ema`, R13); alpha =
    SimScore (R11).  `bootstrap` initialises every pair from msd_pool_divergence stats
    (observation count 1); `update` folds one step's stats of the running chain's
    adjacent pairs into their SimScores; the next chain is Alg. 1's argmin of Eq. 7's T_eff
    over every chain of the pool that ends at the target.  Without a bootstrap a
    pair's SimScore starts at the `prior` (0.5) until the chain first runs it.
    """
    T_ms: list
    W: int
    ema: float = 0.1
    max_len: int = 4
    prior: float = 0.5
    sim: list = field(default_factory=list)          # P x P
    seen: list = field(default_factory=list)         # P x P: pair has an observation
    chain: list = field(default_factory=list)
    t_eff: float | None = None

    def __post_init__(self):
        P = len(self.T_ms)
        if not self.sim:
            self.sim = [[1.0 if i == j else self.prior for j in range(P)] for i in range(P)]
        if not self.seen:
            self.seen = [[i == j for j in range(P)] for i in range(P)]
        if not self.chain:
            self.chain = list(range(P))

    def _fold(self, i, j, stats_row):
        first = not self.seen[i][j]
        v = api.simscore_update(self.sim[i][j], stats_row, self.ema, first)
        self.sim[i][j] = self.sim[j][i] = v
        self.seen[i][j] = self.seen[j][i] = True

    def bootstrap(self, pool_stats) -> list:
        """pool_stats: [P(P-1)/2][8] int64 totals of msd_pool_divergence (pairs i < j in
        lexicographic order, all ranks identical after allreduce_stats)."""
        P = len(self.T_ms)
        q = 0
        for i in range(P):
            for j in range(i + 1, P):
                self.seen[i][j] = self.seen[j][i] = False
                self._fold(i, j, pool_stats[q])
                q += 1
        return self._select()

    def update(self, stats_rows, chain=None) -> list:
        """stats_rows: [len(chain)-1][8] int64 totals of the adjacent pairs of the chain that
        ran (default: the last selected chain)."""
        ran = list(self.chain if chain is None else chain)
        for l in range(len(ran) - 1):
            self._fold(ran[l], ran[l + 1], stats_rows[l])
        return self._select()

    def _select(self) -> list:
        self.chain, self.t_eff = api.select_chain(self.T_ms, self.sim, self.W, max_len=self.max_len)
        return self.chain
