"""Seeded synthetic inputs shaped like the paper's model chains.

This module is the ONLY code shared by the CUDA path and the oracle: it draws
random numbers and lays them out.  It contains none of the method's arithmetic
(no softmax, no acceptance test, no divergence, no rollback).  Recipe (DESIGN.md
"Input recipe"):

* gauss-noise family (throughput + parity): target logits ``Z_L = s * N(0,1)``,
  level l logits ``Z_l = Z_L + sigma_l * N(0,1)`` (per row, per vocab entry),
  rounded to the logit dtype (bf16 for the paper's models).
* draft tokens ``x[b,i] = argmax_v (Z_1[b,i,v] + G_v)`` with Gumbel noise G
  (the Gumbel-max trick draws x ~ softmax(Z_1) without forming the softmax).
* uniforms: float32 in [0, 1).

Every request b draws from its own generator seeded by (seed, global request id),
so shard g of G ranks reproduces exactly the rows of the G=1 run (G-invariance).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Optional

import torch

# Llama-3 / Qwen2.5 / Llama-2 chains of BASELINE.json, sigmas chosen in SURVEY §8(d).
CONFIGS = {
    "tiny": dict(B=4, V=1000, K=4, L=2, dtype="f32", sigmas=(0.75, 0.0), s=4.0, seed=1),
    "llama2": dict(B=64, V=32000, K=5, L=2, dtype="bf16", sigmas=(0.75, 0.0), s=4.0, seed=2),
    "qwen25": dict(B=256, V=151936, K=6, L=3, dtype="bf16", sigmas=(0.7, 0.35, 0.0), s=4.0, seed=3),
    "llama3": dict(B=512, V=128256, K=8, L=3, dtype="bf16", sigmas=(0.7, 0.35, 0.0), s=4.0, seed=4),
    "sweep": dict(B=512, V=128256, K=6, L=4, dtype="bf16", sigmas=(1.5, 1.0, 0.5, 0.0), s=4.0, seed=5),
}

_DT = {"bf16": torch.bfloat16, "f32": torch.float32}


def _mix(seed: int, req: int, salt: int = 0) -> int:
    x = (seed * 0x9E3779B97F4A7C15 + req * 0xBF58476D1CE4E5B9 + salt * 0x94D049BB133111EB)
    x &= (1 << 64) - 1
    x ^= x >> 31
    x = (x * 0xD6E8FEB86659FD93) & ((1 << 64) - 1)
    x ^= x >> 32
    return x & ((1 << 63) - 1)


def level_rows(L: int, K: int, intermediate_bonus: bool = True) -> List[int]:
    """Rows supplied per level: drafter K; verifier l gets K+l rows with intermediate
    bonus (its candidates can grow by one per level), else K+1."""
    return [K] + [(K + l) if intermediate_bonus else (K + 1) for l in range(1, L)]


@dataclass
class ChainInputs:
    levels: List[torch.Tensor]          # L tensors [B, R_l, ld] (first V columns valid)
    draft: torch.Tensor                 # [B, K] int32
    u_acc: torch.Tensor                 # [L-1, B, K+L-1] float32
    u_emit: torch.Tensor                # [L-1, B, K+L-1] float32
    V: int
    K: int
    req0: int = 0
    meta: dict = field(default_factory=dict)

    @property
    def B(self) -> int:
        return self.draft.shape[0]

    @property
    def L(self) -> int:
        return len(self.levels)

    def logit_bytes(self) -> int:
        return sum(t.numel() * t.element_size() for t in self.levels)


def gauss_chain(B: int, V: int, K: int, L: int, sigmas, *, s: float = 4.0, seed: int = 0,
                req0: int = 0, device="cpu", dtype="bf16", ld: Optional[int] = None,
                intermediate_bonus: bool = True) -> ChainInputs:
    """Gauss-noise family for global requests [req0, req0+B)."""
    assert len(sigmas) == L and sigmas[-1] == 0.0
    tdt = _DT[dtype] if isinstance(dtype, str) else dtype
    ld = V if ld is None else ld
    rows = level_rows(L, K, intermediate_bonus)
    R = max(rows)
    W = K + L - 1
    levels = [torch.empty((B, r, ld), dtype=tdt, device=device) for r in rows]
    if ld > V:
        for t in levels:
            t[:, :, V:] = float("nan")          # padding must never be read
    draft = torch.empty((B, K), dtype=torch.int32, device=device)
    u_acc = torch.empty((L - 1, B, W), dtype=torch.float32, device=device)
    u_emit = torch.empty((L - 1, B, W), dtype=torch.float32, device=device)
    gen = torch.Generator(device=device)
    for b in range(B):
        gen.manual_seed(_mix(seed, req0 + b))
        base = torch.randn((R, V), generator=gen, device=device) * s
        for l in range(L):
            noise = torch.randn((rows[l], V), generator=gen, device=device)
            z = base[: rows[l]] + sigmas[l] * noise if sigmas[l] != 0.0 else base[: rows[l]]
            levels[l][b, :, :V] = z.to(tdt)
        g = torch.rand((K, V), generator=gen, device=device).clamp_(min=1e-30)
        gumbel = -torch.log(-torch.log(g))
        draft[b] = (levels[0][b, :K, :V].float() + gumbel).argmax(dim=1).to(torch.int32)
        uu = torch.rand((2, L - 1, W), generator=gen, device=device)
        u_acc[:, b] = uu[0]
        u_emit[:, b] = uu[1]
    return ChainInputs(levels=levels, draft=draft, u_acc=u_acc, u_emit=u_emit, V=V, K=K,
                       req0=req0, meta=dict(family="gauss", sigmas=tuple(sigmas), s=s, seed=seed))


def config_inputs(name: str, *, B: Optional[int] = None, req0: int = 0, device="cpu",
                  seed: Optional[int] = None, V: Optional[int] = None) -> ChainInputs:
    c = dict(CONFIGS[name])
    if B is not None:
        c["B"] = B
    if V is not None:
        c["V"] = V
    return gauss_chain(c["B"], c["V"], c["K"], c["L"], c["sigmas"], s=c["s"],
                       seed=c["seed"] if seed is None else seed, req0=req0, device=device,
                       dtype=c["dtype"])


def uniform_grid(n: int, device="cpu") -> torch.Tensor:
    """Midpoints of n equal intervals of [0,1) (brute-force enumeration pins)."""
    return (torch.arange(n, dtype=torch.float64, device=device) + 0.5) / n


def paged_kv(B: int, n_models: int, *, seed: int, block_size: int = 16, min_len: int = 512,
             max_len: int = 4096, extra: int = 0, device="cpu"):
    """Per-model paged KV metadata: seq_len ~ U[min_len, max_len] (+ extra speculative
    slots), block ids a seeded permutation of the pool, a free stack with room for
    every block.  Returns a list of dicts of tensors."""
    out = []
    for mdl in range(n_models):
        gen = torch.Generator(device="cpu")
        gen.manual_seed(_mix(seed, mdl, salt=7))
        seq = torch.randint(min_len, max_len + 1, (B,), generator=gen, dtype=torch.int32) + extra
        max_blocks = (max_len + extra + block_size - 1) // block_size
        nblk = (seq + block_size - 1) // block_size
        total = int(nblk.sum())
        pool = B * max_blocks
        perm = torch.randperm(pool, generator=gen).to(torch.int32)
        bt = torch.full((B, max_blocks), -1, dtype=torch.int32)
        off = 0
        for b in range(B):
            n = int(nblk[b])
            bt[b, :n] = perm[off: off + n]
            off += n
        free_ids = torch.full((pool,), -1, dtype=torch.int32)
        nfree = pool - total
        free_ids[:nfree] = perm[total:]
        out.append(dict(seq_len=seq.to(device), block_table=bt.to(device),
                        free_ids=free_ids.to(device),
                        free_count=torch.tensor([nfree], dtype=torch.int32, device=device),
                        block_size=block_size, max_blocks=max_blocks))
    return out


def draft_tokens(z: torch.Tensor, K: int, V: int, *, seed: int, req0: int = 0, salt: int = 0) -> torch.Tensor:
    """Draft tokens x[b,i] ~ softmax(z[b,i,:V]) for i < K by the Gumbel-max trick, one generator
    per request (seed, global request id, salt) -- the drafter of a sub-chain that does not start
    at the pool's first model (adaptive sweep)."""
    B = z.shape[0]
    out = torch.empty((B, K), dtype=torch.int32, device=z.device)
    gen = torch.Generator(device=z.device)
    for b in range(B):
        gen.manual_seed(_mix(seed, req0 + b, salt=100 + salt))
        g = torch.rand((K, V), generator=gen, device=z.device).clamp_(min=1e-30)
        out[b] = (z[b, :K, :V].float() - torch.log(-torch.log(g))).argmax(dim=1).to(torch.int32)
    return out
