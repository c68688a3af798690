"""float64 CPU oracle for the SpecRouter (arxiv 2505.07680) verify / divergence /
KV-rollback hot path -- ctypes wrapper around ``oracle/msd_oracle.c``.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this module.
The product package (``paper_2505_07680_b200``) never imports it and shares no code
with it.  Every C function cites the PAPER.md / SPEC.md passage it follows.

Parity pins live in ``tests/test_oracle_*.py``.  Parity unpinned (definitional
choices): the KL direction (R9), the SimScore->alpha mapping (R11),
the EMA weights (R13).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "msd_oracle.c")
_HDR = os.path.join(_HERE, "msd_oracle.h")
_LIB = os.path.join(_HERE, "liboracle.so")


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (plain C, -O2, OpenMP across requests)."""
    stale = (not os.path.exists(_LIB)) or any(
        os.path.getmtime(p) > os.path.getmtime(_LIB) for p in (_SRC, _HDR))
    if force or stale:
        cmd = ["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-o", _LIB, _SRC, "-lm"]
        subprocess.check_call(cmd)
    return _LIB


_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        d, i32, i64, u32 = ctypes.c_double, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint32
        P = ctypes.c_void_p
        L.or_lse.restype = d; L.or_lse.argtypes = [P, i64]
        L.or_argmax.restype = i64; L.or_argmax.argtypes = [P, i64]
        L.or_dtv.restype = d; L.or_dtv.argtypes = [P, d, P, d, i64]
        L.or_kl.restype = d; L.or_kl.argtypes = [P, d, P, d, i64]
        L.or_accept.restype = ctypes.c_int; L.or_accept.argtypes = [d, d, d, d, d, P]
        L.or_sample.restype = i64; L.or_sample.argtypes = [P, d, i64, d, P]
        L.or_sample_residual.restype = i64
        L.or_sample_residual.argtypes = [P, d, P, d, i64, d, P, P]
        L.or_chain_verify.restype = ctypes.c_int
        L.or_chain_verify.argtypes = [P, i32, i32, i32, i64, P, P, P, P, i64, i64,
                                      i32, i32, i32, i32, d, d,
                                      P, P, P, i32, P, P, P, P, P, P, i32]
        L.or_rollback_mask.restype = None
        L.or_rollback_mask.argtypes = [P, i32, i32, P, P, P]
        L.or_rollback_paged.restype = None
        L.or_rollback_paged.argtypes = [P, P, i32, i32, i32, P, P, i32, P, i32, P, P]
        L.or_expected_accepted.restype = d; L.or_expected_accepted.argtypes = [d, i32]
        L.or_theoretical_speedup.restype = d; L.or_theoretical_speedup.argtypes = [d, i32, d]
        L.or_ema.restype = d; L.or_ema.argtypes = [d, d, d, i32]
        L.or_predict_chain_latency.restype = d
        L.or_predict_chain_latency.argtypes = [i32, P, P, i32, i32, i32]
        L.or_select_chain.restype = i32
        L.or_select_chain.argtypes = [i32, P, P, i32, i32, i32, i32, P, P]
        L.or_pool_divergence.restype = None
        L.or_pool_divergence.argtypes = [P, i32, i32, i32, i64, P, P]
        L.or_draft_sample.restype = None
        L.or_draft_sample.argtypes = [P, i64, i32, i64, P, i32, d, P, P, P, P]
        L.or_logits_threshold.restype = d
        L.or_logits_threshold.argtypes = [P, i64, d, i32, d, d, P]
        _ = u32
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


# ---------------------------------------------------------------- primitives
def lse(z) -> float:
    z = _f64(z)
    return lib().or_lse(_p(z), z.size)


def argmax(z) -> int:
    z = _f64(z)
    return int(lib().or_argmax(_p(z), z.size))


def dtv_logits(za, zb) -> float:
    za, zb = _f64(za), _f64(zb)
    return lib().or_dtv(_p(za), lse(za), _p(zb), lse(zb), za.size)


def kl_logits(za, zb) -> float:
    za, zb = _f64(za), _f64(zb)
    return lib().or_kl(_p(za), lse(za), _p(zb), lse(zb), za.size)


def _logp(p):
    p = _f64(p)
    with np.errstate(divide="ignore"):
        return np.log(p)


def dtv(p, q) -> float:
    """Eq. 5 on probability vectors (logits = log p, so softmax(log p) = p)."""
    return dtv_logits(_logp(p), _logp(q))


def kl(p, q) -> float:
    return kl_logits(_logp(p), _logp(q))


def accept(za_t, A, zb_t, B, u):
    tie = ctypes.c_int(0)
    r = lib().or_accept(float(za_t), float(A), float(zb_t), float(B), float(u), ctypes.byref(tie))
    return bool(r), bool(tie.value)


def sample(z, u):
    z = _f64(z)
    tie = ctypes.c_int(0)
    t = lib().or_sample(_p(z), lse(z), z.size, float(u), ctypes.byref(tie))
    return int(t), bool(tie.value)


def sample_residual_logits(za, zb, u):
    za, zb = _f64(za), _f64(zb)
    tie, small = ctypes.c_int(0), ctypes.c_int(0)
    t = lib().or_sample_residual(_p(za), lse(za), _p(zb), lse(zb), za.size, float(u),
                                 ctypes.byref(tie), ctypes.byref(small))
    return int(t), bool(tie.value), bool(small.value)


# ---------------------------------------------------------------- cascade
class _Level(ctypes.Structure):
    _fields_ = [("z", ctypes.c_void_p), ("ld", ctypes.c_int64),
                ("bstride", ctypes.c_int64), ("rows", ctypes.c_int32)]


def chain_verify(levels, cand0, u_acc=None, u_emit=None, *, m0=None, greedy=False,
                 intermediate_bonus=True, final_bonus=True, draft_fed=None,
                 tie_eps=1e-6, tie_eps_draw=None, nthreads=0):
    """Run the whole cascade for every request.

    levels: list of L arrays [B, rows_l, V] (any float dtype; converted exactly to f64).
    cand0:  [B, K] int32 candidates for the first verifier (the draft tokens).
    u_acc, u_emit: [L-1, B, W] float32 uniforms (W >= K+L-1), or None in greedy mode.
    Returns a dict of numpy arrays.
    """
    L = len(levels)
    zs = [_f64(z) for z in levels]
    B, K = cand0.shape
    V = zs[0].shape[2]
    cand0 = np.ascontiguousarray(cand0, dtype=np.int32)
    lv = (_Level * L)()
    for l, z in enumerate(zs):
        assert z.shape[0] == B and z.shape[2] == V
        lv[l].z = z.ctypes.data
        lv[l].ld = V
        lv[l].bstride = z.shape[1] * V
        lv[l].rows = z.shape[1]
    if greedy and u_acc is None:
        u_acc = np.zeros((L - 1, B, K + L - 1), np.float32)
        u_emit = u_acc
    u_acc = np.ascontiguousarray(u_acc, dtype=np.float32)
    u_emit = np.ascontiguousarray(u_emit, dtype=np.float32)
    W = u_acc.shape[2]
    out_ld = K + L - 1
    o = dict(
        n_acc=np.zeros((L - 1, B), np.int32), m_cand=np.zeros((L - 1, B), np.int32),
        out_tok=np.zeros((B, out_ld), np.int32), out_len=np.zeros(B, np.int32),
        rollback=np.zeros((L, B), np.int32), pos_dtv=np.zeros((L - 1, B, K)),
        pos_kl=np.zeros((L - 1, B, K)), near_tie=np.zeros(B, np.int32),
        flags=np.zeros(B, np.uint32))
    m0a = None if m0 is None else np.ascontiguousarray(m0, dtype=np.int32)
    rc = lib().or_chain_verify(
        lv, L, B, K, V, _p(cand0), _p(m0a), _p(u_acc), _p(u_emit), B * W, W,
        int(greedy), int(intermediate_bonus), int(final_bonus),
        int(K - 1 if draft_fed is None else draft_fed), float(tie_eps),
        float(tie_eps if tie_eps_draw is None else tie_eps_draw),
        _p(o["n_acc"]), _p(o["m_cand"]), _p(o["out_tok"]), out_ld, _p(o["out_len"]),
        _p(o["rollback"]), _p(o["pos_dtv"]), _p(o["pos_kl"]), _p(o["near_tie"]),
        _p(o["flags"]), int(nthreads))
    if rc != 0:
        raise ValueError("or_chain_verify: bad arguments")
    return o


# ---------------------------------------------------------------- rollback
def rollback_mask(mask, L_phys, r):
    mask = np.ascontiguousarray(mask, dtype=np.uint8).copy()
    B, cap = mask.shape
    Lp = ctypes.c_int32(int(L_phys))
    r = np.ascontiguousarray(r, dtype=np.int32)
    flags = np.zeros(B, np.uint32)
    lib().or_rollback_mask(_p(mask), B, cap, ctypes.byref(Lp), _p(r), _p(flags))
    return mask, int(Lp.value), flags


def rollback_paged(seq_len, block_table, block_size, free_ids, free_count, r,
                   cache_mask=None):
    seq_len = np.ascontiguousarray(seq_len, dtype=np.int32).copy()
    bt = np.ascontiguousarray(block_table, dtype=np.int32).copy()
    free_ids = np.ascontiguousarray(free_ids, dtype=np.int32).copy()
    fc = ctypes.c_int32(int(free_count))
    r = np.ascontiguousarray(r, dtype=np.int32)
    B, MB = bt.shape
    flags = np.zeros(B, np.uint32)
    cm = None if cache_mask is None else np.ascontiguousarray(cache_mask, dtype=np.uint8).copy()
    lib().or_rollback_paged(_p(seq_len), _p(bt), B, MB, int(block_size), _p(free_ids),
                            ctypes.byref(fc), free_ids.size, _p(cm),
                            0 if cm is None else cm.shape[1], _p(r), _p(flags))
    return dict(seq_len=seq_len, block_table=bt, free_ids=free_ids, free_count=int(fc.value),
                cache_mask=cm, flags=flags)


# ---------------------------------------------------------------- cost model
def expected_accepted(alpha, gamma):
    return lib().or_expected_accepted(float(alpha), int(gamma))


def theoretical_speedup(alpha, gamma, c):
    return lib().or_theoretical_speedup(float(alpha), int(gamma), float(c))


def ema(old, measured, weight, first=False):
    return lib().or_ema(float(old), float(measured), float(weight), int(first))


def predict_chain_latency(T, alpha, W, verify_linear=False, intermediate_bonus=True):
    T = _f64(T)
    a = _f64(alpha if len(alpha) else [0.0])
    return lib().or_predict_chain_latency(T.size, _p(T), _p(a), int(W), int(verify_linear),
                                          int(intermediate_bonus))


def select_chain(T, sim, W, max_len=4, verify_linear=False, intermediate_bonus=True):
    T = _f64(T)
    sim = _f64(sim)
    P = T.size
    out = np.zeros(32, np.int32)
    te = ctypes.c_double(0)
    n = lib().or_select_chain(P, _p(T), _p(sim), int(W), int(max_len), int(verify_linear),
                              int(intermediate_bonus), _p(out), ctypes.byref(te))
    return [int(x) for x in out[:n]], te.value


def pool_divergence(levels):
    """SimScore bootstrap divergences: levels = N arrays [B][K][V] (pool models'
    logits at the same K positions, bf16 values as float) -> (dtv, kl), each
    [N(N-1)/2][B][K] float64, pairs (i < j) in lexicographic order, KL(p_j || p_i)."""
    zs = [_f64(z) for z in levels]
    N = len(zs)
    B, K, V = zs[0].shape
    arr = (_Level * N)(*[_Level(z.ctypes.data, z.shape[2], z.shape[1] * z.shape[2], z.shape[1]) for z in zs])
    npair = N * (N - 1) // 2
    dtv = np.zeros((npair, B, K)); kl = np.zeros((npair, B, K))
    lib().or_pool_divergence(ctypes.addressof(arr), N, B, K, V, _p(dtv), _p(kl))
    return dtv, kl


def bootstrap_sim(levels):
    """Pairwise SimScore matrix [N][N] initialised from the bootstrap (every (i, j)
    SimScore with observation count 1): sim[i][j] = sim[j][i] = 1 - mean DTV over the
    positions; 1 on the diagonal."""
    dtv, _ = pool_divergence(levels)
    N = len(levels)
    sim = np.eye(N)
    pi = 0
    for i in range(N):
        for j in range(i + 1, N):
            sim[i, j] = sim[j, i] = 1.0 - float(dtv[pi].mean())
            pi += 1
    return sim


def draft_sample(z, u, greedy=False, tie_eps_draw=1e-7):
    """Draft-side sampling step: z [B][V] drafter logits,
    u [B] uniforms -> dict(token int32 [B], lse, q_tok float64 [B], near_tie int32 [B])."""
    z = _f64(z)
    B, V = z.shape
    u = np.ascontiguousarray(u, dtype=np.float32)
    out = dict(token=np.zeros(B, np.int32), lse=np.zeros(B), q_tok=np.zeros(B),
               near_tie=np.zeros(B, np.int32))
    lib().or_draft_sample(_p(z), V, B, V, _p(u), int(bool(greedy)), tie_eps_draw,
                          _p(out["token"]), _p(out["lse"]), _p(out["q_tok"]), _p(out["near_tie"]))
    return out


def logits_threshold(z, temperature=1.0, top_k=0, top_p=1.0, eps=1e-6):
    """top-k / top-p threshold of one logit row (R19 / R23):
    returns (tau, near): entries z < tau are removed (ties at tau kept); NaN for NaN / +inf rows."""
    z = _f64(z).ravel()
    near = np.zeros(1, np.int32)
    tau = lib().or_logits_threshold(_p(z), z.size, float(temperature), int(top_k), float(top_p),
                                    float(eps), _p(near))
    return float(tau), int(near[0])


def logits_process(z, temperature=1.0, top_k=0, top_p=1.0, eps=1e-6):
    """Row-wise top-k / top-p over z [..., V] (float64 copy): removed entries are -inf; rows with
    NaN / +inf are returned unchanged.  Returns (z_processed, tau [...], near [...])."""
    z = _f64(z)
    flat = z.reshape(-1, z.shape[-1])
    out = flat.copy()
    tau = np.zeros(flat.shape[0])
    near = np.zeros(flat.shape[0], np.int32)
    for r in range(flat.shape[0]):
        tau[r], near[r] = logits_threshold(flat[r], temperature, top_k, top_p, eps)
        if not np.isnan(tau[r]):
            out[r][flat[r] < tau[r]] = -np.inf
    return out.reshape(z.shape), tau.reshape(z.shape[:-1]), near.reshape(z.shape[:-1])
