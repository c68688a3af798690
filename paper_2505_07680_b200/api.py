"""ctypes binding of libmsd (include/msd.h) -- argument marshalling only.

Every function here forwards torch tensors' device pointers and the current CUDA
stream to the C ABI; all arithmetic of the method runs in libmsd's kernels (or, for
the scheduler feed, in libmsd's host C code).  There is no fallback: if libmsd.so
is missing or the device is not a B200, calls raise ``MsdError``.
"""
from __future__ import annotations

import ctypes
import os
from typing import List, Optional, Sequence

import torch

from .synth import level_rows  # noqa: F401  (re-exported for callers)

_HERE = os.path.dirname(os.path.abspath(__file__))
# MSD_LIB selects an alternative in-tree build (A/B experiments: tools/, never the default)
LIB_PATH = os.path.join(_HERE, os.environ.get("MSD_LIB", "libmsd.so"))

MSD_STOCHASTIC, MSD_GREEDY = 0, 1
MSD_F32, MSD_BF16 = 0, 1
FLAG = dict(NONFINITE=1, TOKEN_OOB=2, RESID_SMALL=4, ROLLBACK_OVF=8, FREELIST_OVF=16,
            KL_INF=32, NEAR_TIE=64, EXACT_DRAW=128, TIMEOUT=256)
DTV_SCALE = 4294967296.0
KL_SCALE = 268435456.0


class MsdError(RuntimeError):
    pass


class msd_logits(ctypes.Structure):
    _fields_ = [("ptr", ctypes.c_void_p), ("dtype", ctypes.c_int32), ("rows", ctypes.c_int32),
                ("ld", ctypes.c_int64), ("batch_stride", ctypes.c_int64)]


class msd_pair_stats(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int64) for n in (
        "dtv_fx", "kl_fx", "positions", "proposed", "accepted", "near_ties", "exact_draws", "kl_inf")]


STATS_FIELDS = [f[0] for f in msd_pair_stats._fields_]


class msd_processors(ctypes.Structure):
    _fields_ = [("temperature", ctypes.c_float), ("top_k", ctypes.c_int32), ("top_p", ctypes.c_float)]


class msd_paged_kv(ctypes.Structure):
    _fields_ = [("seq_len", ctypes.c_void_p), ("block_table", ctypes.c_void_p),
                ("max_blocks", ctypes.c_int32), ("block_size", ctypes.c_int32),
                ("free_ids", ctypes.c_void_p), ("free_count", ctypes.c_void_p),
                ("free_cap", ctypes.c_int32), ("mask_ld", ctypes.c_int32),
                ("cache_mask", ctypes.c_void_p)]


_lib = None


def lib() -> ctypes.CDLL:
    """Load libmsd.so (fails loudly: there is no CPU / eager fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise MsdError(f"{LIB_PATH} is missing; run `python -c 'import __graft_entry__ as g; g.build()'`")
    L = ctypes.CDLL(LIB_PATH)
    P, i32, i64, sz, d = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_size_t, ctypes.c_double
    L.msd_chain_verify.restype = i32
    L.msd_chain_verify.argtypes = [P, i32, i32, i32, i64, P, P, P, i32, i32, i32,
                                   P, P, P, P, P, P, P, P, P, P, sz, P]
    L.msd_chain_verify_proc.restype = i32
    L.msd_chain_verify_proc.argtypes = [P, i32, i32, i32, i64, P, P, P, i32, i32, i32,
                                        P, P, P, P, P, P, P, P, P, P, sz, P, P]
    L.msd_chain_verify_lse.restype = i32
    L.msd_chain_verify_lse.argtypes = [P, i32, i32, i32, i64, P, P, P, i32, i32, i32,
                                       P, P, P, P, P, P, P, P, P, P, sz, P, P]
    L.msd_verify_level.restype = i32
    L.msd_verify_level.argtypes = [msd_logits, msd_logits, i32, i32, i64, P, P, P, P, i32, i32,
                                   P, P, P, P, P, P, P, P, sz, P]
    L.msd_chain_verify_workspace.restype = sz
    L.msd_chain_verify_workspace.argtypes = [i32, i32, i32, i64]
    L.msd_verify_level_workspace.restype = sz
    L.msd_verify_level_workspace.argtypes = [i32, i32, i64]
    L.msd_kv_rollback.restype = i32
    L.msd_kv_rollback.argtypes = [P, i32, i32, P, P, P]
    L.msd_pool_divergence.restype = i32
    L.msd_pool_divergence.argtypes = [P, i32, i32, i32, i64, P, P, P, P, P]
    L.msd_draft_sample.restype = i32
    L.msd_draft_sample.argtypes = [P, i32, i32, i64, P, i32, P, P, P, P, P]
    L.msd_logits_process.restype = i32
    L.msd_logits_process.argtypes = [P, P, i32, i32, i64, P, P, P, P]
    L.msd_predict_chain_latency.restype = i32
    L.msd_predict_chain_latency.argtypes = [i32, P, P, i32, i32, i32, P]
    L.msd_select_chain.restype = i32
    L.msd_select_chain.argtypes = [i32, P, P, i32, i32, i32, i32, P, P, P]
    L.msd_simscore_update.restype = d
    L.msd_simscore_update.argtypes = [d, P, d, i32]
    L.msd_last_error.restype = ctypes.c_char_p
    L.msd_last_error.argtypes = []
    L.msd_abi_version.restype = i32
    L.msd_init.restype = i32
    L.msd_init.argtypes = []
    L.msd_lmhead_workspace.restype = sz
    L.msd_lmhead_workspace.argtypes = [i32, i64]
    L.msd_lmhead_logits.restype = i32
    L.msd_lmhead_logits.argtypes = [P, P, i32, i32, i64, P, P, i64, P, P, P, sz, P]
    L.msd_lmhead_lse.restype = i32
    L.msd_lmhead_lse.argtypes = [P, P, i32, i32, i64, P, P, P, P, sz, P]
    L.msd_prof_enable.restype = i32
    L.msd_prof_enable.argtypes = [i32]
    L.msd_prof_read.restype = i32
    L.msd_prof_read.argtypes = [P, P, P]
    L.msd_debug_set_knobs.restype = i32
    L.msd_debug_set_knobs.argtypes = [i32, i32, i32, i32, i32, d]
    _lib = L
    return L


def _check(status: int, what: str):
    if status != 0:
        raise MsdError(f"{what}: status {status}: {lib().msd_last_error().decode()}")


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def logits_desc(t: torch.Tensor) -> msd_logits:
    """[B, rows, ld] tensor (vocab contiguous) -> msd_logits."""
    if t.dim() != 3 or t.stride(2) != 1:
        raise MsdError("logits must be [B, rows, ld] with a contiguous vocabulary dimension")
    dt = {torch.float32: MSD_F32, torch.bfloat16: MSD_BF16}.get(t.dtype)
    if dt is None:
        raise MsdError(f"unsupported logits dtype {t.dtype}")
    return msd_logits(t.data_ptr(), dt, t.shape[1], t.stride(1), t.stride(0))


def chain_workspace_bytes(L, B, K, V) -> int:
    return int(lib().msd_chain_verify_workspace(L, B, K, V))


def new_workspace(L, B, K, V, device="cuda") -> torch.Tensor:
    """Zero-filled workspace (the ABI requires zero on first use)."""
    n = chain_workspace_bytes(L, B, K, V)
    return torch.zeros(max(n, 256), dtype=torch.uint8, device=device)


def new_stats(L, device="cuda") -> torch.Tensor:
    return torch.zeros((L - 1, len(STATS_FIELDS)), dtype=torch.int64, device=device)


class ChainVerify:
    """Pre-marshalled msd_chain_verify call for fixed tensors (hot loops, benches).

    Outputs are allocated once; ``__call__`` re-issues the C call with the cached
    argument tuple on the current (or given) stream.
    """

    def __init__(self, levels: Sequence[torch.Tensor], draft: torch.Tensor, u_acc=None, u_emit=None,
                 *, V: Optional[int] = None, greedy=False, intermediate_bonus=True,
                 draft_fed: Optional[int] = None, pos_outputs=True, rollback=True, stats=True,
                 ws: Optional[torch.Tensor] = None, temperature: Optional[float] = None,
                 lse: Optional[torch.Tensor] = None):
        dev = draft.device
        _check(lib().msd_init(), "msd_init")   # one-time device setup, outside any graph capture
        self.L = len(levels)
        self.B, self.K = draft.shape
        self.V = levels[0].shape[2] if V is None else V
        L, B, K = self.L, self.B, self.K
        W = K + L - 1
        self.levels = list(levels)
        self.draft = draft
        self.u_acc, self.u_emit = u_acc, u_emit
        self._desc = (msd_logits * L)(*[logits_desc(t) for t in levels])
        i32 = torch.int32
        self.n_acc = torch.zeros((L - 1, B), dtype=i32, device=dev)
        self.m_cand = torch.zeros((L - 1, B), dtype=i32, device=dev)
        self.commit_tok = torch.zeros((B, W), dtype=i32, device=dev)
        self.commit_len = torch.zeros((B,), dtype=i32, device=dev)
        self.rollback = torch.zeros((L, B), dtype=i32, device=dev) if rollback else None
        self.pos_dtv = torch.zeros((L - 1, B, K), dtype=torch.float32, device=dev) if pos_outputs else None
        self.pos_kl = torch.zeros((L - 1, B, K), dtype=torch.float32, device=dev) if pos_outputs else None
        self.stats = new_stats(L, dev) if stats else None
        self.flags = torch.zeros((B,), dtype=torch.int32, device=dev)
        self.ws = ws if ws is not None else new_workspace(L, B, K, self.V, dev)
        self.mode = MSD_GREEDY if greedy else MSD_STOCHASTIC
        self.ib = 1 if intermediate_bonus else 0
        self.draft_fed = K - 1 if draft_fed is None else draft_fed
        self._args = [self._desc, L, B, K, self.V, _ptr(draft), _ptr(u_acc), _ptr(u_emit),
                      self.mode, self.ib, self.draft_fed, _ptr(self.n_acc), _ptr(self.m_cand),
                      _ptr(self.commit_tok), _ptr(self.commit_len), _ptr(self.rollback),
                      _ptr(self.pos_dtv), _ptr(self.pos_kl), _ptr(self.stats), _ptr(self.flags),
                      _ptr(self.ws), self.ws.numel()]
        if lse is not None:     # producer-supplied row normalisers (msd_chain_verify_lse), [L][B][K] f64
            if temperature is not None:
                raise MsdError("lse and temperature cannot be combined")
            if lse.dtype != torch.float64 or tuple(lse.shape) != (L, B, K) or not lse.is_contiguous():
                raise MsdError("lse must be a contiguous float64 [L][B][K] tensor")
            self.lse = lse
            self._args.append(_ptr(lse))
            self._fn = lib().msd_chain_verify_lse
        elif temperature is None:
            self._fn = lib().msd_chain_verify
        else:     # logits processor (msd_chain_verify_proc): softmax(z / T) at every level
            self._proc = msd_processors(float(temperature), 0, 1.0)
            self._args.append(ctypes.byref(self._proc))
            self._fn = lib().msd_chain_verify_proc

    def __call__(self, stream=None):
        _check(self._fn(*self._args, _stream(stream)), "msd_chain_verify")
        return self

    def outputs(self) -> dict:
        o = dict(n_acc=self.n_acc, m_cand=self.m_cand, commit_tok=self.commit_tok,
                 commit_len=self.commit_len, flags=self.flags)
        if self.rollback is not None:
            o["rollback"] = self.rollback
        if self.pos_dtv is not None:
            o["pos_dtv"], o["pos_kl"] = self.pos_dtv, self.pos_kl
        if self.stats is not None:
            o["stats"] = self.stats
        return o


def chain_verify(levels, draft, u_acc=None, u_emit=None, **kw) -> dict:
    """One-shot msd_chain_verify; returns the output tensors (on the device)."""
    cv = ChainVerify(levels, draft, u_acc, u_emit, **kw)
    cv()
    return cv.outputs()


def verify_level(q: torch.Tensor, p: torch.Tensor, cand: torch.Tensor, u_acc=None, u_emit=None, *,
                 m: Optional[torch.Tensor] = None, greedy=False, emit_bonus=True,
                 V: Optional[int] = None, ws=None, stats=None, stream=None) -> dict:
    B, K = cand.shape
    V = q.shape[2] if V is None else V
    dev = cand.device
    i32 = torch.int32
    out = dict(n_acc=torch.zeros(B, dtype=i32, device=dev),
               out_tok=torch.zeros((B, K + 1), dtype=i32, device=dev),
               out_len=torch.zeros(B, dtype=i32, device=dev),
               pos_dtv=torch.zeros((B, K), dtype=torch.float32, device=dev),
               pos_kl=torch.zeros((B, K), dtype=torch.float32, device=dev),
               flags=torch.zeros(B, dtype=i32, device=dev),
               stats=stats if stats is not None else new_stats(2, dev))
    if ws is None:
        ws = torch.zeros(max(int(lib().msd_verify_level_workspace(B, K, V)), 256), dtype=torch.uint8, device=dev)
    st = lib().msd_verify_level(logits_desc(q), logits_desc(p), B, K, V, _ptr(cand), _ptr(m),
                                _ptr(u_acc), _ptr(u_emit), MSD_GREEDY if greedy else MSD_STOCHASTIC,
                                1 if emit_bonus else 0, _ptr(out["n_acc"]), _ptr(out["out_tok"]),
                                _ptr(out["out_len"]), _ptr(out["pos_dtv"]), _ptr(out["pos_kl"]),
                                _ptr(out["stats"]), _ptr(out["flags"]), _ptr(ws), ws.numel(),
                                _stream(stream))
    _check(st, "msd_verify_level")
    return out


class KVRollback:
    """Pre-marshalled msd_kv_rollback for a list of per-model paged-KV tensor dicts
    (keys: seq_len, block_table, free_ids, free_count, block_size[, cache_mask])."""

    def __init__(self, kv: List[dict], rollback: torch.Tensor, flags: torch.Tensor):
        self.kv = kv
        arr = (msd_paged_kv * len(kv))()
        for i, d in enumerate(kv):
            cm = d.get("cache_mask")
            arr[i] = msd_paged_kv(d["seq_len"].data_ptr(), d["block_table"].data_ptr(),
                                  d["block_table"].shape[1], int(d["block_size"]),
                                  d["free_ids"].data_ptr(), d["free_count"].data_ptr(),
                                  d["free_ids"].numel(), 0 if cm is None else cm.shape[1],
                                  None if cm is None else cm.data_ptr())
        self._arr = arr
        self._args = [arr, len(kv), rollback.shape[1], _ptr(rollback), _ptr(flags)]
        self._fn = lib().msd_kv_rollback

    def __call__(self, stream=None):
        _check(self._fn(*self._args, _stream(stream)), "msd_kv_rollback")


def kv_rollback(kv: List[dict], rollback: torch.Tensor, flags: torch.Tensor, stream=None):
    KVRollback(kv, rollback, flags)(stream)


def pool_divergence(models: Sequence[torch.Tensor], K: Optional[int] = None, V: Optional[int] = None,
                    stats: bool = True, stream=None) -> dict:
    """msd_pool_divergence: SimScore bootstrap of an N-model pool.
    models: N tensors [B][rows >= K][ld] (same dtype); returns device tensors pos_dtv / pos_kl
    [N(N-1)/2, B, K] (pairs i < j in lexicographic order; KL(p_j || p_i)), stats
    [N(N-1)/2, 8] int64 and flags [B]."""
    N = len(models)
    B = models[0].shape[0]
    K = models[0].shape[1] if K is None else K
    V = models[0].shape[2] if V is None else V
    dev = models[0].device
    npair = N * (N - 1) // 2
    desc = (msd_logits * N)(*[logits_desc(t) for t in models])
    out = dict(pos_dtv=torch.zeros((npair, B, K), dtype=torch.float32, device=dev),
               pos_kl=torch.zeros((npair, B, K), dtype=torch.float32, device=dev),
               flags=torch.zeros((B,), dtype=torch.int32, device=dev))
    if stats:
        out["stats"] = torch.zeros((npair, len(STATS_FIELDS)), dtype=torch.int64, device=dev)
    st = lib().msd_pool_divergence(desc, N, B, K, V, _ptr(out["pos_dtv"]), _ptr(out["pos_kl"]),
                                   _ptr(out.get("stats")), _ptr(out["flags"]), _stream(stream))
    _check(st, "msd_pool_divergence")
    return out


def draft_sample(drafter: torch.Tensor, u: Optional[torch.Tensor], row: int = 0, V: Optional[int] = None,
                 greedy: bool = False, out: Optional[dict] = None, stream=None) -> dict:
    """msd_draft_sample: one draft-side sampling step.
    drafter: [B][rows][ld] logits (row `row` is sampled); u: [B] f32 uniforms (None if greedy).
    Returns device tensors token int32 [B], lse / q_tok f32 [B], flags [B] (`out` reuses them)."""
    B = drafter.shape[0]
    V = drafter.shape[2] if V is None else V
    dev = drafter.device
    if out is None:
        out = dict(token=torch.empty((B,), dtype=torch.int32, device=dev),
                   lse=torch.empty((B,), dtype=torch.float32, device=dev),
                   q_tok=torch.empty((B,), dtype=torch.float32, device=dev),
                   flags=torch.zeros((B,), dtype=torch.int32, device=dev))
    d = logits_desc(drafter)
    st = lib().msd_draft_sample(ctypes.byref(d), int(row), B, V, _ptr(u), int(bool(greedy)),
                                _ptr(out["token"]), _ptr(out["lse"]), _ptr(out["q_tok"]),
                                _ptr(out["flags"]), _stream(stream))
    _check(st, "msd_draft_sample")
    return out


def logits_process(logits: torch.Tensor, rows: Optional[int] = None, V: Optional[int] = None, *,
                   top_k: int = 0, top_p: float = 1.0, temperature: float = 1.0,
                   out: Optional[torch.Tensor] = None, tau: Optional[torch.Tensor] = None,
                   flags: Optional[torch.Tensor] = None, stream=None):
    """msd_logits_process: top-k / top-p over rows [0, rows) of logits [B][R][ld] (P:150,
    DESIGN.md R19 / R23).  Writes the processed rows (removed entries -inf) to `out` (a new
    tensor shaped like `logits` when None; `out=logits` processes in place).  Returns
    (out, tau [B][rows] f32, flags [B] int32)."""
    B, R = logits.shape[0], logits.shape[1]
    rows = R if rows is None else rows
    V = logits.shape[2] if V is None else V
    dev = logits.device
    if out is None:
        out = torch.empty_like(logits)
    if tau is None:
        tau = torch.empty((B, rows), dtype=torch.float32, device=dev)
    if flags is None:
        flags = torch.zeros((B,), dtype=torch.int32, device=dev)
    di, do = logits_desc(logits), logits_desc(out)
    pr = msd_processors(float(temperature), int(top_k), float(top_p))
    st = lib().msd_logits_process(ctypes.byref(di), ctypes.byref(do), B, int(rows), int(V), ctypes.byref(pr),
                                  _ptr(tau), _ptr(flags), _stream(stream))
    _check(st, "msd_logits_process")
    return out, tau, flags


# ------------------------------------------------------------------ scheduler feed (host C)
def _dbuf(xs):
    a = (ctypes.c_double * max(1, len(xs)))(*[float(x) for x in xs])
    return a


def predict_chain_latency(T, alpha, W, verify_cost=0, intermediate_bonus=True) -> float:
    out = ctypes.c_double(0)
    st = lib().msd_predict_chain_latency(len(T), _dbuf(T), _dbuf(alpha), int(W), int(verify_cost),
                                         int(bool(intermediate_bonus)), ctypes.byref(out))
    _check(st, "msd_predict_chain_latency")
    return out.value


def select_chain(T, sim, W, max_len=4, verify_cost=0, intermediate_bonus=True):
    P = len(T)
    flat = [float(sim[i][j]) for i in range(P) for j in range(P)]
    out = (ctypes.c_int32 * 32)()
    n = ctypes.c_int32(0)
    te = ctypes.c_double(0)
    st = lib().msd_select_chain(P, _dbuf(T), _dbuf(flat), int(W), int(max_len), int(verify_cost),
                                int(bool(intermediate_bonus)), out, ctypes.byref(n), ctypes.byref(te))
    _check(st, "msd_select_chain")
    return [int(out[i]) for i in range(n.value)], te.value


def simscore_update(sim: float, stats_row, weight: float, first: bool = False) -> float:
    s = msd_pair_stats(*[int(x) for x in stats_row])
    return float(lib().msd_simscore_update(float(sim), ctypes.byref(s), float(weight), int(first)))


def debug_knobs(pat_t=-1, pat_r=-1, stages=-1, core_dbg=0, exact_draws=False, z_safe=-1.0):
    """Test / diagnostic overrides of internal choices (msd_debug_set_knobs); call with no
    arguments to restore the release defaults."""
    _check(lib().msd_debug_set_knobs(int(pat_t), int(pat_r), int(stages), int(core_dbg),
                                     int(bool(exact_draws)), float(z_safe)), "msd_debug_set_knobs")


def lmhead_lse(H: torch.Tensor, W: torch.Tensor, cand: Optional[torch.Tensor] = None, stream=None) -> dict:
    """msd_lmhead_lse: row normalisers of H W^T (and the candidate logits) without writing the
    logits.  H [M, D] bf16, W [V, D] bf16 (contiguous)."""
    if H.dtype != torch.bfloat16 or W.dtype != torch.bfloat16 or not H.is_contiguous() or not W.is_contiguous():
        raise MsdError("H and W must be contiguous bf16")
    M, D = H.shape
    V = W.shape[0]
    dev = H.device
    lse = torch.empty(M, dtype=torch.float32, device=dev)
    zc = torch.empty(M, dtype=torch.float32, device=dev)
    ws = torch.empty(max(1, int(lib().msd_lmhead_workspace(M, V))), dtype=torch.uint8, device=dev)
    _check(lib().msd_lmhead_lse(H.data_ptr(), W.data_ptr(), M, D, V, _ptr(cand), lse.data_ptr(), zc.data_ptr(),
                                ws.data_ptr(), ws.numel(), _stream(stream)), "msd_lmhead_lse")
    return dict(lse=lse, z_cand=zc, ws=ws)


def lmhead_logits(H: torch.Tensor, W: torch.Tensor, cand: Optional[torch.Tensor] = None,
                  out: Optional[torch.Tensor] = None, lse64: Optional[torch.Tensor] = None, stream=None) -> dict:
    """msd_lmhead_logits: logits = H W^T written in bf16 (out: [M, ldz] view, new [M, V8] when None)
    plus the float64 normaliser of the written rows (the `lse` msd_chain_verify_lse consumes)."""
    if H.dtype != torch.bfloat16 or W.dtype != torch.bfloat16 or not H.is_contiguous() or not W.is_contiguous():
        raise MsdError("H and W must be contiguous bf16")
    M, D = H.shape
    V = W.shape[0]
    dev = H.device
    if out is None:
        out = torch.empty((M, (V + 7) // 8 * 8), dtype=torch.bfloat16, device=dev)
    if lse64 is None:
        lse64 = torch.empty(M, dtype=torch.float64, device=dev)
    zc = torch.empty(M, dtype=torch.float32, device=dev)
    ws = torch.empty(max(1, int(lib().msd_lmhead_workspace(M, V))), dtype=torch.uint8, device=dev)
    _check(lib().msd_lmhead_logits(H.data_ptr(), W.data_ptr(), M, D, V, _ptr(cand), out.data_ptr(), out.stride(0),
                                   lse64.data_ptr(), zc.data_ptr(), ws.data_ptr(), ws.numel(), _stream(stream)),
           "msd_lmhead_logits")
    return dict(logits=out, lse64=lse64, z_cand=zc, ws=ws)


def prof_enable(on=True):
    _check(lib().msd_prof_enable(1 if on else 0), "msd_prof_enable")


def prof_read():
    ms = ctypes.c_double(0)
    n = ctypes.c_int32(0)
    tot = ctypes.c_int32(0)
    _check(lib().msd_prof_read(ctypes.byref(ms), ctypes.byref(n), ctypes.byref(tot)), "msd_prof_read")
    return ms.value, n.value, tot.value
