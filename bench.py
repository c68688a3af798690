#!/usr/bin/env python
"""Benchmark: one step = one pass of the whole hot path
over a batch of synthetic requests shaped like the paper's model chains:

  msd_chain_verify (softmax normalisers, acceptance, first rejection, residual/bonus
  draws, DTV/KL per position and per-pair stats, commit + per-model rollback lengths)
  -> msd_kv_rollback (paged KV of every model in the chain)
  -> per-pair int64 stats all-reduce across ranks (NCCL, N > 1; on a side stream that
     overlaps the rollback)
  -> host scheduler feed (EMA SimScore -> alpha -> Eq. 7 -> Alg. 1), one step stale.

In the adaptive sweep config (a 4-model pool) the chain Alg. 1 selects at step j is the
chain step j+1 verifies, so the loop of P:197 / Alg. 1 is closed; the line reports the
chain-selection frequencies and per-chain step times.

Usage: python bench.py [--gpus N] [--steps K] [--warmup W] [--config llama3] [--batch B]
       python bench.py --impl reference ...     (the float64 CPU oracle arm)
Multi-GPU: `python bench.py --gpus N` spawns N ranks itself (NCCL, 127.0.0.1); under
torchrun it uses the launcher's ranks.  Default: strong scaling (the config's global batch
split over the ranks); --scaling weak gives every rank the full batch.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2505_07680_b200 import synth  # noqa: E402

METRIC = "verified draft positions/sec and achieved HBM GB/s vs peak at 1/2/4/8 B200"
L2_BYTES = 126 * 2 ** 20          # B200 L2
FLUSH_BYTES = 512 * 2 ** 20       # 512 MB scratch write between steps


def _peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


def _dist(backend="nccl"):
    from paper_2505_07680_b200 import dist as mdist
    return mdist.init_from_env(backend)


class ClockSampler:
    """nvidia-smi sampling of SM clock and throttle reasons during the timed region."""

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.idx), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx.append(float(f[1]))
            except ValueError:
                continue
            for n, v in zip(names, f[3:7]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def cpu_oracle_positions_per_s(inp, sample_B, nthreads):
    """Time the float64 oracle (as it stands) on the first sample_B requests."""
    import oracle
    sel = slice(0, sample_B)
    levels = [t[sel, :, :inp.V].float().cpu().numpy() for t in inp.levels]
    draft = inp.draft[sel].cpu().numpy()
    ua = inp.u_acc[:, sel].cpu().numpy()
    ue = inp.u_emit[:, sel].cpu().numpy()
    t0 = time.perf_counter()
    oracle.chain_verify(levels, draft, ua, ue, nthreads=nthreads)
    dt = time.perf_counter() - t0
    return sample_B * inp.K / dt, dt


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def run_reference(args):
    ws, rank, local = _dist("gloo")
    if rank != 0:
        return
    cfg = synth.CONFIGS[args.config]
    cores = host_cores()
    # bounded sample of the same workload: a few requests per step (~seconds per step)
    inp = synth.gauss_chain(args.ref_sample, cfg["V"], cfg["K"], cfg["L"], cfg["sigmas"], s=cfg["s"],
                            seed=cfg["seed"], device="cpu", dtype=cfg["dtype"])
    for _ in range(args.warmup):
        cpu_oracle_positions_per_s(inp, min(2, args.ref_sample), cores)
    times = []
    for _ in range(args.steps):
        _, dt = cpu_oracle_positions_per_s(inp, args.ref_sample, cores)
        times.append(dt)
    per_step = sum(times) / len(times)
    val = args.ref_sample * cfg["K"] / per_step
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": "positions/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": per_step * 1e3, "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": args.config, "sample_requests": args.ref_sample, "V": cfg["V"],
                   "K": cfg["K"], "L": cfg["L"], "logits": cfg["dtype"]},
        "cpu_baseline": {"value": val, "unit": "positions/s", "cores": cores, "kind": "oracle",
                         "sample": f"first {args.ref_sample} requests of the {args.config} workload per step"},
        "e2e": {"value": val, "unit": "positions/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


class Chains:
    """The chain(s) a step may verify.  Fixed configs: the whole chain [0 .. L-1].  The adaptive
    sweep: every capability-ordered sub-chain of the pool ending at the target, built lazily --
    levels are the pool models' logits (model m holds K + m rows >= the rows its position in any
    sub-chain needs), draft tokens drawn from the chain's first model, uniforms the first
    n-1 levels of the pool's."""

    def __init__(self, api, inp, kv, cfg, req0, adaptive):
        self.api, self.inp, self.kv, self.cfg, self.req0 = api, inp, kv, cfg, req0
        self.adaptive = adaptive
        self.cache = {}
        self.drafts = {0: inp.draft}

    def get(self, chain):
        chain = tuple(chain)
        if chain not in self.cache:
            api, inp = self.api, self.inp
            n, K = len(chain), inp.K
            if chain[0] not in self.drafts:
                self.drafts[chain[0]] = synth.draft_tokens(inp.levels[chain[0]], K, inp.V, seed=self.cfg["seed"],
                                                           req0=self.req0, salt=chain[0])
            ua = inp.u_acc[:n - 1, :, :K + n - 1].contiguous()
            ue = inp.u_emit[:n - 1, :, :K + n - 1].contiguous()
            cv = api.ChainVerify([inp.levels[m] for m in chain], self.drafts[chain[0]], ua, ue, V=inp.V)
            rb = api.KVRollback([self.kv[m] for m in chain], cv.rollback, cv.flags)
            self.cache[chain] = (cv, rb)
        return self.cache[chain]


def run_ours(args):
    from paper_2505_07680_b200 import api
    from paper_2505_07680_b200 import dist as mdist

    ws, rank, local = _dist()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    cfg = dict(synth.CONFIGS[args.config])
    if args.batch:
        cfg["B"] = args.batch
    req0, B = mdist.shard(cfg["B"], ws, rank, args.scaling)
    L, K, V = cfg["L"], cfg["K"], cfg["V"]
    B_global = cfg["B"] if args.scaling == "strong" else cfg["B"] * ws
    esize = 2 if cfg["dtype"] == "bf16" else 4
    adaptive = args.config == "sweep"

    if B > 0:
        inp = synth.gauss_chain(B, V, K, L, cfg["sigmas"], s=cfg["s"], seed=cfg["seed"], req0=req0,
                                device=dev, dtype=cfg["dtype"])
        kv = synth.paged_kv(B, L, seed=cfg["seed"] + 1000 + req0, block_size=16, min_len=512,
                            max_len=4096, extra=K + L, device=dev)
    chains = Chains(api, inp, kv, cfg, req0, adaptive) if B > 0 else None
    # pristine KV metadata -> one multi-tensor copy resets every model per step
    flat_live = [t for d in kv for t in (d["seq_len"], d["block_table"], d["free_ids"], d["free_count"])] \
        if B > 0 else []
    pristine = [t.clone() for t in flat_live]

    def reset_kv():
        if flat_live:
            torch._foreach_copy_(flat_live, pristine)

    T_ms = [1.0, 3.0, 10.0, 40.0][-L:]   # synthetic per-token times (invented)
    sched = mdist.ChainScheduler(T_ms=T_ms, W=K)
    # SimScore bootstrap over every pool pair at "prefill", outside the
    # timed step: one msd_pool_divergence launch over the draft rows, stats all-reduced
    bootstrap_ms = 0.0
    npairs = L * (L - 1) // 2
    pool_stats = torch.zeros((npairs, 8), dtype=torch.int64, device=dev)
    if B > 0:
        api.pool_divergence(inp.levels, K=K, V=V, stats=False)     # module load (not timed)
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record()
        pool = api.pool_divergence(inp.levels, K=K, V=V)
        ev1.record()
        torch.cuda.synchronize()
        bootstrap_ms = ev0.elapsed_time(ev1)
        pool_stats.copy_(pool["stats"])
        del pool
    mdist.allreduce_stats(pool_stats)
    sched.bootstrap(pool_stats.cpu().tolist())
    fixed_chain = list(range(L))

    side = torch.cuda.Stream(device=dev)
    nslot = 3
    pinned = [torch.zeros((L - 1, 8), dtype=torch.int64).pin_memory() for _ in range(nslot)]
    stat_ev = [torch.cuda.Event() for _ in range(nslot)]
    ran = [None] * nslot                     # chain verified in the step that filled a slot
    stats_dev = torch.zeros((L - 1, 8), dtype=torch.int64, device=dev)
    cur = {"chain": fixed_chain}
    freq = {}

    def host_scheduler(j):
        # consume the all-reduced stats of step j-2 (complete by now): EMA SimScore -> Alg. 1
        if j < 2:
            return
        slot = (j - 2) % nslot
        stat_ev[slot].synchronize()
        ch = ran[slot]
        sched.update(pinned[slot][:len(ch) - 1].tolist(), chain=ch)
        if adaptive:
            cur["chain"] = list(sched.chain)

    def step(j, ph=None):
        chain = cur["chain"] if adaptive else fixed_chain
        n = len(chain)
        slot = j % nslot
        main = torch.cuda.current_stream()
        reset_kv()
        if n >= 2 and B > 0:
            cv, rb = chains.get(chain)
            cv.stats.zero_()
            if ph: ph[0].record()
            cv()
            if ph: ph[1].record()
            stats_dev.zero_()
            stats_dev[:n - 1].copy_(cv.stats)
        else:                                # [M_t] alone (or an idle rank): nothing to verify
            stats_dev.zero_()
            rb = None
            if ph: ph[0].record(); ph[1].record()
        # stats all-reduce on a side stream, overlapping the KV rollback on the main stream
        done = torch.cuda.Event()
        if ws > 1:
            side.wait_stream(main)
            with torch.cuda.stream(side):
                mdist.allreduce_stats(stats_dev)
                pinned[slot].copy_(stats_dev, non_blocking=True)
                done.record(side)
        if rb is not None:
            rb()
        if ph: ph[2].record()
        if ws > 1:
            main.wait_event(done)
        else:
            pinned[slot].copy_(stats_dev, non_blocking=True)
        if ph: ph[3].record()
        stat_ev[slot].record()
        ran[slot] = list(chain)
        freq[tuple(chain)] = freq.get(tuple(chain), 0) + 1
        host_scheduler(j)
        return chain

    for j in range(args.warmup):
        step(j)
    torch.cuda.synchronize()
    if ws > 1:
        torch.distributed.barrier()

    # L2: inputs smaller than 4x L2 are flushed between steps by a 512 MB scratch write
    # (outside the per-step events); larger inputs stream from HBM anyway
    in_bytes = inp.logit_bytes() if B > 0 else 0
    flush = torch.empty(FLUSH_BYTES // 4, dtype=torch.float32, device=dev) if in_bytes < 4 * L2_BYTES else None
    freq.clear()
    api.prof_read()
    api.prof_enable(True)
    sampler = ClockSampler(local) if rank == 0 else None
    if sampler:
        sampler.start()
        time.sleep(0.3)
    if ws > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    # CUDA graphs (one rank, fixed chain): each timed step's device work -- KV reset, stats reset,
    # msd_chain_verify (core + tail), rollback -- is one graph replay, so the host's per-call
    # overhead leaves no gaps between the kernels.  One graph per timed step: each holds its own
    # msd_prof event pair around msd_core, so the core's launch duration is still measured with
    # CUDA events on its stream in every timed step (and the launch count is the captured one).
    graphs, graph_note = None, "off"
    if args.graph and ws == 1 and B > 0 and not adaptive:
        cvg, rbg = chains.get(fixed_chain)

        def dev_step():
            reset_kv()
            cvg.stats.zero_()
            cvg()
            stats_dev.zero_()
            stats_dev[:L - 1].copy_(cvg.stats)
            rbg()
        try:
            side_w = torch.cuda.Stream(device=dev)
            side_w.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(side_w):
                dev_step()
            torch.cuda.current_stream().wait_stream(side_w)
            torch.cuda.synchronize()
            api.prof_read()            # drop the warm-up call's events and launch count
            graphs = []
            for _ in range(args.steps):
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g):
                    dev_step()
                graphs.append(g)
            torch.cuda.synchronize()
            graph_note = "one CUDA graph replay per timed step"
        except Exception as exc:      # capture unsupported: time the eager steps instead
            graphs, graph_note = None, f"eager (capture failed: {type(exc).__name__}: {exc})"[:200]
            torch.cuda.synchronize()
            api.prof_read()

    def graph_step(j):
        graphs[j].replay()
        slot = (args.warmup + j) % nslot
        pinned[slot].copy_(stats_dev, non_blocking=True)
        stat_ev[slot].record()
        ran[slot] = list(fixed_chain)
        freq[tuple(fixed_chain)] = freq.get(tuple(fixed_chain), 0) + 1
        host_scheduler(args.warmup + j)
        return fixed_chain

    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    chain_of = []
    for j in range(args.steps):
        if flush is not None:
            flush.fill_(float(j))
        evs[j][0].record()
        chain_of.append(tuple(graph_step(j) if graphs is not None else step(args.warmup + j)))
        evs[j][1].record()
    torch.cuda.synchronize()
    if ws > 1:
        torch.distributed.barrier()
    clocks = sampler.stop() if sampler else None
    api.prof_enable(False)
    core_ms, core_n, launches = api.prof_read()
    step_ms = [a.elapsed_time(b) for a, b in evs]
    ms = sum(step_ms) / args.steps
    t = torch.tensor([ms, core_ms / max(core_n, 1)], dtype=torch.float64, device=dev)
    if ws > 1:
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    ms, core_avg_ms = float(t[0]), float(t[1])

    # per-chain step times and selection frequencies (adaptive sweep)
    per_chain = {}
    for ch, sm in zip(chain_of, step_ms):
        per_chain.setdefault("-".join(map(str, ch)), []).append(sm)
    chain_report = {k: {"steps": len(v), "ms_per_step": statistics.median(v)} for k, v in per_chain.items()}

    # phases (separate instrumented steps, medians): verify (core + tail), rollback, all-reduce
    phases = None
    if B > 0:
        np_ = 5
        phase_ev = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(np_)]
        api.prof_enable(True)
        for j in range(np_):
            if flush is not None:
                flush.fill_(float(j))
            step(args.warmup + args.steps + j, phase_ev[j])
        torch.cuda.synchronize()
        api.prof_enable(False)
        pcore, pn, _ = api.prof_read()
        ver = statistics.median(p[0].elapsed_time(p[1]) for p in phase_ev)
        phases = {"verify_ms": ver, "core_ms": pcore / max(pn, 1), "tail_ms": ver - pcore / max(pn, 1),
                  "rollback_ms": statistics.median(p[1].elapsed_time(p[2]) for p in phase_ev),
                  "allreduce_wait_ms": statistics.median(p[2].elapsed_time(p[3]) for p in phase_ev)}

    # last timed step's stats: near ties and exact draws (counted and reported, north star)
    flags = chains.get(chain_of[-1])[0].flags.cpu() if (B > 0 and len(chain_of[-1]) > 1) else torch.zeros(1, dtype=torch.int32)
    st_last = chains.get(chain_of[-1])[0].stats.cpu() if (B > 0 and len(chain_of[-1]) > 1) else torch.zeros((1, 8), dtype=torch.int64)
    cnt = torch.tensor([int(st_last[:, 5].sum()), int(st_last[:, 6].sum()),
                        int(((flags & api.FLAG["TIMEOUT"]) != 0).sum())], dtype=torch.int64, device=dev)
    if ws > 1:
        torch.distributed.all_reduce(cnt)
    near_ties, exact_draws, n_timeout = (int(x) for x in cnt.tolist())

    # verified positions: B_global * K per step that ran a chain of >= 2 levels ([M_t] alone
    # verifies nothing)
    verified_steps = sum(1 for ch in chain_of if len(ch) >= 2)
    positions = B_global * K
    value = positions * verified_steps / args.steps / (ms * 1e-3)
    # algorithmic bytes per core launch: every draft-position row of the chain read once
    run_L = [len(ch) for ch in chain_of if len(ch) >= 2]
    core_bytes = int(statistics.mean(run_L) * V * esize * B * K) if run_L else 0
    peaks = _peaks()
    peak = peaks.get("hbm_gbs", 6650.0)
    achieved = core_bytes / (core_avg_ms * 1e-3) / 1e9 if core_avg_ms > 0 else 0.0
    traffic = None
    try:
        prof = json.load(open(os.path.join(ROOT, "profiles", "core_traffic.json")))
        traffic = prof.get(args.config, {}).get("dram_bytes_per_launch")
    except Exception:
        pass

    # ---------------- e2e through the public API with host buffers (fixed chain)
    e2e = None
    if args.e2e_steps > 0 and B > 0:
        cv, rb = chains.get(fixed_chain)
        h_levels = [t.cpu().pin_memory() for t in inp.levels]
        h_draft = inp.draft.cpu().pin_memory()
        h_ua, h_ue = inp.u_acc.cpu().pin_memory(), inp.u_emit.cpu().pin_memory()
        h_out = {k: torch.empty_like(v, device="cpu").pin_memory()
                 for k, v in (("commit_tok", cv.commit_tok), ("commit_len", cv.commit_len),
                              ("stats", cv.stats), ("flags", cv.flags))}
        h2d = sum(t.numel() * t.element_size() for t in h_levels + [h_draft, h_ua, h_ue])
        d2h = sum(t.numel() * t.element_size() for t in h_out.values())

        def e2e_step():
            for d_, h_ in zip(inp.levels, h_levels):
                d_.copy_(h_, non_blocking=True)
            inp.draft.copy_(h_draft, non_blocking=True)
            inp.u_acc.copy_(h_ua, non_blocking=True)
            inp.u_emit.copy_(h_ue, non_blocking=True)
            reset_kv()
            cv.stats.zero_()
            cv()
            rb()
            mdist.allreduce_stats(cv.stats)
            h_out["commit_tok"].copy_(cv.commit_tok, non_blocking=True)
            h_out["commit_len"].copy_(cv.commit_len, non_blocking=True)
            h_out["stats"].copy_(cv.stats, non_blocking=True)
            h_out["flags"].copy_(cv.flags, non_blocking=True)

        e2e_step()
        torch.cuda.synchronize()
        if ws > 1:
            torch.distributed.barrier()
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record()
        for _ in range(args.e2e_steps):
            e2e_step()
        a1.record()
        torch.cuda.synchronize()
        ems = a0.elapsed_time(a1) / args.e2e_steps
        te = torch.tensor([ems], dtype=torch.float64, device=dev)
        if ws > 1:
            torch.distributed.all_reduce(te, op=torch.distributed.ReduceOp.MAX)
        e2e = {"value": positions / (float(te[0]) * 1e-3), "unit": "positions/s",
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "ms_per_step": float(te[0])}

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline and B > 0:
        cores = host_cores()
        _, dt1 = cpu_oracle_positions_per_s(inp, 4, cores)
        sample = max(4, min(B, int(4 * args.cpu_seconds / max(dt1, 1e-3))))
        val, dt = cpu_oracle_positions_per_s(inp, sample, cores)
        _, dt1s = cpu_oracle_positions_per_s(inp, 1, 1)
        sample1 = max(1, min(B, int(args.cpu_seconds / 2 / max(dt1s, 1e-3))))
        val1, dts = cpu_oracle_positions_per_s(inp, sample1, 1)
        cpu = {"value": val, "unit": "positions/s", "cores": cores, "kind": "oracle",
               "sample": f"first {sample} of {B} requests of the {args.config} workload ({dt:.1f} s)",
               "single_thread": {"value": val1, "cores": 1,
                                 "sample": f"first {sample1} requests ({dts:.1f} s)"}}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "positions/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": args.config, "global_batch": B_global, "batch_per_gpu": B, "V": V,
                       "K": K, "L": L, "logits": cfg["dtype"], "sigmas": list(cfg["sigmas"]),
                       "parallelism": f"dp{ws} (requests sharded, {args.scaling} scaling)",
                       "l2": (f"inputs {in_bytes / 1e9:.3f} GB/GPU < 4x L2: 512 MB scratch write between steps"
                              if flush is not None else f"inputs {in_bytes / 1e9:.2f} GB/GPU > 4x 126 MB L2 (no flush)"),
                       "kv": "paged, 16-token blocks, seq_len U[512,4096], reset each step",
                       "launch": graph_note},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "kernel": "msd_core",
                         "frac_of_nominal_8tbs": achieved / 8000.0,
                         "algorithmic_bytes_per_launch": core_bytes,
                         "core_ms_per_launch": core_avg_ms,
                         "core_share_of_step": core_avg_ms / ms,
                         "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy)" if "hbm_gbs" in peaks
                         else "fallback 6650 GB/s (B200_PROFILING.md)"},
            "phases": phases,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": int(launches),
            "clocks": clocks,
            "near_ties": near_ties, "exact_draws": exact_draws,
            "scheduler": {"chain": sched.chain, "simscore": sched.sim, "t_eff_ms": sched.t_eff,
                          "bootstrap_ms": bootstrap_ms, "adaptive": adaptive,
                          "chains_run": chain_report},
            "timeouts": n_timeout,
        }
        print(json.dumps(line), flush=True)
    if ws > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _spawned(rank, args, port):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), WORLD_SIZE=str(args.gpus),
                      RANK=str(rank), LOCAL_RANK=str(rank))
    run_ours(args)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="llama3", choices=sorted(synth.CONFIGS))
    ap.add_argument("--batch", type=int, default=0, help="override the config's global batch")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"])
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-sample", type=int, default=16)
    ap.add_argument("--no-graph", dest="graph", action="store_false",
                    help="time eager steps instead of one CUDA graph replay per step")
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    if args.impl == "reference":
        run_reference(args)
    elif args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        n = torch.cuda.device_count()
        if n < args.gpus:
            sys.exit(f"bench.py --gpus {args.gpus}: only {n} CUDA device(s) visible")
        import torch.multiprocessing as mp
        mp.spawn(_spawned, args=(args, _free_port()), nprocs=args.gpus, join=True)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
