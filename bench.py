#!/usr/bin/env python
"""Benchmark: one step = one pass of the whole hot path
over a batch of synthetic requests shaped like the paper's model chains:

  msd_chain_verify (softmax normalisers, acceptance, first rejection, residual/bonus
  draws, DTV/KL per position and per-pair stats, commit + per-model rollback lengths)
  -> msd_kv_rollback (paged KV of every model in the chain)
  -> per-pair int64 stats all-reduce across ranks (NCCL, N > 1)
  -> host scheduler feed (EMA SimScore -> alpha -> Eq. 7 -> Alg. 1), one step stale.

Usage: python bench.py [--gpus N] [--steps K] [--warmup W] [--config llama3]
       python bench.py --impl reference ...     (the float64 CPU oracle arm)
Multi-GPU: torchrun --nproc-per-node N bench.py --gpus N (requests sharded, weak scaling).
"""
from __future__ import annotations

import argparse
import json
import os
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


def build_workload(cfg_name, B, req0, device):
    c = synth.CONFIGS[cfg_name]
    inp = synth.gauss_chain(B, c["V"], c["K"], c["L"], c["sigmas"], s=c["s"], seed=c["seed"],
                            req0=req0, device=device, dtype=c["dtype"])
    # paged KV of every model in the chain, 16-token blocks, seq_len in U[512, 4096]
    # plus this cycle's speculative entries; one pristine copy for reset.
    kv = synth.paged_kv(B, c["L"], seed=c["seed"] + 1000 + req0, block_size=16, min_len=512,
                        max_len=4096, extra=c["K"] + c["L"], device=device)
    return c, inp, kv


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
    dev = "cpu"
    # bounded sample of the same workload: a few requests per step (calibrated to ~10 s/step)
    inp = synth.gauss_chain(args.ref_sample, cfg["V"], cfg["K"], cfg["L"], cfg["sigmas"], s=cfg["s"],
                            seed=cfg["seed"], device=dev, dtype=cfg["dtype"])
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
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": args.config, "sample_requests": args.ref_sample, "V": cfg["V"],
                   "K": cfg["K"], "L": cfg["L"], "logits": cfg["dtype"]},
        "cpu_baseline": {"value": val, "unit": "positions/s", "cores": cores, "kind": "oracle",
                         "sample": f"first {args.ref_sample} requests of the {args.config} workload per step"},
        "e2e": {"value": val, "unit": "positions/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_ours(args):
    from paper_2505_07680_b200 import api
    from paper_2505_07680_b200 import dist as mdist

    ws, rank, local = _dist()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    cfg = synth.CONFIGS[args.config]
    req0, B = mdist.shard(cfg["B"], ws, rank, args.scaling)
    c, inp, kv = build_workload(args.config, B, req0, dev)
    L, K, V = c["L"], c["K"], c["V"]
    esize = 2 if c["dtype"] == "bf16" else 4

    cv = api.ChainVerify(inp.levels, inp.draft, inp.u_acc, inp.u_emit, V=V)
    rb = api.KVRollback(kv, cv.rollback, cv.flags)
    # pristine KV metadata in one flat buffer -> one device copy resets all models per step
    flat_live = [t for d in kv for t in (d["seq_len"], d["block_table"], d["free_ids"], d["free_count"])]
    pristine = [t.clone() for t in flat_live]

    def reset_kv():
        torch._foreach_copy_(flat_live, pristine)

    pinned_stats = [torch.zeros_like(cv.stats, device="cpu").pin_memory() for _ in range(3)]
    stat_ev = [torch.cuda.Event() for _ in range(3)]
    T_ms = [1.0, 3.0, 10.0, 40.0][-L:]   # synthetic per-token times (invented)
    sched = mdist.ChainScheduler(T_ms=T_ms, W=K)
    # SimScore bootstrap over every pool pair at "prefill", outside the
    # timed step: one msd_pool_divergence launch over the draft rows, stats all-reduced
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    api.pool_divergence(inp.levels, K=K, V=V, stats=False)     # module load (not timed)
    ev0.record()
    pool = api.pool_divergence(inp.levels, K=K, V=V)
    ev1.record()
    mdist.allreduce_stats(pool["stats"])
    torch.cuda.synchronize()
    bootstrap_ms = ev0.elapsed_time(ev1)
    sched.bootstrap(pool["stats"].cpu().tolist())
    del pool

    def host_scheduler(j):
        # consume the (all-reduced) stats of step j-2, complete by now: EMA SimScore -> Alg. 1
        if j < 2:
            return
        slot = (j - 2) % 3
        stat_ev[slot].synchronize()
        sched.update(pinned_stats[slot].tolist(), chain=list(range(L)))   # the chain that ran

    def step(j):
        reset_kv()
        cv.stats.zero_()
        cv()
        rb()
        mdist.allreduce_stats(cv.stats)
        slot = j % 3
        pinned_stats[slot].copy_(cv.stats, non_blocking=True)
        stat_ev[slot].record()
        host_scheduler(j)

    for j in range(args.warmup):
        step(j)
    torch.cuda.synchronize()
    if ws > 1:
        torch.distributed.barrier()
    api.prof_read()
    api.prof_enable(True)
    sampler = ClockSampler(local) if rank == 0 else None
    if sampler:
        sampler.start()
        time.sleep(0.3)
    if ws > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for j in range(args.steps):
        step(args.warmup + j)
    e1.record()
    torch.cuda.synchronize()
    if ws > 1:
        torch.distributed.barrier()
    clocks = sampler.stop() if sampler else None
    api.prof_enable(False)
    core_ms, core_n, launches = api.prof_read()
    ms = e0.elapsed_time(e1) / args.steps
    t = torch.tensor([ms, core_ms / max(core_n, 1)], dtype=torch.float64, device=dev)
    if ws > 1:
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    ms, core_avg_ms = float(t[0]), float(t[1])

    flags = cv.flags.cpu()
    n_timeout = int(((flags & api.FLAG["TIMEOUT"]) != 0).sum())
    positions = B * K * ws
    value = positions / (ms * 1e-3)
    core_bytes = L * V * esize * B * K               # every draft-position row read once
    peaks = _peaks()
    peak = peaks.get("hbm_gbs", 6650.0)
    achieved = core_bytes / (core_avg_ms * 1e-3) / 1e9
    traffic = None
    try:
        prof = json.load(open(os.path.join(ROOT, "profiles", "core_traffic.json")))
        traffic = prof.get(args.config, {}).get("dram_bytes_per_launch")
    except Exception:
        pass

    # ---------------- e2e through the public API with host buffers
    e2e = None
    if args.e2e_steps > 0:
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
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        cores = host_cores()
        _, dt1 = cpu_oracle_positions_per_s(inp, 4, cores)
        sample = max(4, min(B, int(4 * args.cpu_seconds / max(dt1, 1e-3))))
        val, dt = cpu_oracle_positions_per_s(inp, sample, cores)
        cpu = {"value": val, "unit": "positions/s", "cores": cores, "kind": "oracle",
               "sample": f"first {sample} of {B} requests of the {args.config} workload ({dt:.1f} s)"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "positions/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": args.config, "global_batch": B * ws if args.scaling == "weak" else cfg["B"],
                       "batch_per_gpu": B, "V": V, "K": K, "L": L, "logits": c["dtype"],
                       "sigmas": list(c["sigmas"]), "parallelism": f"dp{ws} (requests sharded)",
                       "l2": f"inputs {inp.logit_bytes() / 1e9:.2f} GB/GPU >> 126 MB L2 (no flush)",
                       "kv": "paged, 16-token blocks, seq_len U[512,4096], reset each step"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "kernel": "msd_core",
                         "algorithmic_bytes_per_launch": core_bytes,
                         "core_ms_per_launch": core_avg_ms,
                         "core_share_of_step": core_avg_ms / ms,
                         "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy)" if "hbm_gbs" in peaks
                         else "fallback 6650 GB/s (B200_PROFILING.md)"},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": int(launches),
            "clocks": clocks,
            "scheduler": {"chain": sched.chain, "simscore": sched.sim, "t_eff_ms": sched.t_eff,
                          "bootstrap_ms": bootstrap_ms},
            "timeouts": n_timeout,
        }
        print(json.dumps(line), flush=True)
    if ws > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="llama3", choices=sorted(synth.CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"])
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-sample", type=int, default=16)
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
