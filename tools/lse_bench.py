"""Core kernel time with the cross-CTA exchange (msd_chain_verify) vs with producer-supplied row
normalisers (msd_chain_verify_lse), same inputs; msd_prof CUDA events around msd_core."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2505_07680_b200 import api, synth  # noqa: E402

names = [a for a in sys.argv[1:] if not a[0].isdigit() and a[0] != "-"] or ["llama3", "qwen25", "sweep"]
pats = [tuple(int(x) for x in a.split(",")) for a in sys.argv[1:] if a[0].isdigit() or a[0] == "-"] or [(-1, -1, -1)]
for name in names:
    c = synth.CONFIGS[name]
    inp = synth.gauss_chain(c["B"], c["V"], c["K"], c["L"], c["sigmas"], s=c["s"], seed=c["seed"], device="cuda",
                            dtype=c["dtype"])
    lse = torch.stack([torch.logsumexp(t[:, :inp.K, :inp.V].float(), dim=-1).double() for t in inp.levels]).contiguous()
    byts = sum(t.shape[0] * c["K"] * c["V"] * t.element_size() for t in inp.levels)
    for (label, kw), pat in [(x, q) for x in (("exchange", {}), ("lse-fed", {"lse": lse})) for q in pats]:
        api.debug_knobs(pat_t=pat[0], pat_r=pat[1], stages=pat[2])
        cv = api.ChainVerify(inp.levels, inp.draft, inp.u_acc, inp.u_emit, V=inp.V, **kw)
        for _ in range(3):
            cv()
        torch.cuda.synchronize()
        api.prof_read()
        api.prof_enable(True)
        ev = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev[0].record()
        for _ in range(10):
            cv()
        ev[1].record()
        torch.cuda.synchronize()
        ms, n, _ = api.prof_read()
        api.prof_enable(False)
        core = ms / n
        api.debug_knobs()
        print(f"{name} {label} pattern {pat}: core {core:.3f} ms = {byts / core / 1e6:.0f} GB/s; verify (core + tail) "
              f"{ev[0].elapsed_time(ev[1]) / 10:.3f} ms", flush=True)
