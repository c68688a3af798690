"""Time the core kernel alone (msd_prof events) in its debug isolation modes (msd_debug_set_knobs
core_dbg bits: 0 = normal, 1 = pass 1 + TMA ring only, 5 = TMA ring only, 2 = R items skip the
recomputation).  usage: python tools/core_dbg.py [config] [modes, e.g. 0,1] [pat_t,pat_r,stages]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2505_07680_b200 import api, synth
name = sys.argv[1] if len(sys.argv) > 1 else "llama3"
modes = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "0,1").split(",")]
pat = [int(x) for x in (sys.argv[3] if len(sys.argv) > 3 else "-1,-1,-1").split(",")]
c = synth.CONFIGS[name]
inp = synth.gauss_chain(c["B"], c["V"], c["K"], c["L"], c["sigmas"], s=c["s"], seed=c["seed"], device="cuda", dtype=c["dtype"])
cv = api.ChainVerify(inp.levels, inp.draft, inp.u_acc, inp.u_emit, V=c["V"])
byts = sum(t.shape[0] * c["K"] * c["V"] * t.element_size() for t in inp.levels)
for m in modes:
    api.debug_knobs(pat_t=pat[0], pat_r=pat[1], stages=pat[2], core_dbg=m)
    for _ in range(3): cv()
    torch.cuda.synchronize()
    api.prof_enable(True)
    for _ in range(10): cv()
    torch.cuda.synchronize()
    ms, n, _ = api.prof_read()
    api.prof_enable(False)
    print(f"mode {m} pattern {pat}: core {ms / n:.3f} ms  {byts / (ms / n) / 1e6:.0f} GB/s", flush=True)
api.debug_knobs()
