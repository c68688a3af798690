"""Time msd_chain_verify (core + tail) for several core item patterns / ring depths.
usage: python tools/core_sweep.py [config] "T,R,S;T,R,S;..."  (S = MSD_STAGES, -1 = default)"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2505_07680_b200 import api, synth
name = sys.argv[1] if len(sys.argv) > 1 else "llama3"
combos = [tuple(int(x) for x in s.split(",")) for s in (sys.argv[2] if len(sys.argv) > 2 else "5,0,-1;5,4,-1").split(";")]
c = synth.CONFIGS[name]
inp = synth.gauss_chain(c["B"], c["V"], c["K"], c["L"], c["sigmas"], s=c["s"], seed=c["seed"], device="cuda", dtype=c["dtype"])
cv = api.ChainVerify(inp.levels, inp.draft, inp.u_acc, inp.u_emit, V=c["V"])
byts = sum(t.shape[0] * c["K"] * c["V"] * t.element_size() for t in inp.levels)
lib = api.lib()
ref = None
for T, R, S in combos:
    os.environ["MSD_PAT_T"], os.environ["MSD_PAT_R"] = str(T), str(R)
    if S > 0: os.environ["MSD_STAGES"] = str(S)
    else: os.environ.pop("MSD_STAGES", None)
    for _ in range(3): cv()
    api.prof_enable(True) if hasattr(api, "prof_enable") else None
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): cv()
    e1.record(); torch.cuda.synchronize()
    core = None
    if hasattr(api, "prof_read"):
        core = api.prof_read()
        api.prof_enable(False)
    ms = e0.elapsed_time(e1) / 10
    cv(); torch.cuda.synchronize()
    fl = int((cv.flags & api.FLAG["TIMEOUT"]).sum().item())
    d, tok = cv.pos_dtv.clone(), cv.commit_tok.clone()
    if ref is None: ref = (d, tok)
    dd = (d - ref[0]).abs().max().item(); nt = int((tok != ref[1]).any(1).sum().item())
    cms = core[0] / max(1, core[1]) if core else float("nan")
    print(f"T={T} R={R} S={S}: step {ms:.3f} ms  core {cms:.3f} ms ({byts/cms/1e6:.0f} GB/s)  timeouts {fl}  "
          f"max|dtv-ref| {dd:.2e}  token rows differing {nt}", flush=True)
