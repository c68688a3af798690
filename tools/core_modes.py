"""Time the core kernel in its debug isolation modes (MSD_CORE_DBG bit flags):
0 normal; any nonzero = pass-1 warps only (no exchange, no slot waits); 2 no exp,
4 no TMEM store, 8 TMA ring only, 16 no KL.  Prints ms per launch and GB/s of logit bytes."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2505_07680_b200 import api, synth
name = sys.argv[1] if len(sys.argv) > 1 else "llama3"
modes = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [0, 1, 2, 3]
c = synth.CONFIGS[name]
inp = synth.gauss_chain(c["B"], c["V"], c["K"], c["L"], c["sigmas"], s=c["s"], seed=c["seed"], device="cuda", dtype=c["dtype"])
cv = api.ChainVerify(inp.levels, inp.draft, inp.u_acc, inp.u_emit, V=c["V"])
nbytes = c["B"] * c["K"] * c["L"] * c["V"] * inp.levels[0].element_size()
for m in modes:
    os.environ["MSD_CORE_DBG"] = str(m)
    for _ in range(3):
        cv()
    torch.cuda.synchronize()
    api.prof_enable(True)
    for _ in range(10):
        cv()
    torch.cuda.synchronize()
    ms, n, _ = api.prof_read()
    api.prof_enable(False)
    print(f"mode {m}: core {ms / max(n, 1):.3f} ms  {nbytes / (ms / max(n, 1)) / 1e6:.0f} GB/s")
os.environ["MSD_CORE_DBG"] = "0"
