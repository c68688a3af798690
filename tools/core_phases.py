"""Pass-1 phase cycle profile (MSD_CORE_DBG bit 64): average SM cycles per item spent by a
pass-1 warp in each phase.  argv: config, extra dbg flags (e.g. 0 for the normal pipeline)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2505_07680_b200 import api, synth
name = sys.argv[1] if len(sys.argv) > 1 else "llama3"
c = synth.CONFIGS[name]
inp = synth.gauss_chain(c["B"], c["V"], c["K"], c["L"], c["sigmas"], s=c["s"], seed=c["seed"], device="cuda", dtype=c["dtype"])
cv = api.ChainVerify(inp.levels, inp.draft, inp.u_acc, inp.u_emit, V=c["V"])
lib = api.lib(); lib.msd_debug_set_trace.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
n_items = c["B"] * c["K"] * 64
names = ["full wait", "load+max+rel", "slot wait", "exp loop", "folds", "r1 wait+st", "tm wait+sync"]
for flags in [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "0,1,23").split(",")]:
    buf = torch.zeros(n_items * 16, dtype=torch.int64, device="cuda")
    os.environ["MSD_CORE_DBG"] = str(64 | flags)
    cv(); torch.cuda.synchronize(); buf.zero_()
    lib.msd_debug_set_trace(buf.data_ptr(), buf.numel() * 8)
    cv(); torch.cuda.synchronize()
    lib.msd_debug_set_trace(None, 0)
    a = buf[:64].view(8, 8).cpu().double()
    per = a[:, :7].sum(0) / a[:, 7].sum()
    print(f"flags {flags}: " + "  ".join(f"{n} {v:.0f}" for n, v in zip(names, per.tolist())) + f"  total {per.sum():.0f}")
os.environ["MSD_CORE_DBG"] = "0"
