"""Cycle profile of the core kernel's warp roles (build variant libmsd_prof.so, -DMSD_PROF).

Prints, per role, the average SM cycles per item spent in each phase (summed over warps of
the role, divided by the items those warps processed), plus the kernel time.
usage: MSD_LIB=libmsd_prof.so python tools/core_prof.py [config] [pat_t,pat_r,stages]"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2505_07680_b200 import api, synth
name = sys.argv[1] if len(sys.argv) > 1 else "llama3"
c = synth.CONFIGS[name]
pat = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "-1,-1,-1").split(",")]
api.debug_knobs(pat_t=pat[0], pat_r=pat[1], stages=pat[2])
inp = synth.gauss_chain(c["B"], c["V"], c["K"], c["L"], c["sigmas"], s=c["s"], seed=c["seed"], device="cuda", dtype=c["dtype"])
cv = api.ChainVerify(inp.levels, inp.draft, inp.u_acc, inp.u_emit, V=c["V"])
lib = api.lib(); lib.msd_debug_set_trace.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
n_items = c["B"] * c["K"] * 64
buf = torch.zeros(n_items * 16, dtype=torch.int64, device="cuda")
roles = {0: ("pass1", ["full", "slots", "run", "folds+release", "r1", "tm+arrive"]),
         1: ("pass2", ["rowf", "data", "compute", "fold", "r2+store"]),
         2: ("publisher", ["r1 wait", "stores", "loads", "redux+exp", "shuffles"]),
         3: ("fetcher", ["poll", "combine", "rowfE wait", "rowf", "(between)"]),
         4: ("reducer", ["r2 wait", "work"]),
         5: ("producer", ["empty wait", "issue"])}
cv(); torch.cuda.synchronize()
lib.msd_debug_set_trace(buf.data_ptr(), buf.numel() * 8)
buf.zero_()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); cv(); e1.record(); torch.cuda.synchronize()
lib.msd_debug_set_trace(None, 0)
a = buf[:96].view(6, 16).cpu().double()
print(f"{name}: step (core+tail, profiled) {e0.elapsed_time(e1):.3f} ms  pattern {pat}")
for r, (rn, ph) in roles.items():
    n = a[r, 15].item()
    if n == 0:
        continue
    v = a[r, :len(ph)] / n
    print(f"  {rn:9s} items {int(n):7d}  " + "  ".join(f"{p} {x:.0f}" for p, x in zip(ph, v.tolist())) + f"  | total {v.sum():.0f} cyc/item")

# per-CTA view: the CTAs whose pass-1 warps waited least for slots pace their group
G = 148
pc = buf[128:128 + G * 8 * 16].view(G, 8, 16).cpu().double()
n1 = pc[:, 0, 15].clamp(min=1)
slots = pc[:, 0, 1] / n1
full = pc[:, 0, 0] / n1
order = torch.argsort(slots)
print("per-CTA pass-1 cycles/item (fewest slot waits first):")
for g in order[:6].tolist() + order[-3:].tolist():
    v = pc[g, 0, :6] / n1[g]
    w = pc[g, 1, :5] / pc[g, 1, 15].clamp(min=1)
    print(f"  cta {g:3d}: p1 " + " ".join(f"{x:.0f}" for x in v.tolist()) + " | p2 " + " ".join(f"{x:.0f}" for x in w.tolist()))
