"""Per-CTA pass-1 progress from the core trace: time of the last pass-1 end stamp per CTA
and the SM each CTA ran on is not visible, so report the spread and the slowest CTAs."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2505_07680_b200 import api, synth
name = sys.argv[1] if len(sys.argv) > 1 else "llama3"
c = synth.CONFIGS[name]
inp = synth.gauss_chain(c["B"], c["V"], c["K"], c["L"], c["sigmas"], s=c["s"], seed=c["seed"], device="cuda", dtype=c["dtype"])
cv = api.ChainVerify(inp.levels, inp.draft, inp.u_acc, inp.u_emit, V=c["V"])
lib = api.lib(); lib.msd_debug_set_trace.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
def geo(V, VS=4096, REF=148):
    cmin = (V + VS - 1) // VS; best = cmin; used = (REF // cmin) * cmin; cc = cmin + 1
    while cc <= cmin + cmin // 4 and cc <= REF and used < REF:
        u = (REF // cc) * cc
        if u > used: used = u; best = cc
        cc += 1
    return best
C = geo(c["V"]); U = c["B"] * c["K"]; n_items = U * C
kg = 148 // C
for rep in range(2):
    buf = torch.zeros(n_items * 16, dtype=torch.int64, device="cuda")
    cv(); torch.cuda.synchronize()
    lib.msd_debug_set_trace(buf.data_ptr(), buf.numel() * 8)
    cv(); torch.cuda.synchronize()
    lib.msd_debug_set_trace(None, 0)
    t = buf.view(n_items, 16).cpu().numpy().astype(np.float64)
    t0 = t[t > 0].min(); t = np.where(t > 0, t - t0, np.nan) / 1e3
    uu = np.arange(n_items) // C; ss = np.arange(n_items) % C
    cta = (uu % kg) * C + ss
    end = np.array([np.nanmax(t[cta == g, 3]) for g in range(kg * C)])
    mid = np.array([np.nanmedian(t[cta == g, 3][400:600]) if (cta == g).sum() > 600 else np.nan for g in range(kg * C)])
    print(f"rep {rep}: p1 end per CTA min {end.min():.1f} med {np.median(end):.1f} max {end.max():.1f} us")
    o = np.argsort(-end)
    print("  slowest:", [(int(g), round(float(end[g]), 1)) for g in o[:10]])
    print("  fastest:", [(int(g), round(float(end[g]), 1)) for g in o[-6:]])
    print("  item-500 time spread: min %.1f max %.1f" % (np.nanmin(mid), np.nanmax(mid)))
