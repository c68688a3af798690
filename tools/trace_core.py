"""Run a workload once with the core-kernel stage trace and summarise latencies."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2505_07680_b200 import api, synth
name = sys.argv[1] if len(sys.argv) > 1 else "llama3"
c = synth.CONFIGS[name]
inp = synth.gauss_chain(c["B"], c["V"], c["K"], c["L"], c["sigmas"], s=c["s"], seed=c["seed"], device="cuda", dtype=c["dtype"])
cv = api.ChainVerify(inp.levels, inp.draft, inp.u_acc, inp.u_emit, V=c["V"])
C = (c["V"] + 4095) // 4096
n_items = c["B"] * c["K"] * C
buf = torch.zeros(n_items * 8, dtype=torch.int64, device="cuda")
lib = api.lib(); lib.msd_debug_set_trace.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
cv(); torch.cuda.synchronize()
lib.msd_debug_set_trace(buf.data_ptr(), buf.numel() * 8)
cv(); torch.cuda.synchronize()
lib.msd_debug_set_trace(None, 0)
t = buf.view(n_items, 8).cpu().numpy().astype(np.float64)
t0 = t[t > 0].min()
t = np.where(t > 0, t - t0, np.nan) / 1e3   # us
names = ["tma_issue", "p1_start", "p1_end", "published", "cnt_seen", "rowf_ready", "p2_start", "p2_end"]
print("kernel span us", np.nanmax(t))
for a, b in [(0, 1), (1, 2), (2, 3), (3, 4), (4, 5), (5, 6), (6, 7), (2, 6)]:
    d = t[:, b] - t[:, a]
    print(f"{names[a]:>10} -> {names[b]:<10} median {np.nanmedian(d):8.2f}  p90 {np.nanpercentile(d, 90):8.2f}  max {np.nanmax(d):8.2f}")
G = 148
p1 = t[:, 1]
cta = np.arange(n_items) % G
for g in (0, 1, 77, 147):
    s = p1[cta == g]
    print("cta", g, "items", s.size, "p1-start spacing median", np.nanmedian(np.diff(s)), "first", np.round(s[:6], 2))
U = n_items // C
pub = t[:, 3].reshape(U, C)
print("unit publish spread (max-min) median", np.nanmedian(np.nanmax(pub, 1) - np.nanmin(pub, 1)),
      "p90", np.nanpercentile(np.nanmax(pub, 1) - np.nanmin(pub, 1), 90))
lastpub = np.repeat(np.nanmax(pub, 1), C)
print("cnt_seen - last publish median", np.nanmedian(t[:, 4] - lastpub), "p90", np.nanpercentile(t[:, 4] - lastpub, 90))
print("p1_start(j) spacing global median (all ctas)", np.nanmedian(np.diff(np.sort(p1))))
