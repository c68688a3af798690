"""Run a workload once with the core-kernel stage trace (16 stamps / item) and summarise."""
import ctypes, os, sys
os.environ.setdefault("MSD_LIB", "libmsd_trace.so")   # stamps are compiled in with -DMSD_TRACE only
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2505_07680_b200 import api, synth
name = sys.argv[1] if len(sys.argv) > 1 and not sys.argv[1].startswith("-") else "llama3"
c = synth.CONFIGS[name]
inp = synth.gauss_chain(c["B"], c["V"], c["K"], c["L"], c["sigmas"], s=c["s"], seed=c["seed"], device="cuda", dtype=c["dtype"])
kw = {}
if "--lse" in sys.argv:   # producer-supplied normalisers (msd_chain_verify_lse): no exchange
    kw["lse"] = torch.stack([torch.logsumexp(t[:, :c["K"], :c["V"]].float(), dim=-1).double() for t in inp.levels]).contiguous()
cv = api.ChainVerify(inp.levels, inp.draft, inp.u_acc, inp.u_emit, V=c["V"], **kw)
def geo(V, VS=4096, REF=148):
    """core slices per unit: ceil(C / 2) CTAs for the tail's C slices (msd_common.cuh)"""
    used = lambda cc: (REF // ((cc + 1) // 2)) * ((cc + 1) // 2)
    cmin = (V + VS - 1) // VS; best = cmin; u0 = used(cmin)
    for cc in range(cmin + 1, cmin + cmin // 4 + 1):
        if used(cc) > u0 or (used(cc) == u0 and best % 2 and not cc % 2): u0 = used(cc); best = cc
    return (best + 1) // 2 if c["dtype"] == "bf16" else best
C = geo(c["V"])
n_items = c["B"] * c["K"] * C
buf = torch.zeros(n_items * 2 * 16 + 16, dtype=torch.int64, device="cuda")   # >= units x tail slices
lib = api.lib(); lib.msd_debug_set_trace.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
cv(); torch.cuda.synchronize()
lib.msd_debug_set_trace(buf.data_ptr(), buf.numel() * 8)
cv(); torch.cuda.synchronize()
lib.msd_debug_set_trace(None, 0)
t = buf[:n_items * 16].view(n_items, 16).cpu().numpy().astype(np.float64)
t0 = t[t > 0].min()
t = np.where(t > 0, t - t0, np.nan) / 1e3   # us
N = ["tma", "p1.full", "p1.tmE", "p1.end", "f.loads", "pub.done", "f.start", "p1.last", "pub.wake", "pub.calc",
     "f.done", "p2.rowf", "p2.tmF", "p2.end", "red.r2", "red.end"]
print("kernel span us %.1f" % np.nanmax(t))
def d(a, b):
    x = t[:, b] - t[:, a]
    return f"{N[a]:>8} -> {N[b]:<8} med {np.nanmedian(x):7.2f} p90 {np.nanpercentile(x, 90):7.2f}"
for a, b in [(0, 1), (1, 2), (2, 3), (3, 7), (7, 8), (8, 9), (9, 5), (3, 5), (6, 4), (4, 10), (10, 12), (3, 12), (12, 13), (13, 15), (5, 4)]:
    print(d(a, b))
U = n_items // C
pub = t[:, 5].reshape(U, C)
last = np.repeat(np.nanmax(pub, 1), C)
print("last publish -> records seen  med %.2f p90 %.2f" % (np.nanmedian(t[:, 4] - last), np.nanpercentile(t[:, 4] - last, 90)))
print("unit publish spread med %.2f" % np.nanmedian(np.nanmax(pub, 1) - np.nanmin(pub, 1)))
G = (148 // C) * C
kg = G // C
uu = np.arange(n_items) // C
ss = np.arange(n_items) % C
cta = (uu % kg) * C + ss
for g in (0, 100):
    sel = cta == g
    for k in (1, 3, 5, 10, 13):
        print(f"cta {g} {N[k]:>8} spacing med {np.nanmedian(np.diff(t[sel, k])):6.2f}", end=";")
    print()
# who is last in each unit: distribution of CTA index of the last publisher
lastc = np.nanargmax(pub, 1)
print("C", C, "groups", kg)
# per-CTA start / end (first TMA issue, last stamp of any kind)
first = np.array([np.nanmin(t[cta == g, 0]) for g in range(G)])
lastx = np.array([np.nanmax(t[cta == g]) for g in range(G)])
print("CTA first-issue us: min %.1f med %.1f max %.1f" % (first.min(), np.median(first), first.max()))
print("CTA last-stamp  us: min %.1f med %.1f max %.1f" % (lastx.min(), np.median(lastx), lastx.max()))
print("slowest CTAs:", np.argsort(-lastx)[:8].tolist(), "earliest-finishing:", np.argsort(lastx)[:8].tolist())
# --- who publishes last, and why: per unit, the last publisher's phase times vs the others'
last_c = np.nanargmax(pub, 1)
T = t.reshape(U, C, 16)
uu = np.arange(U)
lastT = T[uu, last_c]                       # (U, 16) stamps of the last publisher
def med(x): return np.nanmedian(x)
print("last publisher: slot wait (p1.full->p1.tmE) med %.2f, p1 compute (tmE->end) %.2f, tma->full %.2f, end->pub %.2f"
      % (med(lastT[:, 2] - lastT[:, 1]), med(lastT[:, 3] - lastT[:, 2]), med(lastT[:, 1] - lastT[:, 0]), med(lastT[:, 5] - lastT[:, 3])))
print("all CTAs:       slot wait med %.2f, p1 compute %.2f, tma->full %.2f, end->pub %.2f"
      % (med(T[:, :, 2] - T[:, :, 1]), med(T[:, :, 3] - T[:, :, 2]), med(T[:, :, 1] - T[:, :, 0]), med(T[:, :, 5] - T[:, :, 3])))
# is the last publisher of unit u also late on u-k?  (persistence of slowness)
lc = last_c.reshape(-1)
for lag in (kg, 2 * kg, 4 * kg):
    same = np.mean(lc[lag:] == lc[:-lag])
    print(f"P(last publisher of unit u == of unit u-{lag}) = {same:.2f}  (chance {1 / C:.3f})")
print("last-publisher slice histogram (top):", np.bincount(lc, minlength=C).argsort()[::-1][:8].tolist())
# --- timeline of the most frequent last publisher (per group) vs a typical CTA
cta_of_last = (uu % kg) * C + lc
for g in range(min(kg, 2)):
    sel_units = (uu % kg) == g
    vals, cnts = np.unique(cta_of_last[sel_units], return_counts=True)
    straggler = int(vals[np.argmax(cnts)])
    for name, cta_id in (("straggler", straggler), ("typical", g * C + (straggler % C + 7) % C)):
        Tc = t[cta == cta_id]
        seg = lambda a, b: np.nanmedian(Tc[:, b] - Tc[:, a])
        gap = np.nanmedian(np.diff(Tc[:, 1]))
        print(f"group {g} {name:9s} cta {cta_id:3d}: period {gap:.2f}  tma->full {seg(0,1):.2f} slot {seg(1,2):.2f} "
              f"p1 {seg(2,3):.2f} end->pub {seg(3,5):.2f} pub->seen {seg(5,4):.2f} combine {seg(4,10):.2f} "
              f"->p2 {seg(10,12):.2f} p2 {seg(12,13):.2f} | p1.end->p2 {seg(3,12):.2f}")
