"""Cycle profile of the tail kernel's phases (libmsd_prof.so, -DMSD_PROF): thread 0 of every
CTA, summed; printed per request.  usage: MSD_LIB=libmsd_prof.so python tools/tail_prof.py [config]"""
import ctypes, os, sys
os.environ.setdefault("MSD_LIB", "libmsd_prof.so")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2505_07680_b200 import api, synth
name = sys.argv[1] if len(sys.argv) > 1 else "llama3"
c = synth.CONFIGS[name]
inp = synth.gauss_chain(c["B"], c["V"], c["K"], c["L"], c["sigmas"], s=c["s"], seed=c["seed"], device="cuda", dtype=c["dtype"])
cv = api.ChainVerify(inp.levels, inp.draft, inp.u_acc, inp.u_emit, V=c["V"])
lib = api.lib()
buf = (ctypes.c_ulonglong * 16)()
cv(); torch.cuda.synchronize()
lib.msd_debug_tail_prof(buf, 1)
req0 = (ctypes.c_ulonglong * (4096 * 16))()
lib.msd_debug_tail_req(req0)
cv(); torch.cuda.synchronize()
lib.msd_debug_tail_prof(buf, 1)
names = ["combine rows", "extra rows", "acceptance", "dtv/kl", "emission(rest)", "next cands", "outputs", "emit: weights", "emit: draw_slices"]
B = c["B"]
print(f"{name}: tail cycles per request (thread 0): " + "  ".join(f"{n} {buf[k] / B:.0f}" for k, n in enumerate(names)))
print(f"fast-path slice scans {buf[15]}, of which undecided (float64 rescan) {buf[14]}; cycles per scan: loads+weights {buf[9] / max(buf[15], 1):.0f} scan_find {buf[10] / max(buf[15], 1):.0f} decision {buf[11] / max(buf[15], 1):.0f}")
fl = cv.flags.cpu()
print("requests with EXACT_DRAW:", int(((fl & api.FLAG['EXACT_DRAW']) != 0).sum()), " RESID_SMALL:", int(((fl & api.FLAG['RESID_SMALL']) != 0).sum()))
print("n_acc mean per level:", cv.n_acc.float().mean(1).tolist(), " m_cand mean:", cv.m_cand.float().mean(1).tolist())

import numpy as np
cta = (ctypes.c_ulonglong * (4096 * 2))()
lib.msd_debug_tail_cta(cta)
a = np.frombuffer(cta, dtype=np.uint64).reshape(4096, 2)[:B].astype(np.float64)
t0 = a[:, 0].min()
st, en = (a[:, 0] - t0) / 1e3, (a[:, 1] - t0) / 1e3
dur = en - st
print(f"tail span {en.max():.1f} us; per-request duration us: p50 {np.percentile(dur, 50):.1f} p90 {np.percentile(dur, 90):.1f} max {dur.max():.1f}")
print(f"start times: p50 {np.percentile(st, 50):.1f} max {st.max():.1f}")
na = cv.n_acc.cpu().numpy(); mc = cv.m_cand.cpu().numpy()
order = np.argsort(-dur)[:10]
for r in order:
    print(f"  req {r}: start {st[r]:.1f} dur {dur[r]:.1f}  n_acc {na[:, r].tolist()} m_cand {mc[:, r].tolist()} flags {int(fl[r])}")

req1 = (ctypes.c_ulonglong * (4096 * 16))()
lib.msd_debug_tail_req(req1)
rq = (np.frombuffer(req1, dtype=np.uint64).astype(np.float64) - np.frombuffer(req0, dtype=np.uint64).astype(np.float64)).reshape(4096, 16)[:B]
for r in order[:3]:
    t11, t9, t10 = rq[r, 11], rq[r, 9], rq[r, 10]
    if t11 > 0:
        print(f"  req {r} exact draw: normalisers {t9 - t11:.0f} cycles, weights {t10 - t9:.0f}")
    print(f"  req {r} phases (cycles): " + "  ".join(f"{n} {rq[r, k]:.0f}" for k, n in enumerate(names)))
med = np.argsort(dur)[B // 2]
print(f"  median req {med} phases (cycles): " + "  ".join(f"{n} {rq[med, k]:.0f}" for k, n in enumerate(names)))

# per-phase cycles (thread 0) of the slowest requests
rq = np.frombuffer(req0, dtype=np.uint64).reshape(4096, 16)[:B].astype(np.float64)
print("phases of the slowest requests (cycles):", names)
for r in order[:5]:
    print(f"  req {r}: " + " ".join(f"{rq[r, k]:.0f}" for k in range(len(names))))
print("median request:", " ".join(f"{np.median(rq[:, k]):.0f}" for k in range(len(names))))
ex = [r for r in range(B) if int(fl[r]) & api.FLAG['EXACT_DRAW']]
for r in ex[:4]:
    print(f"  exact-draw req {r}: normalisers {rq[r, 9] - rq[r, 11]:.0f} cycles, slice masses {rq[r, 10] - rq[r, 9]:.0f} cycles")
print("prologue split (median cycles): prefetch+gathers", f"{np.median(rq[:, 12]):.0f}", " row combines", f"{np.median(rq[:, 13]):.0f}", " rest of 'combine rows'", f"{np.median(rq[:, 0]):.0f}")
