"""Print GPU-vs-oracle differences for one config (debug aid; test infrastructure)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2505_07680_b200 import api, synth
from tests._parity import run_oracle, to_np, compare

name = sys.argv[1] if len(sys.argv) > 1 else "sweep"
B = int(sys.argv[2]) if len(sys.argv) > 2 else 8
if name.startswith("ragged"):
    V = int(name[6:])
    inp = synth.gauss_chain(B, V, 3, 3, (0.9, 0.4, 0.0), seed=11, device="cuda", dtype="bf16", ld=(V + 7) // 8 * 8)
else:
    c = dict(synth.CONFIGS[name])
    inp = synth.gauss_chain(B, c["V"], c["K"], c["L"], c["sigmas"], s=c["s"], seed=c["seed"], device="cuda", dtype=c["dtype"])
o = to_np(api.chain_verify(inp.levels, inp.draft, inp.u_acc, inp.u_emit, V=inp.V)); torch.cuda.synchronize()
ref = run_oracle(inp)
rep = compare(o, ref)
print("report", {k: v for k, v in rep.items()})
kd = np.abs(o["pos_kl"].astype(np.float64) - ref["pos_kl"])
w = np.unravel_index(np.argmax(kd - 1e-4 * np.abs(ref["pos_kl"])), kd.shape)
print("worst KL", w, o["pos_kl"][w], ref["pos_kl"][w], "dtv", o["pos_dtv"][w], ref["pos_dtv"][w])
for b in rep["mismatch"]:
    print("req", b, "flags", o["flags"][b])
    print("  gpu n", o["n_acc"][:, b], "m", o["m_cand"][:, b], "tok", o["commit_tok"][b], "rb", o["rollback"][:, b])
    print("  ref n", ref["n_acc"][:, b], "m", ref["m_cand"][:, b], "tok", ref["out_tok"][b], "rb", ref["rollback"][:, b], "tie", ref["near_tie"][b])
    print("  dtv gpu", o["pos_dtv"][:, b], "\n  dtv ref", ref["pos_dtv"][:, b])
os.environ["MSD_EXACT_DRAWS"] = "1"
o2 = to_np(api.chain_verify(inp.levels, inp.draft, inp.u_acc, inp.u_emit, V=inp.V)); torch.cuda.synchronize()
print("exact-draw report", compare(o2, ref))
