import os, sys
sys.path.insert(0, "/root/repo")
import numpy as np, torch
from paper_2505_07680_b200 import api, synth
from tests._parity import run_oracle, to_np
c = synth.CONFIGS["llama3"]
inp = synth.gauss_chain(4, c["V"], c["K"], c["L"], c["sigmas"], seed=4, device="cuda", dtype="bf16")
o = to_np(api.chain_verify(inp.levels, inp.draft, inp.u_acc, inp.u_emit)); torch.cuda.synchronize()
ref = run_oracle(inp)
np.set_printoptions(precision=5, suppress=True, linewidth=200)
print("gpu dtv\n", o["pos_dtv"][:, :2]); print("ref dtv\n", ref["pos_dtv"][:, :2])
print("ratio\n", o["pos_dtv"][:, :2] / ref["pos_dtv"][:, :2])
print("gpu kl\n", o["pos_kl"][:, :2]); print("ref kl\n", ref["pos_kl"][:, :2])
print("n gpu", o["n_acc"], "\nn ref", ref["n_acc"])
