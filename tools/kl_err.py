"""KL / DTV error of the GPU path vs the oracle on near-identical levels: the worst positions."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2505_07680_b200 import api, synth
from tests._parity import run_oracle, to_np
for sig, seed in (((0.12, 0.06, 0.0), 3), ((0.3, 0.05, 0.0), 4), ((0.7, 0.35, 0.0), 5)):
    c = synth.CONFIGS["llama3"]
    inp = synth.gauss_chain(40, 60000, c["K"], c["L"], sig, s=c["s"], seed=seed, device="cuda", dtype="bf16")
    o = to_np(api.chain_verify(inp.levels, inp.draft, inp.u_acc, inp.u_emit, V=inp.V))
    ref = run_oracle(inp)
    for key in ("pos_kl", "pos_dtv"):
        d, dr = o[key].astype(np.float64), ref[key]
        e = np.abs(d - dr)
        ex = e - (1e-4 * np.abs(dr) + 1e-7)
        i = np.unravel_index(np.argmax(ex), ex.shape)
        print(f"{sig} {key}: worst excess {ex.max():.3e} at {i}: gpu {d[i]:.9e} ref {dr[i]:.9e} abs {e[i]:.3e}; "
              f"median ref {np.median(dr):.3e}, abs err p50 {np.median(e):.2e} p99 {np.percentile(e, 99):.2e} max {e.max():.2e}, "
              f"rel p50 {np.median(e / np.maximum(np.abs(dr), 1e-30)):.2e}")
