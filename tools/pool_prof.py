"""Time msd_pool_divergence (SimScore bootstrap) on a config's draft rows; prints ms and the
algorithmic bandwidth 2 * N * V * elem * B * K bytes / time (two streaming passes)."""
import argparse
import sys
import os

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_07680_b200 import api, synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="llama3")
ap.add_argument("--iters", type=int, default=20)
a = ap.parse_args()
c = synth.CONFIGS[a.config]
inp = synth.config_inputs(a.config, device="cuda")
K, V, N = c["K"], c["V"], c["L"]
for _ in range(3):
    api.pool_divergence(inp.levels, K=K, V=V)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
e0.record()
for _ in range(a.iters):
    api.pool_divergence(inp.levels, K=K, V=V)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / a.iters
esz = 2 if c["dtype"] == "bf16" else 4
by = 2 * N * V * esz * c["B"] * K
print(f"{a.config}: N={N} B={c['B']} K={K} V={V}: {ms:.3f} ms, {by / ms / 1e6:.0f} GB/s algorithmic (2 passes)")
