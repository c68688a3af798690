"""Time msd_draft_sample on a config's drafter rows (B requests, one row each); prints ms and
the algorithmic bandwidth B * V * elem bytes / time (one streaming read)."""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_07680_b200 import api, synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="llama3")
ap.add_argument("--iters", type=int, default=50)
ap.add_argument("--greedy", action="store_true")
a = ap.parse_args()
c = synth.CONFIGS[a.config]
inp = synth.config_inputs(a.config, device="cuda")
z, V, B = inp.levels[0], c["V"], c["B"]
u = torch.rand((B,), device="cuda")
out = api.draft_sample(z, u, V=V, greedy=a.greedy)
# K draft steps (rows 0..K-1, K * B * V * elem > L2, so every launch streams from HBM)
# captured in one CUDA graph: no host launch gaps inside the timed region
K = c["K"]
s_ = torch.cuda.Stream()
with torch.cuda.stream(s_):
    for k in range(K):
        api.draft_sample(z, u, row=k, V=V, greedy=a.greedy, out=out)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s_):
        for k in range(K):
            api.draft_sample(z, u, row=k, V=V, greedy=a.greedy, out=out)
torch.cuda.synchronize()
for _ in range(3):
    g.replay()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
e0.record()
for _ in range(a.iters):
    g.replay()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / (a.iters * K)
by = B * V * (2 if c["dtype"] == "bf16" else 4)
print(f"{a.config}{' greedy' if a.greedy else ''}: B={B} V={V}: {ms * 1e3:.1f} us per step, "
      f"{by / ms / 1e6:.0f} GB/s algorithmic ({K} rows per graph, {K * by / 1e6:.0f} MB > L2)")
