"""Time msd_logits_process (top-k / top-p) on Llama-3 / Qwen-shaped draft-position rows."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2505_07680_b200 import api  # noqa: E402

for V, B, R in ((128256, 512, 8), (151936, 256, 6)):
    x = (torch.randn((B, R, V), device="cuda") * 2.5).to(torch.bfloat16)
    out = torch.empty_like(x)
    for k, p in ((50, 1.0), (0, 0.9), (50, 0.9), (0, 0.99)):
        api.logits_process(x, top_k=k, top_p=p, out=out)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(3):
            api.logits_process(x, top_k=k, top_p=p, out=out)
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / 3
        print(f"V={V} rows={B * R} top_k={k} top_p={p}: {ms:.3f} ms  {2 * x.numel() * 2 / ms / 1e6:.0f} GB/s "
              f"(one read + one write of the rows)", flush=True)
