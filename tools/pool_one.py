import sys, os
sys.path.insert(0, os.getcwd())
import torch
from paper_2505_07680_b200 import api, synth
c = synth.CONFIGS["llama3"]
inp = synth.config_inputs("llama3", device="cuda")
for _ in range(2):
    api.pool_divergence(inp.levels, K=c["K"], V=c["V"])
torch.cuda.synchronize()
