"""Runs forward+backward(indices) so the fused forward runs without its epilogue (for ncu)."""
import sys
import torch
from paper_2206_10581_b200 import engine as E
from paper_2206_10581_b200.config import workload_inputs
cfg, idx, up, cores = workload_inputs("papers", 2026)
emb = E.TTEmbedding(cfg)
emb.set_cores(cores)
emb.set_path(sys.argv[1] if len(sys.argv) > 1 else "auto")
ti, tu = torch.tensor(idx, device="cuda"), torch.tensor(up, device="cuda")
for _ in range(2):
    emb.backward(tu, ti)
torch.cuda.synchronize()
emb.sync()
print("ok")
