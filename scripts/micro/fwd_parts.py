"""Diagnostic: forward main-kernel time with and without the last-level
epilogue (backward(indices) re-plans with a forward that writes no rows)."""
import torch
from paper_2206_10581_b200 import engine as E
from paper_2206_10581_b200.config import WORKLOADS, workload_inputs

for name in ("papers",):
    cfg, idx, up, cores = workload_inputs(name, 2026)
    emb = E.TTEmbedding(cfg)
    emb.set_cores(cores)
    ti, tu = torch.tensor(idx, device="cuda"), torch.tensor(up, device="cuda")
    out = torch.empty((len(idx), cfg.emb_dim), device="cuda")
    for _ in range(3):
        emb.forward(ti, out); emb.backward(tu, ti)
    torch.cuda.synchronize(); emb.sync(); emb.profile_read()
    emb.set_profiling(True)
    for _ in range(5):
        emb.forward(ti, out)
    torch.cuda.synchronize()
    with_out = emb.profile_read()
    for _ in range(5):
        emb.backward(tu, ti)
    torch.cuda.synchronize()
    no_out = emb.profile_read()
    f = lambda p, k: p[k][0] / max(p[k][1], 1)
    print(name, "fwd_main with epilogue %.3f ms, without %.3f ms; plan %.3f" % (f(with_out, "fwd_main"), f(no_out, "fwd_main"), f(with_out, "plan")))
