"""Repeat the saved-plan vs recompute backward at a config and report
mismatching cores / slices (race hunting)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2206_10581_b200 import config as C  # noqa: E402
from paper_2206_10581_b200 import engine as E  # noqa: E402
from paper_2206_10581_b200 import synth  # noqa: E402

name, path, reps = sys.argv[1], sys.argv[2], int(sys.argv[3])
cfg = C.WORKLOADS[name]["cfg"]()
B = 512
cores = synth.gaussian_cores(cfg, 5)
idx = synth.zipf_ids(6, B, 1.1, cfg.num_nodes)
up = synth.normal(7, 1, B * cfg.emb_dim).reshape(B, cfg.emb_dim)
def fresh():
    e = E.TTEmbedding(cfg)
    e.set_cores(cores)
    e.set_path(path)
    return e


emb = fresh()
ti, tu = torch.tensor(idx, device="cuda"), torch.tensor(up, device="cuda")
ref = None
bad = 0
for r in range(reps):
    if os.environ.get("FRESH"):
        del emb
        emb = fresh()
    if r % 2 == 0 or os.environ.get("DEVICE_ONLY"):  # device path (torch's stream)
        out = emb.forward(ti).cpu().numpy()
        emb.backward(tu)
        emb.sync()
        g = emb._fetch_grads()
    else:  # host-buffer path (the engine's own stream), as tests/test_gpu_parity.py does
        out = E.lookup_batch(emb, idx)
        g = E.backward_lookup(emb, idx, up).grads
    if ref is None:
        ref = (out, g)
        continue
    diff_out = np.flatnonzero(np.any(out != ref[0], axis=1))
    diffs = [(k, np.argwhere(g[k] != ref[1][k])) for k in range(cfg.d)]
    msg = [f"core {k}: {len(w)} entries, slices {sorted(set(int(x) for x in w[:, 1]))[:6]}" for k, w in diffs if len(w)]
    if len(diff_out) or msg:
        bad += 1
        print(f"rep {r}: out rows differ {len(diff_out)}; " + "; ".join(msg), flush=True)
print(f"{name} {path}: {bad} of {reps - 1} repetitions differ")
