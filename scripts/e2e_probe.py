"""Where the pipelined host-buffer step's time goes (papers): the
tt_train_step_submit/_wait loop with / without the per-step core restore and
with / without the row download."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2206_10581_b200 import engine as E  # noqa: E402
from paper_2206_10581_b200.config import WORKLOADS, workload_inputs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "papers"
cfg, idx, up, cores = workload_inputs(name, 2026)
emb = E.TTEmbedding(cfg, 0)
emb.set_cores(cores)
emb.configure_optimizer(E.OptimizerState.make(cfg, getattr(E.OptKind, WORKLOADS[name]["opt"]), 0.01))
emb.snapshot_cores()
h_idx = torch.tensor(idx).pin_memory()
h_up = torch.tensor(up).pin_memory()
h_out = torch.empty((len(idx), cfg.emb_dim), dtype=torch.float32).pin_memory()


DEPTH = int(sys.argv[2]) if len(sys.argv) > 2 else 3


def run(n, restore, out):
    inflight = 0
    for i in range(n):
        if restore:
            emb.restore_cores_on_engine_stream()
        emb.train_step_submit(h_idx, h_up, h_out if out else None)
        inflight += 1
        if inflight >= DEPTH:
            emb.train_step_wait()
            inflight -= 1
    for _ in range(inflight):
        emb.train_step_wait()


for restore in (True, False):
    for out in (True, False):
        run(3, restore, out)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        run(10, restore, out)
        torch.cuda.synchronize()
        ms = (time.perf_counter() - t0) / 10 * 1e3
        print(f"restore={restore} download={out}: {ms:.3f} ms/step, {len(idx) / ms / 1e3:.2f} M rows/s")
