"""Generates the committed golden fixtures (TEST INFRASTRUCTURE ONLY).

Run here, where /root/reference exists:  python tests/golden/make_golden.py

* ref_digits.npz  -- mixed-radix digits, parameter counts and the auto planner's
  factors produced by the REFERENCE's own tt_config.cpp (oracle/_ref).
* fwd_bwd_*.npz   -- embeddings, core gradients (fp64 C oracle, pinned by the
  reference's KATs) and the condition bounds a_ref, on seeded inputs from
  paper_2206_10581_b200.synth (inputs are regenerated from the seeds; their
  checksums are stored).
The GPU box has no /root/reference: these files carry the pins there.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from paper_2206_10581_b200 import config as C  # noqa: E402
from paper_2206_10581_b200 import synth  # noqa: E402

DIGIT_CFGS = {
    "node46": C.plan_factorization(48, 8, [3, 4, 4], [2, 2, 2], [1, 2, 2, 1]),
    "small": C.WORKLOADS["small"]["cfg"](),
    "products": C.WORKLOADS["products"]["cfg"](),
    "papers": C.WORKLOADS["papers"]["cfg"](),
    "billion": C.WORKLOADS["billion"]["cfg"](),
    "d2": C.plan_factorization(99 * 101, 4, [99, 101], [2, 2], [1, 3, 1]),
}

FWD_CASES = {
    # name: (cfg, seed, B, distribution)
    "tiny": (C.plan_factorization(12, 8, [2, 3, 2], [2, 2, 2], [1, 3, 2, 1]), 21, 40, "uniform"),
    "sweep8": (C.WORKLOADS["sweep8"]["cfg"](), 22, 96, "zipf"),
    "small": (C.WORKLOADS["small"]["cfg"](), 23, 48, "uniform"),
}


def inputs(cfg, seed, B, dist):
    idx = synth.uniform_ids(seed, B, cfg.num_nodes) if dist == "uniform" else synth.zipf_ids(seed, B, 1.1, cfg.num_nodes)
    up = synth.normal(seed, 7, B * cfg.emb_dim).reshape(B, cfg.emb_dim)
    cores = synth.gaussian_cores(cfg, seed, 0.1)
    return idx, up, cores


def main():
    assert oracle.ref() is not None, "needs oracle/_ref (the reference's tt_config.cpp)"
    out = {}
    for name, cfg in DIGIT_CFGS.items():
        rows = np.concatenate([np.arange(min(cfg.padded_rows(), 200)),
                               synth.bounded(99, 1, 300, min(cfg.padded_rows(), 1 << 32)),
                               [cfg.padded_rows() - 1]]).astype(np.int64)
        dig, bad = oracle.ref_digits(cfg, rows)
        assert bad == -1
        out[f"{name}_rows"] = rows
        out[f"{name}_digits"] = dig
        out[f"{name}_params"] = np.int64(oracle.ref_count_params(cfg))
        out[f"{name}_m"] = np.array(cfg.m, np.int64)
        out[f"{name}_n"] = np.array(cfg.n, np.int64)
        out[f"{name}_R"] = np.array(cfg.R, np.int64)
        out[f"{name}_M"] = np.int64(cfg.num_nodes)
        out[f"{name}_N"] = np.int64(cfg.emb_dim)
    for M, N, d in [(169363, 128, 3), (2449029, 100, 3), (1000, 64, 2), (100000, 256, 4)]:
        R = [1] + [4] * (d - 1) + [1]
        m, n = oracle.ref_plan_auto(M, N, d, R, True)
        out[f"plan_{M}_{N}_{d}"] = np.array(m + n, np.int64)
    np.savez_compressed(os.path.join(HERE, "ref_digits.npz"), **out)

    for name, (cfg, seed, B, dist) in FWD_CASES.items():
        idx, up, cores = inputs(cfg, seed, B, dist)
        c64 = [c.astype(np.float64) for c in cores]
        y, _ = oracle.lookup_batch(cfg, c64, idx)
        ya, _ = oracle.lookup_batch(cfg, [np.abs(c) for c in c64], idx)
        g, _ = oracle.backward_lookup(cfg, c64, idx, up)
        ga, _ = oracle.backward_lookup(cfg, [np.abs(c) for c in c64], idx, np.abs(up.astype(np.float64)))
        rec = {"seed": np.int64(seed), "B": np.int64(B), "dist": np.array(dist),
               "idx_sum": np.array(synth.checksum(idx)), "up_sum": np.array(synth.checksum(up)),
               "cores_sum": np.array(synth.checksum(np.concatenate([c.ravel() for c in cores]))),
               "out": y, "out_abs": ya}
        for k in range(cfg.d):
            rec[f"grad{k}"] = g[k]
            rec[f"grad_abs{k}"] = ga[k]
        np.savez_compressed(os.path.join(HERE, f"fwd_bwd_{name}.npz"), **rec)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
