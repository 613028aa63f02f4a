"""ID-owner sharding (dist.OwnerShardedTT) with the real CUDA engine: two
ranks on cuda:0 as threads (tests/threadcomm.py) against the oracle on the
full batch.  Rows must come back to their positions; the replicated cores'
all-reduced gradients and each owner's level-F slices must equal the
full-batch gradient (1e-5 a_ref); the update must leave the
replicated cores bitwise identical on every rank."""
import numpy as np
import pytest

import oracle
from paper_2206_10581_b200 import config as C
from paper_2206_10581_b200 import dist as D
from paper_2206_10581_b200 import synth
from threadcomm import run_ranks

pytestmark = pytest.mark.gpu
TOL = 1e-5


def _close(x, ref, aref, what):
    err = np.abs(np.asarray(x, np.float64) - ref)
    worst = float(np.max(err / (TOL * aref + 1e-30))) if err.size else 0.0
    assert worst <= 1.0, f"{what}: {worst:.3g}"


@pytest.mark.parametrize("name,path,world", [("products", "auto", 2), ("products", "tc", 3), ("billion", "auto", 2)])
def test_owner_sharded_step(name, path, world):
    import torch
    from paper_2206_10581_b200 import engine as E
    cfg = C.WORKLOADS[name]["cfg"]()
    F = cfg.d - 2
    B = 1536
    cores = synth.gaussian_cores(cfg, 11)
    idx = synth.zipf_ids(12, B, 1.1, cfg.num_nodes)
    up = synth.normal(13, 1, B * cfg.emb_dim).reshape(B, cfg.emb_dim)
    c64 = [c.astype(np.float64) for c in cores]
    ref_rows, _ = oracle.lookup_batch(cfg, c64, idx)
    aref_rows, _ = oracle.lookup_batch(cfg, [np.abs(c) for c in c64], idx)
    ref_g, _ = oracle.backward_lookup(cfg, c64, idx, up)
    aref_g, _ = oracle.backward_lookup(cfg, [np.abs(c) for c in c64], idx, np.abs(up.astype(np.float64)))
    bnd = D.owner_bounds(cfg, world)
    res = {}

    def rank_fn(r, comm):
        emb = E.TTEmbedding(cfg, 0)
        emb.set_cores(cores)
        emb.set_path(path)
        emb.configure_optimizer(E.OptimizerState.make(cfg, E.OptKind.sgd, 0.01))
        dp = D.OwnerShardedTT(emb, comm=comm)
        lo, hi = D.shard_bounds(B, r, world)
        rows = dp.forward(torch.tensor(idx[lo:hi], device="cuda:0"))
        dp.backward(torch.tensor(up[lo:hi], device="cuda:0"))
        dp.allreduce()
        emb.sync()
        g = emb._fetch_grads()
        dp.emb.step()  # gradients already reduced
        emb.sync()
        res[r] = (rows.cpu().numpy(), g, emb.get_cores(np.float32), lo, hi)
        del dp, emb

    run_ranks(world, rank_fn)
    for r in range(world):
        rows, g, new, lo, hi = res[r]
        _close(rows, ref_rows[lo:hi], aref_rows[lo:hi], f"rank {r} rows")
        a, b = bnd[r], bnd[r + 1]
        for k in range(cfg.d):
            if k == F:
                _close(g[k][:, a:b], ref_g[k][:, a:b], aref_g[k][:, a:b], f"rank {r} owned dG_{k}")
                mask = np.ones(cfg.m[k], bool)
                mask[a:b] = False
                assert np.all(g[k][:, mask] == 0.0)
            else:
                _close(g[k], ref_g[k], aref_g[k], f"rank {r} replicated dG_{k}")
        for k in range(cfg.d):
            if k != F:
                np.testing.assert_array_equal(new[k], res[0][2][k])  # replicated cores identical
