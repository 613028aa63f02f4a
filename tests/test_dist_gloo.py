"""The data-parallel decomposition on CPU (world_size 2, gloo): each rank
takes a position shard of the batch, computes its core gradients (oracle,
fp64), packs them with per-slice touch counts into the engine's flat gradient
buffer layout (paper_2206_10581_b200.dist), and the ranks sum-all-reduce the
buffer exactly as bench.py / DataParallelTT do over NCCL on GPUs.  The
reduced buffer must equal the full-batch gradient, its counters the union of
touched slices, and the touched-only update the reference's dense update."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2206_10581_b200 import config as C
from paper_2206_10581_b200 import dist as D
from paper_2206_10581_b200 import synth


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _cfg():
    return C.plan_factorization(2449029, 128, [126, 140, 140], [4, 4, 8], [1, 4, 4, 1])


def _worker(rank, world, port, B, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = _cfg()
    cores = [c.astype(np.float64) for c in synth.gaussian_cores(cfg, 5)]
    idx = synth.zipf_ids(6, B, 1.1, cfg.num_nodes)
    up = synth.normal(7, 1, B * 128, 1.0, np.float64).reshape(B, 128)
    lo, hi = D.shard_bounds(B, rank, world)
    g, bad = oracle.backward_lookup(cfg, cores, idx[lo:hi], up[lo:hi])
    assert bad == -1
    buf = torch.from_numpy(D.pack_grad_buffer(cfg, g, D.touch_counts(cfg, idx[lo:hi])))
    dist.all_reduce(buf)
    if rank == 0:
        np.save(out, buf.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_allreduce_equals_full_batch(tmp_path, world):
    B = 600
    out = str(tmp_path / "buf.npy")
    mp.start_processes(_worker, args=(world, _free_port(), B, out), nprocs=world, start_method="spawn")
    buf = np.load(out)
    cfg = _cfg()
    assert buf.size == D.grad_buffer_len(cfg)
    grads, touched = D.unpack_grad_buffer(cfg, buf)
    cores = [c.astype(np.float64) for c in synth.gaussian_cores(cfg, 5)]
    idx = synth.zipf_ids(6, B, 1.1, cfg.num_nodes)
    up = synth.normal(7, 1, B * 128, 1.0, np.float64).reshape(B, 128)
    full, _ = oracle.backward_lookup(cfg, cores, idx, up)
    for k in range(cfg.d):
        np.testing.assert_allclose(grads[k], full[k], rtol=1e-11, atol=1e-12)
    # counters: union of touched slices (a slice is touched iff its count > 0)
    want = D.touch_counts(cfg, idx)
    for k in range(cfg.d):
        np.testing.assert_array_equal(touched[k] > 0, want[k] > 0)
        untouched = ~(touched[k] > 0)
        assert np.all(grads[k][:, untouched] == 0.0)
    # touched-only Adagrad on the reduced buffer == the reference's dense update
    dense = [c.copy() for c in cores]
    opt = oracle.OptState(cfg, oracle.ADAGRAD, 0.01)
    assert oracle.apply_update(cfg, dense, full, opt) == -1
    sparse = [c.copy() for c in cores]
    for k in range(cfg.d):
        live = touched[k] > 0
        gk = grads[k][:, live]
        h = gk * gk
        sparse[k][:, live] -= 0.01 * gk / (np.sqrt(h) + 1e-10)
        np.testing.assert_allclose(sparse[k], dense[k], rtol=1e-12, atol=1e-15)


def test_shard_bounds_partition():
    for B in (0, 1, 7, 4096, 262144):
        for world in (1, 2, 3, 8):
            parts = [D.shard_bounds(B, r, world) for r in range(world)]
            assert parts[0][0] == 0 and parts[-1][1] == B
            assert all(parts[i][1] == parts[i + 1][0] for i in range(world - 1))
            assert max(h - l for l, h in parts) - min(h - l for l, h in parts) <= 1


def test_pack_unpack_roundtrip():
    cfg = C.plan_factorization(1000, 30, [7, 11, 13], [2, 3, 5], [1, 5, 3, 1])
    g = [synth.normal(1, k, cfg.core_size(k), 1.0, np.float64).reshape(cfg.core_shape(k)) for k in range(3)]
    t = [np.arange(cfg.m[k], dtype=np.float64) for k in range(3)]
    g2, t2 = D.unpack_grad_buffer(cfg, D.pack_grad_buffer(cfg, g, t))
    for a, b in zip(g, g2):
        np.testing.assert_array_equal(a, b)
    for a, b in zip(t, t2):
        np.testing.assert_array_equal(a, b)


# ---------------------------------------------------------------------------
# ID-owner sharding (paper_2206_10581_b200.dist.OwnerShardedTT): the routing
# helpers are exercised with gloo, the per-rank compute is the oracle.

def _owner_worker(rank, world, port, B, d4, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = _cfg4() if d4 else _cfg()
    F = cfg.d - 2
    cores = [c.astype(np.float64) for c in synth.gaussian_cores(cfg, 5)]
    idx = synth.zipf_ids(6, B, 1.1, cfg.num_nodes)
    up = synth.normal(7, 1, B * cfg.emb_dim, 1.0, np.float64).reshape(B, cfg.emb_dim)
    lo, hi = D.shard_bounds(B, rank, world)
    li = torch.from_numpy(idx[lo:hi].copy())
    recv, route = D.route_to_owners(cfg, li)
    # every routed ID is owned here
    bnd = D.owner_bounds(cfg, world)
    suffix = int(np.prod(cfg.m[F + 1:]))
    dig = (recv.numpy() // suffix) % cfg.m[F]
    assert np.all((dig >= bnd[rank]) & (dig < bnd[rank + 1]))
    # forward on the owner, rows routed back to their positions
    rows, bad = oracle.lookup_batch(cfg, cores, recv.numpy())
    assert bad == -1
    back = D.route_back(torch.from_numpy(rows), route).numpy()
    full_rows, _ = oracle.lookup_batch(cfg, cores, idx[lo:hi])
    np.testing.assert_array_equal(back, full_rows)  # same oracle, same IDs: bitwise
    # backward on the owner with the routed upstream rows
    up_r = D.route_rows(torch.from_numpy(up[lo:hi].copy()), route).numpy()
    g, bad = oracle.backward_lookup(cfg, cores, recv.numpy(), up_r)
    assert bad == -1
    buf = torch.from_numpy(D.pack_grad_buffer(cfg, g, D.touch_counts(cfg, recv.numpy())))
    for o, n in D.replicated_segments(cfg):
        dist.all_reduce(buf[o: o + n])
    np.save(os.path.join(out_dir, f"buf{rank}.npy"), buf.numpy())
    dist.barrier()
    dist.destroy_process_group()


def _cfg4():
    return C.plan_factorization(9 ** 4, 16, [9, 9, 9, 9], [2, 2, 2, 2], [1, 3, 4, 4, 1])


@pytest.mark.parametrize("world,d4", [(2, False), (3, False), (2, True)])
def test_owner_sharding_equals_full_batch(tmp_path, world, d4):
    B = 700
    mp.start_processes(_owner_worker, args=(world, _free_port(), B, d4, str(tmp_path)), nprocs=world,
                       start_method="spawn")
    cfg = _cfg4() if d4 else _cfg()
    F = cfg.d - 2
    bnd = D.owner_bounds(cfg, world)
    cores = [c.astype(np.float64) for c in synth.gaussian_cores(cfg, 5)]
    idx = synth.zipf_ids(6, B, 1.1, cfg.num_nodes)
    up = synth.normal(7, 1, B * cfg.emb_dim, 1.0, np.float64).reshape(B, cfg.emb_dim)
    full, _ = oracle.backward_lookup(cfg, cores, idx, up)
    want_t = D.touch_counts(cfg, idx)
    per = [D.unpack_grad_buffer(cfg, np.load(str(tmp_path / f"buf{r}.npy"))) for r in range(world)]
    for r, (grads, touched) in enumerate(per):
        lo, hi = bnd[r], bnd[r + 1]
        for k in range(cfg.d):
            if k == F:  # sharded core: the owner holds exactly its digit range
                np.testing.assert_allclose(grads[k][:, lo:hi], full[k][:, lo:hi], rtol=1e-11, atol=1e-12)
                mask = np.ones(cfg.m[k], bool)
                mask[lo:hi] = False
                assert np.all(grads[k][:, mask] == 0.0) and np.all(touched[k][mask] == 0.0)
                np.testing.assert_array_equal(touched[k][lo:hi] > 0, want_t[k][lo:hi] > 0)
            else:  # replicated cores: the all-reduced sum is the full-batch gradient on every rank
                np.testing.assert_allclose(grads[k], full[k], rtol=1e-11, atol=1e-12)
                np.testing.assert_array_equal(touched[k] > 0, want_t[k] > 0)
    # each ID's prefix at level F is computed by exactly one rank
    tot = sum(int((per[r][1][F] > 0).sum()) for r in range(world))
    assert tot == int((want_t[F] > 0).sum())


def test_owner_bounds_and_segments():
    for name in ("small", "products", "papers", "billion"):
        cfg = C.WORKLOADS[name]["cfg"]()
        F = cfg.d - 2
        for world in (1, 2, 8):
            b = D.owner_bounds(cfg, world)
            assert b[0] == 0 and b[-1] == cfg.m[F] and all(x < y for x, y in zip(b, b[1:]))
        seg = D.replicated_segments(cfg)
        n = D.grad_buffer_len(cfg)
        covered = sum(l for _, l in seg)
        assert covered == n - cfg.core_size(F) - cfg.m[F]
        assert all(o + l <= n for o, l in seg)
