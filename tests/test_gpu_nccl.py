"""The engine's own NCCL data plane (tt_comm_init_rank / tt_allreduce_grads)
through dist.DataParallelTT, in a 1-rank NCCL job on one GPU: the all-reduce
over one rank is the identity, so a step must equal the plain single-engine
step bit for bit (forward rows, core gradients, updated cores), eagerly and
replayed from a CUDA graph that captured the NCCL call.  (Multi-rank runs
need one GPU per rank: bench.py --gpus N under torchrun.)"""
import os

import numpy as np
import pytest

from paper_2206_10581_b200 import config as C
from paper_2206_10581_b200 import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def nccl_world1():
    import torch.distributed as dist
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29533")
    import torch
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    yield dist
    dist.destroy_process_group()


@pytest.mark.parametrize("name,path", [("products", "auto"), ("papers", "auto"), ("papers", "tc"), ("billion", "auto")])
def test_native_nccl_step_equals_single_engine(nccl_world1, name, path):
    import torch
    from paper_2206_10581_b200 import engine as E
    from paper_2206_10581_b200.dist import DataParallelTT
    cfg = C.WORKLOADS[name]["cfg"]()
    B = 4096
    idx = torch.tensor(synth.zipf_ids(3, B, 1.1, cfg.num_nodes), device="cuda")
    up = torch.tensor(synth.normal(4, 1, B * cfg.emb_dim).reshape(B, cfg.emb_dim), device="cuda")
    cores = synth.gaussian_cores(cfg, 5)
    kind = getattr(E.OptKind, C.WORKLOADS[name]["opt"])
    outs, cs = [], []
    for native in (False, True):
        emb = E.TTEmbedding(cfg, 0)
        emb.set_cores(cores)
        emb.set_path(path)
        emb.configure_optimizer(E.OptimizerState.make(cfg, kind, 0.01))
        dp = DataParallelTT(emb) if native else None
        if native:
            assert dp.native
        o = emb.forward(idx)
        emb.backward(up)
        if native:
            dp.allreduce()
        emb.step()
        emb.sync()
        outs.append(o.cpu().numpy())
        cs.append(emb.get_cores(np.float32))
        if native:  # the same step captured in a CUDA graph (NCCL inside) and replayed
            emb.set_cores(cores)
            s = torch.cuda.Stream()
            s.wait_stream(torch.cuda.current_stream())
            g = torch.cuda.CUDAGraph()
            with torch.cuda.stream(s):
                with torch.cuda.graph(g, stream=s):
                    emb.forward(idx, o)
                    emb.backward(up)
                    dp.allreduce()
                    emb.step()
            torch.cuda.current_stream().wait_stream(s)
            emb.set_cores(cores)
            emb.configure_optimizer(E.OptimizerState.make(cfg, kind, 0.01))
            g.replay()
            torch.cuda.synchronize()
            emb.sync()
            for a, b in zip(cs[0], emb.get_cores(np.float32)):
                np.testing.assert_array_equal(a, b)
    np.testing.assert_array_equal(outs[0], outs[1])
    for a, b in zip(cs[0], cs[1]):
        np.testing.assert_array_equal(a, b)


@pytest.mark.parametrize("name,path", [("products", "auto"), ("papers", "auto"), ("billion", "auto"), ("papers", "tc")])
def test_native_owner_step_equals_single_engine(nccl_world1, name, path):
    """tt_owner_forward / _backward / _step (ID-owner sharding in the engine,
    NCCL point-to-point routing) on a 1-rank communicator == the plain step,
    bit for bit; an out-of-range index fails the routed batch."""
    import torch
    from paper_2206_10581_b200 import config as Cf
    from paper_2206_10581_b200 import engine as E
    from paper_2206_10581_b200.dist import OwnerShardedTT
    cfg = C.WORKLOADS[name]["cfg"]()
    B = 4096
    idx = torch.tensor(synth.zipf_ids(13, B, 1.1, cfg.num_nodes), device="cuda")
    up = torch.tensor(synth.normal(14, 1, B * cfg.emb_dim).reshape(B, cfg.emb_dim), device="cuda")
    cores = synth.gaussian_cores(cfg, 15)
    kind = getattr(E.OptKind, C.WORKLOADS[name]["opt"])
    res = []
    for native in (False, True):
        emb = E.TTEmbedding(cfg, 0)
        emb.set_cores(cores)
        emb.set_path(path)
        emb.configure_optimizer(E.OptimizerState.make(cfg, kind, 0.01))
        if native:
            dp = OwnerShardedTT(emb)
            assert dp.native
            o = dp.forward(idx)
            assert emb.owner_rows() == B
            dp.backward(up)
            dp.step()
        else:
            o = emb.forward(idx)
            emb.backward(up)
            emb.step()
        emb.sync()
        res.append((o.cpu().numpy(), emb.get_cores(np.float32)))
        if native:
            bad = idx.clone()
            bad[7] = cfg.num_nodes
            with pytest.raises(Cf.OutOfRange, match="position 7"):
                dp.forward(bad)
    np.testing.assert_array_equal(res[0][0], res[1][0])
    for a, b in zip(res[0][1], res[1][1]):
        np.testing.assert_array_equal(a, b)
