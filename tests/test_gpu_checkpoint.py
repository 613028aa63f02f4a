"""Device checkpoints (tt_io.save_checkpoint / load_checkpoint): cores and
optimizer state of a training engine resume bit-exactly -- two steps in one
engine equal one step, checkpoint, a fresh engine from the files, one step."""
import numpy as np
import pytest

from paper_2206_10581_b200 import config as C
from paper_2206_10581_b200 import synth

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("opt", ["sgd", "adagrad", "adam"])
def test_checkpoint_resume_bit_exact(tmp_path, opt):
    import torch
    from paper_2206_10581_b200 import engine as E
    from paper_2206_10581_b200.tt_io import load_checkpoint, save_checkpoint
    cfg = C.WORKLOADS["products"]["cfg"]()
    B = 1024
    cores = synth.gaussian_cores(cfg, 21)
    batches = [(synth.zipf_ids(22 + i, B, 1.1, cfg.num_nodes), synth.normal(30 + i, 1, B * cfg.emb_dim).reshape(B, cfg.emb_dim))
               for i in range(2)]
    kind = getattr(E.OptKind, opt)

    def step(emb, i):
        idx, up = batches[i]
        emb.forward(torch.tensor(idx, device="cuda:0"))
        emb.backward(torch.tensor(up, device="cuda:0"))
        emb.step()
        emb.sync()

    a = E.TTEmbedding(cfg, 0)
    a.set_cores(cores)
    a.configure_optimizer(E.OptimizerState.make(cfg, kind, 0.01))
    step(a, 0)
    p = str(tmp_path / "ck.tte")
    save_checkpoint(a, p)
    step(a, 1)
    b = load_checkpoint(p, 0)
    assert b.opt_step() == 1
    step(b, 1)
    assert b.opt_step() == 2
    for x, y in zip(a.get_cores(np.float32), b.get_cores(np.float32)):
        np.testing.assert_array_equal(x, y)
    sa, sb = a.get_opt_state(), b.get_opt_state()
    for arrs_a, arrs_b in zip(sa[:2], sb[:2]):
        if arrs_a is None:
            assert arrs_b is None
            continue
        for x, y in zip(arrs_a, arrs_b):
            np.testing.assert_array_equal(x, y)


def test_pipelined_host_steps_equal_synchronous_steps():
    """tt_train_step_submit / _wait (two steps in flight) == tt_train_step_host
    step by step: same rows, same cores after 3 steps; errors surface at the
    wait of the failing step."""
    from paper_2206_10581_b200 import engine as E
    cfg = C.WORKLOADS["products"]["cfg"]()
    B = 2048
    cores = synth.gaussian_cores(cfg, 31)
    batches = [(synth.zipf_ids(40 + i, B, 1.1, cfg.num_nodes),
                synth.normal(50 + i, 1, B * cfg.emb_dim).reshape(B, cfg.emb_dim).astype(np.float32)) for i in range(3)]
    outs = []
    engines = []
    for pipelined in (False, True):
        emb = E.TTEmbedding(cfg, 0)
        emb.set_cores(cores)
        emb.configure_optimizer(E.OptimizerState.make(cfg, E.OptKind.adagrad, 0.01))
        rows = [np.empty((B, cfg.emb_dim), np.float32) for _ in batches]
        for i, (idx, up) in enumerate(batches):
            if pipelined:
                emb.train_step_submit(idx, up, rows[i])
                if i > 0:
                    emb.train_step_wait()
            else:
                emb.train_step_host(idx, up, rows[i])
        if pipelined:
            emb.train_step_wait()
        outs.append(rows)
        engines.append(emb)
    for a, b in zip(*outs):
        np.testing.assert_array_equal(a, b)
    for x, y in zip(engines[0].get_cores(np.float32), engines[1].get_cores(np.float32)):
        np.testing.assert_array_equal(x, y)
    assert engines[1].opt_step() == 3
    bad = batches[0][0].copy()
    bad[5] = cfg.num_nodes
    emb = engines[1]
    emb.train_step_submit(batches[1][0], batches[1][1])
    emb.train_step_submit(bad, batches[0][1])
    emb.train_step_wait()
    with pytest.raises(C.OutOfRange, match="position 5"):
        emb.train_step_wait()
