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
