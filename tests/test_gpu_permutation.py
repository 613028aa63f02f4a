"""Node relabelling on the device (graph.cpp:218-252
apply_permutation): with a permutation set, lookups and gradients of IDs v
equal those of perm[v] without it, bitwise; range checks and error positions
stay on the caller's IDs; invalid permutations are rejected."""
import numpy as np
import pytest

from paper_2206_10581_b200 import config as C
from paper_2206_10581_b200 import synth

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name,path", [("products", "auto"), ("products", "tc"), ("tiny", "generic")])
def test_permuted_lookup_and_backward(name, path):
    import torch
    from paper_2206_10581_b200 import engine as E
    cfg = (C.WORKLOADS[name]["cfg"]() if name != "tiny"
           else C.plan_factorization(12, 8, [2, 3, 2], [2, 2, 2], [1, 3, 2, 1]))
    B = min(2048, 4 * cfg.num_nodes)
    cores = synth.gaussian_cores(cfg, 51)
    rng = np.random.default_rng(5)
    perm = rng.permutation(cfg.num_nodes).astype(np.int64)
    idx = synth.uniform_ids(52, B, cfg.num_nodes)
    up = synth.normal(53, 1, B * cfg.emb_dim).reshape(B, cfg.emb_dim)
    outs, grads = [], []
    for use_perm in (True, False):
        emb = E.TTEmbedding(cfg, 0)
        emb.set_cores(cores)
        emb.set_path(path)
        if use_perm:
            emb.set_permutation(perm)
        ids = idx if use_perm else perm[idx]
        out = emb.forward(torch.tensor(ids, device="cuda:0"))
        emb.backward(torch.tensor(up, device="cuda:0"))
        emb.sync()
        outs.append(out.cpu().numpy())
        grads.append(emb._fetch_grads())
    np.testing.assert_array_equal(outs[0], outs[1])
    for a, b in zip(grads[0], grads[1]):
        np.testing.assert_array_equal(a, b)


def test_permutation_errors():
    import torch
    from paper_2206_10581_b200 import engine as E
    cfg = C.plan_factorization(12, 8, [2, 3, 2], [2, 2, 2], [1, 3, 2, 1])
    emb = E.TTEmbedding(cfg, 0)
    emb.set_cores(synth.gaussian_cores(cfg, 1))
    with pytest.raises(E.InvalidArgument, match="size mismatch"):
        emb.set_permutation(np.arange(11))
    bad = np.arange(12)
    bad[3] = 4
    with pytest.raises(E.InvalidArgument, match="not a permutation"):
        emb.set_permutation(bad)
    emb.set_permutation(np.arange(12)[::-1].copy())
    with pytest.raises(E.OutOfRange, match="index 12 at batch position 2"):
        emb.forward(torch.tensor([0, 5, 12, 3], device="cuda:0"))
        emb.sync()
    emb.set_permutation(None)
    out = emb.forward(torch.tensor([0, 11], device="cuda:0")).cpu().numpy()
    emb.sync()
    assert out.shape == (2, 8)
