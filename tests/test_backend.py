"""EmbeddingBackend (gnn.hpp:38-72, gnn.cpp:37-128): the full-table kind on
the host (CPU tests) and the tensor-train kind on the CUDA engine (GPU tests,
against the oracle's backward_lookup over all rows + apply_update)."""
import numpy as np
import pytest

import oracle
from paper_2206_10581_b200 import config as C
from paper_2206_10581_b200 import synth
from paper_2206_10581_b200.backend import BackendKind, EmbeddingBackend
from paper_2206_10581_b200.config import InvalidArgument, OutOfRange

SGD, ADAM, ADAGRAD = 0, 1, 2


def test_full_table_lookup_and_errors():
    b = EmbeddingBackend.full_table(50, 6, 3, 0.1, ADAM, 0.01)
    assert b.kind() == BackendKind.full and b.num_nodes() == 50 and b.emb_dim() == 6 and b.param_count() == 300
    t = b.lookup_all()
    np.testing.assert_array_equal(b.lookup([4, 4, 9]), t[[4, 4, 9]])
    with pytest.raises(OutOfRange, match="index 50 at batch position 1"):
        b.lookup([0, 50])
    with pytest.raises(InvalidArgument, match="bad gradient shape"):
        b.apply_gradients(np.zeros((49, 6)))
    g = np.zeros((50, 6))
    g[3, 2] = np.nan
    with pytest.raises(InvalidArgument, match="non-finite"):
        b.apply_gradients(g)
    np.testing.assert_array_equal(b.lookup_all(), t)  # rejected update left the table untouched
    with pytest.raises(RuntimeError, match="not tensor-train"):
        b.tt()


@pytest.mark.parametrize("opt", [SGD, ADAM])
def test_full_table_update_matches_reference_formulas(opt):
    rng = np.random.default_rng(1)
    tab = rng.standard_normal((20, 4))
    b = EmbeddingBackend.full_table_from(tab, opt, 0.05)
    p, m, v = tab.copy(), np.zeros_like(tab), np.zeros_like(tab)
    for step in (1, 2, 3):
        g = rng.standard_normal((20, 4))
        b.apply_gradients(g)
        if opt == SGD:
            p -= 0.05 * g
        else:  # adam_step, autodiff.cpp:135-145
            m = 0.9 * m + 0.1 * g
            v = 0.999 * v + 0.001 * g * g
            p -= 0.05 * (m / (1 - 0.9 ** step)) / (np.sqrt(v / (1 - 0.999 ** step)) + 1e-8)
    np.testing.assert_allclose(b.table(), p, rtol=1e-14, atol=1e-15)


@pytest.mark.gpu
@pytest.mark.parametrize("opt", [SGD, ADAGRAD])
def test_tt_backend_matches_oracle(opt):
    from paper_2206_10581_b200 import engine as E
    cfg = C.plan_factorization(3000, 24, [12, 15, 17], [2, 3, 4], [1, 8, 8, 1])
    cores = synth.gaussian_cores(cfg, 41)
    emb = E.TTEmbedding(cfg, 0)
    emb.set_cores(cores)
    b = EmbeddingBackend.tensor_train(emb, opt, 0.01)
    assert b.kind() == BackendKind.tt and b.num_nodes() == 3000 and b.emb_dim() == 24
    c64 = [c.astype(np.float64) for c in cores]
    allidx = np.arange(cfg.num_nodes, dtype=np.int64)
    ref, _ = oracle.lookup_batch(cfg, c64, allidx)
    aref, _ = oracle.lookup_batch(cfg, [np.abs(c) for c in c64], allidx)
    got = b.lookup_all()
    assert np.all(np.abs(got - ref) <= 1e-5 * aref + 1e-30)
    g = synth.normal(42, 1, cfg.num_nodes * cfg.emb_dim, 1.0, np.float64).reshape(cfg.num_nodes, cfg.emb_dim)
    b.apply_gradients(g.astype(np.float32))
    grads, _ = oracle.backward_lookup(cfg, c64, allidx, g.astype(np.float32).astype(np.float64))
    kind = {SGD: oracle.SGD, ADAGRAD: oracle.ADAGRAD}[opt]
    st = oracle.OptState(cfg, kind, 0.01)
    new = [c.copy() for c in c64]
    assert oracle.apply_update(cfg, new, grads, st) == -1
    after = b.tt().get_cores(np.float64)
    gabs, _ = oracle.backward_lookup(cfg, [np.abs(c) for c in c64], allidx, np.abs(g))
    for k in range(cfg.d):
        if opt == SGD:  # |lr (g - g_ref)| within the gradient bound
            assert np.all(np.abs(after[k] - new[k]) <= 0.01 * 1e-5 * gabs[k] + 1e-7 * np.abs(new[k]) + 1e-12)
        else:  # Adagrad step 1 is sign-sensitive where |g_ref| is within fp32 noise
            safe = np.abs(grads[k]) > 1e-5 * gabs[k]
            assert np.all(np.abs(after[k] - new[k])[safe] <= 1e-6)
    with pytest.raises(RuntimeError, match="not a full table"):
        b.table()
