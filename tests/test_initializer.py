"""Initializers (initializer.cpp:91-132; the reference's test_initializer.cpp
cases restated).  Ortho-core runs on the GPU in fp64: each core's slice
vectors are orthonormal to 1e-10, a feasible table is semi-orthogonal
(W^T W = alpha I), infeasible ranks name the offending core and bound."""
import numpy as np
import pytest

import oracle
from paper_2206_10581_b200 import config as C
from paper_2206_10581_b200.initializer import InfeasibleRanksError, init_gaussian, init_ortho_core


def slice_gram(cfg, cores, k):
    """Gram of core k's n_k R_{k-1} slice vectors (r, j) -> G_k(r, :, j, :)."""
    R0, m, n, R1 = cfg.core_shape(k)
    v = cores[k].transpose(0, 2, 1, 3).reshape(R0 * n, m * R1)
    return v @ v.T


def materialize(cfg, cores):
    W, bad = oracle.lookup_batch(cfg, cores, np.arange(cfg.num_nodes, dtype=np.int64))
    assert bad == -1
    return W


def test_infeasible_ranks_rejected_with_core_and_bound():  # test_initializer.cpp:104-113
    cfg = C.plan_factorization(169363, 128, [55, 55, 56], [8, 4, 4], [1, 32, 32, 1])
    with pytest.raises(InfeasibleRanksError) as e:
        init_ortho_core(cfg, 1)
    assert (e.value.core_index, e.value.num_vectors, e.value.vector_dim) == (2, 128, 56)
    small = C.plan_factorization(4, 4, [2, 2], [2, 2], [1, 2, 1])
    with pytest.raises(InfeasibleRanksError):
        init_ortho_core(small, 3)


def test_gaussian_init_deterministic_and_std():
    cfg = C.plan_factorization(1000, 16, [10, 10, 10], [2, 2, 4], [1, 8, 8, 1])
    a, b = init_gaussian(cfg, 7, 0.1), init_gaussian(cfg, 7, 0.1)
    for x, y in zip(a, b):
        np.testing.assert_array_equal(x, y)
    allv = np.concatenate([x.ravel() for x in a])
    assert abs(allv.std() - 0.1) < 0.01 and abs(allv.mean()) < 0.01
    with pytest.raises(ValueError):
        init_gaussian(cfg, 7, -1.0)


@pytest.mark.gpu
def test_ortho_slices_orthonormal():  # test_initializer.cpp:115-122
    cfg = C.plan_factorization(169363, 128, [55, 55, 56], [8, 4, 4], [1, 8, 8, 1])
    cores = init_ortho_core(cfg, 1)
    for k in range(cfg.d):
        g = slice_gram(cfg, cores, k)
        assert np.max(np.abs(g - np.eye(g.shape[0]))) <= 1e-10


@pytest.mark.gpu
def test_ortho_semi_orthogonal_table():  # test_initializer.cpp:73-95
    cfg = C.plan_factorization(4, 4, [2, 2], [2, 2], [1, 1, 1])
    W = materialize(cfg, init_ortho_core(cfg, 3))
    gram = W.T @ W
    alpha = gram[0, 0]
    assert alpha > 0 and np.max(np.abs(gram - alpha * np.eye(4))) <= 1e-10
    wide = C.plan_factorization(8, 4, [2, 4], [2, 2], [1, 2, 1])
    W = materialize(wide, init_ortho_core(wide, 5))
    gram = W.T @ W
    assert np.max(np.abs(gram - gram[0, 0] * np.eye(4))) <= 1e-10


@pytest.mark.gpu
def test_ortho_unit_norm_column():  # test_initializer.cpp:97-102
    cfg = C.plan_factorization(12, 1, [3, 4], [1, 1], [1, 1, 1])
    W = materialize(cfg, init_ortho_core(cfg, 5))
    assert abs(np.linalg.norm(W[:, 0]) - 1.0) <= 1e-12


@pytest.mark.gpu
def test_ortho_random_feasible_configs_and_target_scale():  # test_initializer.cpp:125-152, 176-182
    rng = np.random.default_rng(99)
    accepted = 0
    while accepted < 12:
        d = int(rng.integers(2, 4))
        m = [int(x) for x in rng.integers(2, 17, d)]
        n = [int(x) for x in rng.integers(1, 5, d)]
        R = [1] + [int(x) for x in rng.integers(1, 9, d - 1)] + [1]
        if np.prod(m) > 4096 or np.prod(n) > 64:
            continue
        if any(n[k] * R[k] > m[k] * R[k + 1] for k in range(d)):
            continue
        accepted += 1
        cfg = C.plan_factorization(int(np.prod(m)), int(np.prod(n)), m, n, R)
        cores = init_ortho_core(cfg, accepted)
        for k in range(d):
            g = slice_gram(cfg, cores, k)
            assert np.max(np.abs(g - np.eye(g.shape[0]))) <= 1e-10
        W = materialize(cfg, cores)
        gram = W.T @ W
        assert np.max(np.abs(gram - gram[0, 0] * np.eye(gram.shape[0]))) <= 1e-8 * gram[0, 0]
    cfg = C.plan_factorization(8, 4, [2, 4], [2, 2], [1, 2, 1])
    W = materialize(cfg, init_ortho_core(cfg, 5, target_scale=0.25))
    assert abs((W.T @ W)[0, 0] - 0.25) <= 1e-12
