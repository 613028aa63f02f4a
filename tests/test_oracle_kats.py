"""Pins the C oracle against every hot-path known-answer / property test the
reference holds.  Each test names the reference test it
restates.  The reference seeds its random fixtures with std::mt19937_64 +
std::normal_distribution (implementation-defined streams), so the random
fixtures here come from the portable generator; the properties are the same.
"""
import math

import numpy as np
import pytest

import oracle
from paper_2206_10581_b200 import synth
from paper_2206_10581_b200.config import plan_factorization


def rand_cores(cfg, seed, scale=1.0):
    return [synth.normal(seed, 100 + k, cfg.core_size(k), scale, np.float64).reshape(cfg.core_shape(k))
            for k in range(cfg.d)]


# ---- tt_config (tests/test_tt_config.cpp) ----------------------------------
def test_node46():  # test_tt_config.cpp:72-75
    cfg = plan_factorization(48, 8, [3, 4, 4], [2, 2, 2], [1, 2, 2, 1])
    assert oracle.index_to_coordinate(cfg, 46) == [2, 3, 2]


def test_odometer_125():  # test_tt_config.cpp:77-89
    cfg = plan_factorization(125, 8, [5, 5, 5], [2, 2, 2], [1, 2, 2, 1])
    allc = [[a, b, c] for a in range(5) for b in range(5) for c in range(5)]
    for i in range(125):
        assert oracle.index_to_coordinate(cfg, i) == allc[i]
        assert oracle.coordinate_to_index(cfg, allc[i]) == i
    assert oracle.index_to_coordinate(cfg, 124) == [4, 4, 4]
    assert oracle.index_to_coordinate(cfg, 0) == [0, 0, 0]
    assert oracle.index_to_coordinate(cfg, 125) is None
    assert oracle.index_to_coordinate(cfg, -1) is None


@pytest.mark.parametrize("factors", [[47, 45, 47], [99, 101], [7, 3, 9, 11]])
def test_round_trip_1e5(factors):  # test_tt_config.cpp:91-103
    rows = math.prod(factors)
    assert rows <= 100000
    cfg = plan_factorization(rows, 1, factors, [1] * len(factors), [1] * (len(factors) + 1))
    for i in range(0, rows, 7):
        assert oracle.coordinate_to_index(cfg, oracle.index_to_coordinate(cfg, i)) == i


def _arxiv(r):
    return plan_factorization(169363, 128, [55, 55, 56], [8, 4, 4], [1, r, r, 1])


def _products(r):
    return plan_factorization(2449029, 100, [125, 140, 140], [4, 5, 5], [1, r, r, 1])


def _papers(r):
    return plan_factorization(111059956, 128, [480, 500, 500], [8, 4, 4], [1, r, r, 1])


TABLE4 = [(_arxiv, 16, 66944, 323), (_arxiv, 32, 246528, 88), (_arxiv, 64, 943616, 23),
          (_products, 16, 198400, 1580), (_products, 32, 755200, 415), (_products, 64, 2944000, 106),
          (_papers, 16, 605440, 23479), (_papers, 32, 2234880, 6360), (_papers, 64, 8565760, 1659)]


@pytest.mark.parametrize("mk,r,params,reduction", TABLE4)
def test_table4_counts(mk, r, params, reduction):  # test_tt_config.cpp:105-126
    cfg = mk(r)
    assert oracle.count_params(cfg) == params
    ratio = cfg.num_nodes * 128.0 / params
    assert math.floor(ratio) == reduction or round(ratio) == reduction


def test_validate_codes():  # tt_config.cpp:92-113 / test_tt_config.cpp:52-59
    from paper_2206_10581_b200.config import TTConfig
    good = plan_factorization(8, 8, [2, 2, 2], [2, 2, 2], [1, 1, 1, 1])
    assert oracle.validate(good) == 0
    assert oracle.validate(TTConfig(8, 8, [2, 2, 2], [2, 2, 2], [2, 2, 2, 2])) != 0
    assert oracle.validate(TTConfig(9, 8, [2, 2, 2], [2, 2, 2], [1, 2, 2, 1])) != 0


# ---- forward (tests/test_tt_embedding.cpp) -----------------------------------
def test_all_ones_rank1():  # test_tt_embedding.cpp:25-35
    cfg = plan_factorization(8, 8, [2, 2, 2], [2, 2, 2], [1, 1, 1, 1])
    cores = [np.ones(cfg.core_shape(k)) for k in range(3)]
    out, bad = oracle.lookup_batch(cfg, cores, np.arange(8))
    assert bad == -1 and out.shape == (8, 8) and np.all(out == 1.0)


def test_chain_matches_scalar_oracle():  # test_tt_embedding.cpp:37-46
    cfg = plan_factorization(12, 8, [2, 3, 2], [2, 2, 2], [1, 2, 2, 1])
    cores = rand_cores(cfg, 7)
    out, _ = oracle.lookup_batch(cfg, cores, [0, 5, 11])
    for b, i in enumerate([0, 5, 11]):
        for j in range(8):
            assert out[b, j] == pytest.approx(oracle.ttm_entry(cfg, cores, i, j), rel=1e-12)


def test_random_small_shapes_vs_scalar():  # test_tt_embedding.cpp:48-71
    rng = np.random.default_rng(123)
    trials = 0
    while trials < 10:
        d = int(rng.integers(2, 4))
        m = [int(x) for x in rng.integers(1, 5, d)]
        n = [int(x) for x in rng.integers(1, 5, d)]
        if math.prod(m) > 64 or math.prod(n) > 16:
            continue
        R = [1] + [int(x) for x in rng.integers(1, 5, d - 1)] + [1]
        cfg = plan_factorization(math.prod(m), math.prod(n), m, n, R)
        cores = rand_cores(cfg, 1000 + trials)
        out, _ = oracle.lookup_batch(cfg, cores, np.arange(cfg.num_nodes))
        for i in range(cfg.num_nodes):
            for j in range(cfg.emb_dim):
                assert out[i, j] == pytest.approx(oracle.ttm_entry(cfg, cores, i, j), rel=1e-12, abs=1e-300)
        trials += 1


def test_batch_contract():  # test_tt_embedding.cpp:106-137
    cfg = plan_factorization(12, 8, [2, 3, 2], [2, 2, 2], [1, 3, 2, 1])
    cores = rand_cores(cfg, 17)
    out, bad = oracle.lookup_batch(cfg, cores, np.zeros(0, np.int64))
    assert out.shape == (0, 8) and bad == -1
    out, _ = oracle.lookup_batch(cfg, cores, [7, 7, 7])
    assert np.array_equal(out[0], out[1]) and np.array_equal(out[1], out[2])
    idx = synth.bounded(17, 1, 16, 12)
    batch, _ = oracle.lookup_batch(cfg, cores, idx)
    for b, i in enumerate(idx):
        row, _ = oracle.lookup_batch(cfg, cores, [i])
        assert np.array_equal(batch[b], row[0])  # bitwise
    _, bad = oracle.lookup_batch(cfg, cores, [0, 1, 99])
    assert bad == 2  # "position 2"


def test_padded_rows_not_served():  # test_tt_embedding.cpp:88-104 (rejection half)
    cfg = plan_factorization(7, 4, [4, 2], [2, 2], [1, 4, 1])
    cores = rand_cores(cfg, 3)
    _, bad = oracle.lookup_batch(cfg, cores, [0, 6, 7])
    assert bad == 2


# ---- backward / update (tests/test_autodiff.cpp) -----------------------------
def quad_loss(cfg, cores, idx, target):
    out, _ = oracle.lookup_batch(cfg, cores, idx)
    return 0.5 * float(np.sum((out - target) ** 2))


def test_zero_upstream():  # test_autodiff.cpp:66-76
    cfg = plan_factorization(12, 8, [2, 3, 2], [2, 2, 2], [1, 2, 2, 1])
    g, bad = oracle.backward_lookup(cfg, rand_cores(cfg, 1), [0, 5, 11], np.zeros((3, 8)))
    assert bad == -1 and all(np.all(x == 0.0) for x in g)


def test_rank1_product_rule():  # test_autodiff.cpp:78-103
    cfg = plan_factorization(6, 4, [2, 3], [2, 2], [1, 1, 1])
    cores = rand_cores(cfg, 2)
    up = np.array([[0.3, -0.7, 1.1, 0.25]])
    g, _ = oracle.backward_lookup(cfg, cores, [4], up)
    a = cores[0].reshape(2, 2)  # (i1, j1)
    b = cores[1].reshape(3, 2)  # (i2, j2)
    u = up.reshape(2, 2)
    for j1 in range(2):
        expect = sum(b[1, j2] * u[j1, j2] for j2 in range(2))
        assert g[0].reshape(2, 2)[1, j1] == pytest.approx(expect, rel=1e-14)
    for j2 in range(2):
        assert g[1].reshape(3, 2)[1, j2] == pytest.approx(a[1, 0] * u[0, j2] + a[1, 1] * u[1, j2], rel=1e-14)
    assert g[0].reshape(2, 2)[0, 0] == 0.0 and g[1].reshape(3, 2)[0, 0] == 0.0


@pytest.mark.parametrize("trial", range(3))
def test_finite_differences(trial):  # test_autodiff.cpp:105-123
    cfg = plan_factorization(12, 8, [3, 2, 2], [2, 2, 2], [1, 3, 2, 1])
    cores = rand_cores(cfg, 30 + trial)
    idx = synth.bounded(40 + trial, 1, 5, 12)
    target = synth.normal(50 + trial, 1, 40, 1.0, np.float64).reshape(5, 8)
    out, _ = oracle.lookup_batch(cfg, cores, idx)
    g, _ = oracle.backward_lookup(cfg, cores, idx, out - target)
    h = 1e-6
    worst = 0.0
    for k in range(cfg.d):
        flat = cores[k].reshape(-1)
        for e in range(flat.size):
            save = flat[e]
            flat[e] = save + h
            up_ = quad_loss(cfg, cores, idx, target)
            flat[e] = save - h
            dn = quad_loss(cfg, cores, idx, target)
            flat[e] = save
            fd = (up_ - dn) / (2 * h)
            an = g[k].reshape(-1)[e]
            worst = max(worst, abs(an - fd) / max(abs(an), abs(fd), 1e-8))
    assert worst <= 1e-4


def test_linearity_and_additivity():  # test_autodiff.cpp:125-162
    cfg = plan_factorization(12, 8, [2, 3, 2], [2, 2, 2], [1, 2, 2, 1])
    cores = rand_cores(cfg, 4)
    idx = [1, 3, 7, 7]
    u = synth.normal(4, 1, 32, 1.0, np.float64).reshape(4, 8)
    v = synth.normal(4, 2, 32, 1.0, np.float64).reshape(4, 8)
    gu, _ = oracle.backward_lookup(cfg, cores, idx, u)
    gv, _ = oracle.backward_lookup(cfg, cores, idx, v)
    gm, _ = oracle.backward_lookup(cfg, cores, idx, 0.7 * u - 1.3 * v)
    for k in range(3):
        np.testing.assert_allclose(gm[k], 0.7 * gu[k] - 1.3 * gv[k], rtol=1e-12, atol=1e-14)
    g1, _ = oracle.backward_lookup(cfg, cores, [6], u[:1])
    g2, _ = oracle.backward_lookup(cfg, cores, [6, 6], np.vstack([u[:1], u[:1]]))
    for k in range(3):
        np.testing.assert_allclose(g2[k], 2.0 * g1[k], rtol=1e-12)


def test_backward_index_error():  # test_autodiff.cpp:164-176 (index half)
    cfg = plan_factorization(12, 8, [2, 3, 2], [2, 2, 2], [1, 2, 2, 1])
    _, bad = oracle.backward_lookup(cfg, rand_cores(cfg, 6), [0, 12], np.zeros((2, 8)))
    assert bad == 1


def test_sgd_zero_grad_noop():  # test_autodiff.cpp:178-188
    cfg = plan_factorization(12, 8, [2, 3, 2], [2, 2, 2], [1, 2, 2, 1])
    cores = rand_cores(cfg, 7)
    before = [c.copy() for c in cores]
    opt = oracle.OptState(cfg, oracle.SGD, 1e-3)
    assert oracle.apply_update(cfg, cores, [np.zeros(cfg.core_size(k)) for k in range(3)], opt) == -1
    assert all(np.array_equal(a, b) for a, b in zip(cores, before)) and opt.step == 1


def test_sgd_descent():  # test_autodiff.cpp:190-202
    cfg = plan_factorization(12, 8, [3, 2, 2], [2, 2, 2], [1, 3, 2, 1])
    cores = rand_cores(cfg, 8)
    idx = [0, 4, 9]
    target = np.zeros((3, 8))
    before = quad_loss(cfg, cores, idx, target)
    out, _ = oracle.lookup_batch(cfg, cores, idx)
    g, _ = oracle.backward_lookup(cfg, cores, idx, out - target)
    opt = oracle.OptState(cfg, oracle.SGD, 1e-3)
    oracle.apply_update(cfg, cores, g, opt)
    assert quad_loss(cfg, cores, idx, target) < before


def test_adam_first_step():  # test_autodiff.cpp:204-218
    cfg = plan_factorization(4, 4, [2, 2], [2, 2], [1, 2, 1])
    cores = [np.zeros(cfg.core_shape(k)) for k in range(2)]
    opt = oracle.OptState(cfg, oracle.ADAM, 1e-3)
    oracle.apply_update(cfg, cores, [np.full(cfg.core_size(k), 37.5) for k in range(2)], opt)
    for c in cores:
        np.testing.assert_allclose(np.abs(c), 1e-3, rtol=1e-4)


def test_nonfinite_rejected():  # test_autodiff.cpp:220-235
    cfg = plan_factorization(4, 4, [2, 2], [2, 2], [1, 2, 1])
    cores = rand_cores(cfg, 9)
    before = [c.copy() for c in cores]
    opt = oracle.OptState(cfg, oracle.ADAM, 1e-3)
    g = [np.zeros(cfg.core_size(k)) for k in range(2)]
    g[1][0] = np.nan
    assert oracle.apply_update(cfg, cores, g, opt) == 1  # "core 1"
    assert all(np.array_equal(a, b) for a, b in zip(cores, before)) and opt.step == 0
    g[1][0] = np.inf
    assert oracle.apply_update(cfg, cores, g, opt) == 1


def test_adagrad_pinned_formula():  # new
    cfg = plan_factorization(4, 4, [2, 2], [2, 2], [1, 2, 1])
    cores = rand_cores(cfg, 10)
    p0 = [c.copy() for c in cores]
    g1 = [synth.normal(10, 20 + k, cfg.core_size(k), 1.0, np.float64) for k in range(2)]
    g2 = [synth.normal(10, 30 + k, cfg.core_size(k), 1.0, np.float64) for k in range(2)]
    opt = oracle.OptState(cfg, oracle.ADAGRAD, 0.01, eps=1e-10)
    oracle.apply_update(cfg, cores, g1, opt)
    oracle.apply_update(cfg, cores, g2, opt)
    for k in range(2):
        h1 = g1[k] ** 2
        p1 = p0[k].ravel() - 0.01 * g1[k] / (np.sqrt(h1) + 1e-10)
        h2 = h1 + g2[k] ** 2
        p2 = p1 - 0.01 * g2[k] / (np.sqrt(h2) + 1e-10)
        np.testing.assert_array_equal(cores[k].ravel(), p2)
    assert opt.step == 2


def test_200_sgd_steps_fit():  # test_autodiff.cpp:237-256
    cfg = plan_factorization(32, 8, [2, 4, 4], [2, 2, 2], [1, 4, 4, 1])
    truth = rand_cores(cfg, 10, 0.5)
    allidx = np.arange(32)
    target, _ = oracle.lookup_batch(cfg, truth, allidx)
    cores = rand_cores(cfg, 11, 0.3)
    opt = oracle.OptState(cfg, oracle.SGD, 0.05)
    initial = quad_loss(cfg, cores, allidx, target)
    for _ in range(200):
        out, _ = oracle.lookup_batch(cfg, cores, allidx)
        g, _ = oracle.backward_lookup(cfg, cores, allidx, out - target)
        oracle.apply_update(cfg, cores, g, opt)
    assert quad_loss(cfg, cores, allidx, target) <= initial / 100.0


# ---- sort / unique / prefixes (new) -------------------------
def test_sort_unique_stable():
    keys = synth.bounded(3, 1, 5000, 700)
    perm, uniq = oracle.sort_unique(keys)
    np.testing.assert_array_equal(perm, np.argsort(keys, kind="stable"))
    np.testing.assert_array_equal(uniq, np.unique(keys))


def test_prefix_counts():
    cfg = plan_factorization(2449029, 128, [126, 140, 140], [4, 4, 8], [1, 8, 8, 1])
    idx = synth.zipf_ids(5, 20000, 1.1, cfg.num_nodes)
    got = oracle.prefix_counts(cfg, idx)
    want = [len(set(idx // (140 * 140))), len(set(idx // 140)), len(set(idx))]
    assert got == want


def test_multithreaded_matches_single():
    cfg = plan_factorization(2449029, 128, [126, 140, 140], [4, 4, 8], [1, 8, 8, 1])
    cores = rand_cores(cfg, 12, 0.1)
    idx = synth.zipf_ids(6, 300, 1.1, cfg.num_nodes)
    up = synth.normal(6, 2, 300 * 128, 1.0, np.float64).reshape(300, 128)
    o1, _ = oracle.lookup_batch(cfg, cores, idx, 1)
    o4, _ = oracle.lookup_batch(cfg, cores, idx, 4)
    np.testing.assert_array_equal(o1, o4)
    g1, _ = oracle.backward_lookup(cfg, cores, idx, up, 1)
    g4, _ = oracle.backward_lookup(cfg, cores, idx, up, 4)
    for a, b in zip(g1, g4):
        np.testing.assert_allclose(a, b, rtol=1e-12, atol=1e-12)
