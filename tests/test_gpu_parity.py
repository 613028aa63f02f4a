"""GPU parity: the CUDA engine (through the C-ABI) against the C oracle on
identical seeded inputs.

Tolerances (BASELINE.json north_star):
* digits, sort permutation, unique IDs and per-level prefix counts: bit-exact;
* embeddings, core gradients, updated cores: |x - x_ref| <= 1e-5 * a_ref, where
  x_ref is the fp64 oracle on the same fp32 inputs and a_ref the same
  contraction on absolute values (|G|, |U|) -- a condition-scaled relative
  bound; the naive max elementwise relative error is reported alongside;
* Adagrad step 1 is sign-sensitive (lr g/(|g|+eps)): the update kernel is
  checked on the oracle's own gradient, and end to end entries with
  |g_ref| < 1e-5 a_ref are excluded and counted.
"""
import numpy as np
import pytest

import oracle
from paper_2206_10581_b200 import config as C
from paper_2206_10581_b200 import synth

pytestmark = pytest.mark.gpu

TOL = 1e-5


def eng():
    from paper_2206_10581_b200 import engine
    return engine


def make(cfg, seed, path="auto", std=0.1):
    e = eng()
    cores = synth.gaussian_cores(cfg, seed, std)
    emb = e.TTEmbedding(cfg)
    emb.set_cores(cores)
    emb.set_path(path)
    return emb, cores


def ids_for(cfg, seed, B, dist="zipf"):
    if dist == "zipf":
        return synth.zipf_ids(seed, B, 1.1, cfg.num_nodes)
    if dist == "uniform":
        return synth.uniform_ids(seed, B, cfg.num_nodes)
    return synth.locality_ids(seed, B, cfg.num_nodes, cfg.m[-1] * cfg.m[-2], run=64)


def abs_cores(cores):
    return [np.abs(c.astype(np.float64)) for c in cores]


def check_close(x, ref, aref, what):
    x = np.asarray(x, np.float64)
    err = np.abs(x - ref)
    bound = TOL * aref + 1e-30
    worst = float(np.max(err / bound)) if err.size else 0.0
    naive = float(np.max(err / np.maximum(np.abs(ref), 1e-30))) if err.size else 0.0
    assert worst <= 1.0, f"{what}: max err/(1e-5 a_ref) = {worst:.3g} (naive rel {naive:.3g})"
    return worst, naive


SHAPES = {
    "tiny": (lambda: C.plan_factorization(12, 8, [2, 3, 2], [2, 2, 2], [1, 3, 2, 1]), 40, "uniform"),
    "d2": (lambda: C.plan_factorization(99 * 101, 4, [99, 101], [2, 2], [1, 3, 1]), 300, "uniform"),
    "small": (lambda: C.WORKLOADS["small"]["cfg"](), 2048, "uniform"),
    "products": (lambda: C.WORKLOADS["products"]["cfg"](), 2048, "zipf"),
    "papers": (lambda: C.WORKLOADS["papers"]["cfg"](), 1024, "zipf"),
    "sweep8": (lambda: C.WORKLOADS["sweep8"]["cfg"](), 2048, "locality"),
    "sweep16": (lambda: C.WORKLOADS["sweep16"]["cfg"](), 2048, "locality"),
    "sweep32": (lambda: C.WORKLOADS["sweep32"]["cfg"](), 2048, "locality"),
    "sweep64": (lambda: C.WORKLOADS["sweep64"]["cfg"](), 1024, "locality"),
    "sweep128": (lambda: C.WORKLOADS["sweep128"]["cfg"](), 512, "locality"),
    "billion": (lambda: C.WORKLOADS["billion"]["cfg"](), 512, "zipf"),
    "ragged": (lambda: C.plan_factorization(1000, 30, [7, 11, 13], [2, 3, 5], [1, 5, 3, 1]), 700, "zipf"),
    # the paper's Table 4: ogbn-arxiv (55,55,56)/(8,4,4) and
    # ogbn-papers100M (480,500,500)/(8,4,4) at R = 32 and 64
    "arxivT4_r32": (lambda: C.plan_factorization(169_363, 128, [55, 55, 56], [8, 4, 4], [1, 32, 32, 1]), 1024, "uniform"),
    "papersT4_r64": (lambda: C.plan_factorization(111_059_956, 128, [480, 500, 500], [8, 4, 4], [1, 64, 64, 1]), 1024,
                     "zipf"),
    # emb_dim < prod(n): rows truncated (tt_embedding.cpp:122), upstream zero-padded
    # (autodiff.cpp:96-97) on the fused path
    "papers_trunc": (lambda: C.plan_factorization(111_059_956, 120, [480, 481, 482], [4, 8, 4], [1, 64, 64, 1]), 1024,
                     "zipf"),
    # ogbn-products (125,140,140)/(4,5,5), dim 100: n_d = 5, NC = 5R
    "productsT4_r32": (lambda: C.plan_factorization(2_449_029, 100, [125, 140, 140], [4, 5, 5], [1, 32, 32, 1]), 2048,
                       "zipf"),
    "productsT4_r64": (lambda: C.plan_factorization(2_449_029, 100, [125, 140, 140], [4, 5, 5], [1, 64, 64, 1]), 1024,
                       "zipf"),
}


# shapes the fused FFMA kernels cover (every BASELINE shape; the tiny, d2 and
# ragged test shapes run the generic path).  tests/test_instantiations.py
# checks that every compiled (K, BN, RP, NL) instantiation is reached by one
# of these.
FUSED_SHAPES = {"small", "products", "papers", "sweep8", "sweep16", "sweep32", "sweep64", "sweep128", "billion",
                "arxivT4_r32", "papersT4_r64", "productsT4_r32", "productsT4_r64", "papers_trunc"}

# shapes with tcgen05 kernels (rank >= 32)
TC_SHAPES = ("products", "papers", "billion", "sweep32", "sweep64", "sweep128", "papers_trunc")


@pytest.mark.parametrize("name", list(SHAPES))
def test_plan_bit_exact(name):
    mk, B, dist = SHAPES[name]
    cfg = mk()
    emb, _ = make(cfg, 1)
    idx = ids_for(cfg, 2, B, dist)
    out = emb.forward(__import__("torch").tensor(idx, device="cuda"))
    del out
    keys, pos = emb.plan_sorted()
    perm, uniq = oracle.sort_unique(idx)
    np.testing.assert_array_equal(pos, perm)
    np.testing.assert_array_equal(keys, idx[perm])
    ids, dig = emb.plan_digits()
    np.testing.assert_array_equal(ids, uniq)
    want = np.array([oracle.index_to_coordinate(cfg, int(i)) for i in uniq])
    np.testing.assert_array_equal(dig, want)
    assert emb.plan_stats() == oracle.prefix_counts(cfg, idx)


@pytest.mark.parametrize("path", ["generic", "auto", "tc"])
@pytest.mark.parametrize("name", list(SHAPES))
def test_forward_parity(name, path):
    import torch
    mk, B, dist = SHAPES[name]
    cfg = mk()
    emb, cores = make(cfg, 3, path)
    idx = ids_for(cfg, 4, B, dist)
    out = emb.forward(torch.tensor(idx, device="cuda")).cpu().numpy()
    emb.sync()
    if path == "tc" and name in TC_SHAPES:
        assert emb.last_path() == "fused-tc"  # the tcgen05 kernels ran, not the FFMA ones
    if path == "auto" and name in FUSED_SHAPES:
        assert emb.last_path() == "fused"  # a BASELINE shape never falls back to the generic path
    ref, bad = oracle.lookup_batch(cfg, cores, idx, 0)
    aref, _ = oracle.lookup_batch(cfg, abs_cores(cores), idx, 0)
    assert bad == -1
    check_close(out, ref, aref, f"{name}/{path} forward")
    # duplicates identical, batch == single-row lookups bitwise
    dup = np.flatnonzero(idx == idx[0])
    assert all(np.array_equal(out[dup[0]], out[j]) for j in dup)
    e = eng()
    one = e.lookup_batch(emb, idx[:3])
    np.testing.assert_array_equal(one, out[:3])


@pytest.mark.parametrize("path", ["generic", "auto", "tc"])
@pytest.mark.parametrize("name", list(SHAPES))
def test_backward_parity(name, path):
    import torch
    mk, B, dist = SHAPES[name]
    cfg = mk()
    emb, cores = make(cfg, 5, path)
    idx = ids_for(cfg, 6, B, dist)
    up = synth.normal(7, 1, B * cfg.emb_dim).reshape(B, cfg.emb_dim)
    ti, tu = torch.tensor(idx, device="cuda"), torch.tensor(up, device="cuda")
    emb.forward(ti)
    emb.backward(tu)  # saved plan
    emb.sync()
    g_saved = emb._fetch_grads()
    e = eng()
    g = e.backward_lookup(emb, idx, up)  # full recompute, host buffers
    assert g.batch_count == B
    ref, bad = oracle.backward_lookup(cfg, cores, idx, up, 0)
    aref, _ = oracle.backward_lookup(cfg, abs_cores(cores), idx, np.abs(up.astype(np.float64)), 0)
    assert bad == -1
    for k in range(cfg.d):
        np.testing.assert_array_equal(g_saved[k], g.grads[k])
        check_close(g.grads[k], ref[k], aref[k], f"{name}/{path} dG_{k}")
        assert np.all(g.grads[k][aref[k] == 0] == 0.0)  # untouched slices exactly 0


@pytest.mark.parametrize("name", ["tiny", "small", "products", "papers", "billion"])
@pytest.mark.parametrize("kind", ["sgd", "adagrad", "adam"])
def test_update_kernel_on_oracle_gradient(name, kind):
    e = eng()
    mk, B, dist = SHAPES[name]
    cfg = mk()
    emb, cores = make(cfg, 8)
    idx = ids_for(cfg, 9, B, dist)
    up = synth.normal(10, 1, B * cfg.emb_dim).reshape(B, cfg.emb_dim)
    gref, _ = oracle.backward_lookup(cfg, cores, idx, up, 0)
    gref32 = [g.astype(np.float32).astype(np.float64) for g in gref]
    kid = {"sgd": oracle.SGD, "adagrad": oracle.ADAGRAD, "adam": oracle.ADAM}[kind]
    lr = 0.01
    opt = e.OptimizerState.make(cfg, getattr(e.OptKind, kind), lr)
    ost = oracle.OptState(cfg, kid, lr)
    p64 = [c.astype(np.float64).copy() for c in cores]
    for it in range(2):
        e.apply_update(emb, e.CoreGradients(gref32, B), opt)
        assert oracle.apply_update(cfg, p64, gref32, ost) == -1
    assert opt.step == ost.step == 2
    got = emb.get_cores(np.float64)
    for k in range(cfg.d):
        scale = np.abs(p64[k]) + lr * 2
        err = np.abs(got[k] - p64[k]) / scale
        assert float(err.max()) <= 1e-5, f"{kind} core {k}: {err.max():.3g}"


@pytest.mark.parametrize("name", ["small", "products", "papers", "billion"])
def test_train_step_end_to_end(name):
    """forward -> backward(saved) -> step on the device path vs the oracle."""
    import torch
    e = eng()
    mk, B, dist = SHAPES[name]
    cfg = mk()
    kind = C.WORKLOADS[name]["opt"]
    emb, cores = make(cfg, 11)
    idx = ids_for(cfg, 12, B, dist)
    up = synth.normal(13, 1, B * cfg.emb_dim).reshape(B, cfg.emb_dim)
    opt = e.OptimizerState.make(cfg, getattr(e.OptKind, kind), 0.01)
    emb.configure_optimizer(opt)
    emb.forward(torch.tensor(idx, device="cuda"))
    emb.backward(torch.tensor(up, device="cuda"))
    emb.step()
    emb.sync()
    got = emb.get_cores(np.float64)
    gref, _ = oracle.backward_lookup(cfg, cores, idx, up, 0)
    aref, _ = oracle.backward_lookup(cfg, abs_cores(cores), idx, np.abs(up.astype(np.float64)), 0)
    p64 = [c.astype(np.float64).copy() for c in cores]
    ost = oracle.OptState(cfg, {"sgd": oracle.SGD, "adagrad": oracle.ADAGRAD}[kind], 0.01)
    oracle.apply_update(cfg, p64, gref, ost)
    excluded = 0
    for k in range(cfg.d):
        if kind == "adagrad":
            amb = np.abs(gref[k]) < TOL * aref[k]
            excluded += int(np.count_nonzero(amb & (aref[k] > 0)))
            ok = ~amb
            # |dp| <= lr * |dg| / |g|-ish: bound the update error by the gradient's
            err = np.abs(got[k] - p64[k])[ok]
            bound = (0.01 * TOL * aref[k] / np.maximum(np.abs(gref[k]), 1e-30))[ok] * 4 + 1e-6 * np.abs(p64[k])[ok] + 1e-9
            assert np.all(err <= bound), f"core {k}"
        else:
            err = np.abs(got[k] - p64[k])
            assert np.all(err <= 0.01 * TOL * aref[k] + 1e-7 * np.abs(p64[k]) + 1e-12), f"core {k}"
    print(f"{name}: adagrad sign-ambiguous entries excluded: {excluded}")


def test_index_errors_fail_whole_batch():
    import torch
    e = eng()
    cfg = SHAPES["tiny"][0]()
    emb, cores = make(cfg, 14)
    with pytest.raises(C.OutOfRange, match="position 2") as ei:
        e.lookup_batch(emb, [0, 1, 99])
    assert ei.value.position == 2 and ei.value.value == 99
    with pytest.raises(C.OutOfRange, match="position 1"):
        e.lookup_batch(emb, [0, -5, 12, 3])
    # device path: no row written, error deferred to sync
    out = torch.full((3, 8), 7.0, device="cuda")
    emb.forward(torch.tensor([0, 12, 13], device="cuda"), out)
    with pytest.raises(C.OutOfRange, match="position 1"):
        emb.sync()
    assert bool((out == 7.0).all())
    with pytest.raises(C.OutOfRange):
        e.backward_lookup(emb, [0, 12], np.zeros((2, 8), np.float32))
    with pytest.raises(C.InvalidArgument):
        e.backward_lookup(emb, [0, 1], np.zeros((3, 8), np.float32))
    with pytest.raises(C.InvalidArgument):
        e.backward_lookup(emb, [0, 1], np.zeros((2, 7), np.float32))
    # the engine stays usable
    np.testing.assert_array_equal(e.lookup_batch(emb, [3])[0], e.lookup_batch(emb, [3, 4])[0])


def test_nonfinite_rejected_state_untouched():
    e = eng()
    cfg = C.plan_factorization(4, 4, [2, 2], [2, 2], [1, 2, 1])
    emb, cores = make(cfg, 15, std=1.0)
    before = emb.get_cores(np.float64)
    opt = e.OptimizerState.make(cfg, e.OptKind.adam, 1e-3)
    g = e.CoreGradients.zeros(cfg)
    g.grads[1].reshape(-1)[0] = np.nan
    with pytest.raises(C.InvalidArgument, match="core 1"):
        e.apply_update(emb, g, opt)
    assert opt.step == 0
    for a, b in zip(before, emb.get_cores(np.float64)):
        np.testing.assert_array_equal(a, b)
    g.grads[1].reshape(-1)[0] = np.inf
    with pytest.raises(C.InvalidArgument):
        e.apply_update(emb, g, opt)
    g.grads[1].reshape(-1)[0] = 0.0
    e.apply_update(emb, g, opt)
    assert opt.step == 1


def test_empty_batch_and_zero_upstream():
    e = eng()
    cfg = SHAPES["tiny"][0]()
    emb, _ = make(cfg, 16)
    assert e.lookup_batch(emb, []).shape == (0, 8)
    g = e.backward_lookup(emb, [0, 5, 11], np.zeros((3, 8), np.float32))
    assert g.batch_count == 3 and all(np.all(x == 0) for x in g.grads)
    opt = e.OptimizerState.make(cfg, e.OptKind.sgd, 1e-3)
    before = emb.get_cores(np.float64)
    e.apply_update(emb, g, opt)
    assert opt.step == 1
    for a, b in zip(before, emb.get_cores(np.float64)):
        np.testing.assert_array_equal(a, b)


@pytest.mark.parametrize("path", ["generic", "auto"])
def test_linearity_and_additivity(path):
    e = eng()
    cfg = SHAPES["products"][0]()
    emb, cores = make(cfg, 17, path)
    idx = ids_for(cfg, 18, 256, "zipf")
    u = synth.normal(19, 1, 256 * 128).reshape(256, 128)
    v = synth.normal(19, 2, 256 * 128).reshape(256, 128)
    gu = [x.copy() for x in e.backward_lookup(emb, idx, u).grads]
    gv = [x.copy() for x in e.backward_lookup(emb, idx, v).grads]
    gm = e.backward_lookup(emb, idx, (0.5 * u - 2.0 * v).astype(np.float32)).grads
    au, _ = oracle.backward_lookup(cfg, abs_cores(cores), idx, np.abs(u) + np.abs(v), 0)
    for k in range(3):
        check_close(gm[k], 0.5 * gu[k] - 2.0 * gv[k], 3 * au[k], f"linearity core {k}")
    g1 = [x.copy() for x in e.backward_lookup(emb, [6], u[:1]).grads]
    g2 = e.backward_lookup(emb, [6, 6], np.vstack([u[:1], u[:1]])).grads
    for k in range(3):
        np.testing.assert_allclose(g2[k], 2.0 * g1[k], rtol=1e-6, atol=1e-12)


def test_200_sgd_steps_fit():  # test_autodiff.cpp:237-256 on the device
    e = eng()
    cfg = C.plan_factorization(32, 8, [2, 4, 4], [2, 2, 2], [1, 4, 4, 1])
    truth = [synth.normal(10, 100 + k, cfg.core_size(k), 0.5, np.float64) for k in range(3)]
    allidx = np.arange(32)
    target, _ = oracle.lookup_batch(cfg, truth, allidx)
    emb, _ = make(cfg, 11, std=0.3)
    opt = e.OptimizerState.make(cfg, e.OptKind.sgd, 0.05)

    def loss():
        return 0.5 * float(np.sum((e.lookup_batch(emb, allidx) - target) ** 2))

    initial = loss()
    for _ in range(200):
        out = e.lookup_batch(emb, allidx)
        e.apply_update(emb, e.backward_lookup(emb, allidx, (out - target).astype(np.float32)), opt)
    assert loss() <= initial / 100.0
    assert opt.step == 200


def test_lr_schedule_keeps_optimizer_state():
    """apply_update reads opt.learning_rate on every call (autodiff.cpp:147-173):
    changing it on the same state object must not reset the Adagrad/Adam
    moments or the step."""
    e = eng()
    cfg = SHAPES["products"][0]()
    for kind, kid in (("adagrad", oracle.ADAGRAD), ("adam", oracle.ADAM)):
        emb, cores = make(cfg, 23)
        opt = e.OptimizerState.make(cfg, getattr(e.OptKind, kind), 0.01)
        ost = oracle.OptState(cfg, kid, 0.01)
        p64 = [c.astype(np.float64).copy() for c in cores]
        for it, lr in enumerate((0.01, 0.005, 0.0025)):
            idx = ids_for(cfg, 30 + it, 512, "zipf")
            up = synth.normal(40 + it, 1, 512 * cfg.emb_dim).reshape(512, cfg.emb_dim)
            gref, _ = oracle.backward_lookup(cfg, cores, idx, up, 0)
            g32 = [g.astype(np.float32).astype(np.float64) for g in gref]
            opt.learning_rate = lr
            ost.lr = lr
            e.apply_update(emb, e.CoreGradients(g32, 512), opt)
            assert oracle.apply_update(cfg, p64, g32, ost) == -1
        assert opt.step == ost.step == 3
        got = emb.get_cores(np.float64)
        for k in range(cfg.d):
            err = np.abs(got[k] - p64[k]) / (np.abs(p64[k]) + 0.03)
            assert float(err.max()) <= 1e-5, f"{kind} core {k}: {err.max():.3g}"


def test_forward_rejects_bad_out_buffer():
    import torch
    cfg = SHAPES["tiny"][0]()
    emb, _ = make(cfg, 24)
    idx = torch.tensor([0, 1, 2], device="cuda")
    for bad in (torch.empty((3, 8), dtype=torch.float64, device="cuda"),
                torch.empty((2, 8), device="cuda"),
                torch.empty((8, 3), device="cuda").t(),
                torch.empty((3, 8))):
        with pytest.raises(C.InvalidArgument):
            emb.forward(idx, bad)
    with pytest.raises(C.InvalidArgument):
        emb.forward(idx.cpu())


@pytest.mark.parametrize("path", ["auto", "tc"])
def test_second_backward_of_one_forward(path):
    # the tensor backward writes dC over the saved P_F blocks (k_fused_wdc): a
    # second backward of the same forward recomputes P_F first, and matches
    # the first bitwise (a different upstream in between)
    import torch
    mk, B, dist = SHAPES["papers"]
    cfg = mk()
    emb, cores = make(cfg, 41, path)
    idx = ids_for(cfg, 42, B, dist)
    up = synth.normal(43, 1, B * cfg.emb_dim).reshape(B, cfg.emb_dim)
    up2 = synth.normal(43, 2, B * cfg.emb_dim).reshape(B, cfg.emb_dim)
    ti, tu, tu2 = (torch.tensor(x, device="cuda") for x in (idx, up, up2))
    emb.forward(ti)
    emb.backward(tu)
    emb.sync()
    g1 = [x.copy() for x in emb._fetch_grads()]
    emb.backward(tu2)
    emb.backward(tu)
    emb.sync()
    g2 = emb._fetch_grads()
    for k in range(cfg.d):
        np.testing.assert_array_equal(g1[k], g2[k])


def test_forward_parity_with_fused_last_level():
    # k_fused_fwd8<..., LL> (TT_FWD_LL=1, off by default: measured slower) writes
    # the output rows from the forward's tile epilogue; same parity bound
    import os
    import subprocess
    import sys
    env = dict(os.environ, TT_FWD_LL="1")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider", __file__,
                        "-k", "test_forward_parity and papers and auto"], env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
