"""BASELINE's full sizes on the device, through properties that do not need a
full oracle run (the oracle checks exactness at small sizes elsewhere):

* the plan is bit-exact against numpy's stable sort / unique at the full batch
  (262,144 IDs at papers; 1,048,576 at billion);
* forward rows at a random sample of positions match the oracle (1e-5 a_ref);
  every position of one ID carries the identical row; the extreme IDs 0 and
  num_nodes - 1 are served;
* the backward is linear at full size: g(2 u1 + u2) = 2 g(u1) + g(u2) within
  the fp32 condition-scaled bound."""
import numpy as np
import pytest

import oracle
from paper_2206_10581_b200 import config as C
from paper_2206_10581_b200 import synth

pytestmark = pytest.mark.gpu


def _abs(cores):
    return [np.abs(c.astype(np.float64)) for c in cores]


@pytest.mark.parametrize("name,path", [("papers", "auto"), ("papers", "tc"), ("billion", "auto"), ("billion", "tc")])
def test_full_batch_plan_and_sampled_rows(name, path):
    import torch
    from paper_2206_10581_b200 import engine as E
    cfg, idx, _, cores = C.workload_inputs(name, 2026) if name == "papers" else (None, None, None, None)
    if name == "billion":  # the bench's ID stream without the 1 GB upstream
        cfg = C.WORKLOADS[name]["cfg"]()
        w = C.WORKLOADS[name]
        idx = synth.zipf_ids(2026, w["batch"], w["alpha"], cfg.num_nodes)
        cores = synth.gaussian_cores(cfg, 2026, 0.1)
    idx = idx.copy()
    idx[:3] = [0, cfg.num_nodes - 1, 0]  # extremes, and a duplicate of position 0
    emb = E.TTEmbedding(cfg)
    emb.set_cores(cores)
    emb.set_path(path)
    out = emb.forward(torch.tensor(idx, device="cuda"))
    emb.sync()
    keys, pos = emb.plan_sorted()
    perm = np.argsort(idx, kind="stable")
    np.testing.assert_array_equal(pos, perm)
    np.testing.assert_array_equal(keys, idx[perm])
    assert emb.plan_stats()[-1] == len(np.unique(idx))
    rng = np.random.default_rng(1)
    sample = np.concatenate([[0, 1, 2], rng.choice(len(idx), 253, replace=False)])
    got = out[torch.tensor(sample, device="cuda")].cpu().numpy()
    c64 = [c.astype(np.float64) for c in cores]
    ref, bad = oracle.lookup_batch(cfg, c64, idx[sample])
    aref, _ = oracle.lookup_batch(cfg, _abs(cores), idx[sample])
    assert bad == -1
    assert np.all(np.abs(got - ref) <= 1e-5 * aref + 1e-30)
    np.testing.assert_array_equal(got[0], got[2])  # duplicates: identical rows
    # every position of the most frequent ID carries the same row
    vals, counts = np.unique(idx, return_counts=True)
    hot = np.flatnonzero(idx == vals[np.argmax(counts)])[:64]
    rows = out[torch.tensor(hot, device="cuda")].cpu().numpy()
    assert np.all(rows == rows[0])


@pytest.mark.parametrize("path", ["auto", "tc"])
def test_full_batch_backward_linearity(path):
    import torch
    from paper_2206_10581_b200 import engine as E
    cfg, idx, up1, cores = C.workload_inputs("papers", 2026)
    up2 = synth.normal(77, 3, up1.size).reshape(up1.shape)
    emb = E.TTEmbedding(cfg)
    emb.set_cores(cores)
    emb.set_path(path)
    ti = torch.tensor(idx, device="cuda")
    grads = []
    for up in (up1, up2, 2.0 * up1 + up2):
        emb.forward(ti)
        emb.backward(torch.tensor(np.ascontiguousarray(up, np.float32), device="cuda"))
        emb.sync()
        grads.append(emb._fetch_grads())
    # bound: per entry, the same contraction on |G| and |u| (2|u1| + |u2|) times fp32 noise
    for k in range(cfg.d):
        lhs, rhs = grads[2][k], 2.0 * grads[0][k] + grads[1][k]
        scale = 2.0 * np.abs(grads[0][k]) + np.abs(grads[1][k]) + np.abs(grads[2][k])
        err = np.abs(lhs - rhs)
        # entries of a sum over many rows: allow 1e-4 of the magnitudes involved
        # plus an absolute floor for cancelling entries
        assert np.all(err <= 1e-4 * scale + 1e-3), f"core {k}: {float(np.max(err - 1e-4 * scale))}"


# ---------------------------------------------------------------------------
# Full-batch backward and update against the oracle.  The engine runs the
# whole BASELINE batch (so the plan, the digit grouping, the FB_NB multi-batch
# node loop -- billion: 1,567 level-F nodes in one group --, the FB_IDS > 512
# digit-staging fallback -- sweep: up to 978 distinct IDs per 256-node batch --
# and the heavy-ID paths all run at full size), with the upstream gradient
# zeroed outside a seeded sample of positions.  Rows with a zero upstream add
# exactly 0 to every gradient entry, so the result must equal the oracle's
# gradient over the sampled rows alone (autodiff.cpp:48-118), and the updated
# cores the oracle's update with that gradient (autodiff.cpp:147-173).
FULL_CASES = [("papers", "auto", 3000), ("papers", "tc", 3000), ("billion", "auto", 2000),
              ("billion", "tc", 2000), ("sweep64", "auto", 3000), ("sweep64", "tc", 3000),
              ("sweep16", "auto", 3000), ("sweep128", "auto", 1500), ("sweep128", "tc", 1500)]


def _full_inputs(name):
    cfg = C.WORKLOADS[name]["cfg"]()
    w = C.WORKLOADS[name]
    if w["dist"] == "zipf":
        idx = synth.zipf_ids(2026, w["batch"], w["alpha"], cfg.num_nodes)
    elif w["dist"] == "uniform":
        idx = synth.uniform_ids(2026, w["batch"], cfg.num_nodes)
    else:
        idx = synth.locality_ids(2026, w["batch"], cfg.num_nodes, w["block"])
    return cfg, idx, synth.gaussian_cores(cfg, 2026, 0.1)


@pytest.mark.parametrize("name,path,S", FULL_CASES)
def test_full_batch_backward_and_update_vs_oracle(name, path, S):
    import torch
    from paper_2206_10581_b200 import engine as E
    cfg, idx, cores = _full_inputs(name)
    B = len(idx)
    rng = np.random.default_rng(7)
    sample = np.sort(rng.choice(B, S, replace=False))
    up_s = synth.normal(99, 5, S * cfg.emb_dim).reshape(S, cfg.emb_dim)
    emb = E.TTEmbedding(cfg)
    emb.set_cores(cores)
    emb.set_path(path)
    kind = C.WORKLOADS[name]["opt"]
    lr = 0.01
    opt = E.OptimizerState.make(cfg, getattr(E.OptKind, kind), lr)
    emb.configure_optimizer(opt)
    up = torch.zeros((B, cfg.emb_dim), dtype=torch.float32, device="cuda")
    up[torch.tensor(sample, device="cuda")] = torch.tensor(up_s, device="cuda")
    emb.forward(torch.tensor(idx, device="cuda"))
    if path == "tc":
        assert emb.last_path() == "fused-tc"
    else:
        assert emb.last_path() == "fused"
    emb.backward(up)
    emb.sync()
    got = emb._fetch_grads()
    emb.step()
    emb.sync()
    new = emb.get_cores(np.float64)

    c64 = [c.astype(np.float64) for c in cores]
    gref, bad = oracle.backward_lookup(cfg, c64, idx[sample], up_s, 0)
    assert bad == -1
    aref, _ = oracle.backward_lookup(cfg, _abs(cores), idx[sample], np.abs(up_s.astype(np.float64)), 0)
    for k in range(cfg.d):
        err = np.abs(got[k] - gref[k])
        worst = float(np.max(err / (1e-5 * aref[k] + 1e-30)))
        assert worst <= 1.0, f"{name}/{path} dG_{k}: max err/(1e-5 a_ref) = {worst:.3g}"
        assert np.all(got[k][aref[k] == 0] == 0.0)  # slices only zero-upstream rows touch: exactly 0
    p64 = [c.copy() for c in c64]
    ost = oracle.OptState(cfg, {"sgd": oracle.SGD, "adagrad": oracle.ADAGRAD}[kind], lr)
    assert oracle.apply_update(cfg, p64, gref, ost) == -1
    assert emb.opt_step() == ost.step == 1
    excluded = 0
    for k in range(cfg.d):
        if kind == "adagrad":
            # step 1 is lr g/(|g| + eps): entries with |g_ref| below the fp32
            # noise of the gradient are sign-ambiguous -- excluded, counted
            amb = np.abs(gref[k]) < 1e-5 * aref[k]
            excluded += int(np.count_nonzero(amb & (aref[k] > 0)))
            ok = ~amb
            err = np.abs(new[k] - p64[k])[ok]
            bound = (lr * 1e-5 * aref[k] / np.maximum(np.abs(gref[k]), 1e-30))[ok] * 4 + 1e-6 * np.abs(p64[k])[ok] + 1e-9
        else:
            err = np.abs(new[k] - p64[k]).ravel()
            bound = (lr * 1e-5 * aref[k] + 1e-7 * np.abs(p64[k]) + 1e-12).ravel()
        assert np.all(err <= bound), f"{name}/{path} updated core {k}: {float(np.max(err - bound)):.3g} over"
    print(f"{name}/{path}: B={B} sample={S} adagrad sign-ambiguous entries excluded: {excluded}")
