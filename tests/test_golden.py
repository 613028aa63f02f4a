"""Golden fixtures (tests/golden/, made by make_golden.py from the reference's
own tt_config.cpp and the pinned oracle): the CPU oracle and the host mirror
must reproduce them (CPU tests), and the CUDA engine must match them on the
GPU (gpu tests) -- the pins travel to the GPU box this way."""
import os

import numpy as np
import pytest

import oracle
from paper_2206_10581_b200 import config as C
from paper_2206_10581_b200 import synth

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
REF = np.load(os.path.join(HERE, "ref_digits.npz"))
NAMES = sorted({k[:-7] for k in REF.files if k.endswith("_digits")})
FWD = {"tiny": (C.plan_factorization(12, 8, [2, 3, 2], [2, 2, 2], [1, 3, 2, 1]),),
       "sweep8": (C.WORKLOADS["sweep8"]["cfg"](),),
       "small": (C.WORKLOADS["small"]["cfg"](),)}


def cfg_of(name):
    return C.TTConfig(int(REF[f"{name}_M"]), int(REF[f"{name}_N"]), [int(x) for x in REF[f"{name}_m"]],
                      [int(x) for x in REF[f"{name}_n"]], [int(x) for x in REF[f"{name}_R"]])


def load_case(name):
    z = np.load(os.path.join(HERE, f"fwd_bwd_{name}.npz"))
    cfg = FWD[name][0]
    seed, B, dist = int(z["seed"]), int(z["B"]), str(z["dist"])
    idx = synth.uniform_ids(seed, B, cfg.num_nodes) if dist == "uniform" else synth.zipf_ids(seed, B, 1.1, cfg.num_nodes)
    up = synth.normal(seed, 7, B * cfg.emb_dim).reshape(B, cfg.emb_dim)
    cores = synth.gaussian_cores(cfg, seed, 0.1)
    assert synth.checksum(idx) == str(z["idx_sum"])
    assert synth.checksum(up) == str(z["up_sum"])
    assert synth.checksum(np.concatenate([c.ravel() for c in cores])) == str(z["cores_sum"])
    return cfg, z, idx, up, cores


@pytest.mark.parametrize("name", NAMES)
def test_reference_digits_golden(name):
    cfg = cfg_of(name)
    rows, want = REF[f"{name}_rows"], REF[f"{name}_digits"]
    for r, w in zip(rows, want):
        assert oracle.index_to_coordinate(cfg, int(r)) == list(w)
        assert C.index_to_coordinate(cfg, int(r)) == list(w)
    assert oracle.count_params(cfg) == int(REF[f"{name}_params"]) == C.count_params(cfg)


def test_reference_planner_golden():
    for k in REF.files:
        if not k.startswith("plan_"):
            continue
        _, M, N, d = k.split("_")
        M, N, d = int(M), int(N), int(d)
        cfg = C.plan_factorization(M, N, d, [1] + [4] * (d - 1) + [1])
        assert cfg.m + cfg.n == [int(x) for x in REF[k]]


@pytest.mark.parametrize("name", list(FWD))
def test_oracle_reproduces_golden(name):
    cfg, z, idx, up, cores = load_case(name)
    c64 = [c.astype(np.float64) for c in cores]
    y, _ = oracle.lookup_batch(cfg, c64, idx)
    np.testing.assert_array_equal(y, z["out"])
    g, _ = oracle.backward_lookup(cfg, c64, idx, up)
    for k in range(cfg.d):
        np.testing.assert_array_equal(g[k], z[f"grad{k}"])


@pytest.mark.gpu
@pytest.mark.parametrize("path", ["generic", "auto"])
@pytest.mark.parametrize("name", list(FWD))
def test_engine_matches_golden(name, path):
    from paper_2206_10581_b200 import engine as E
    cfg, z, idx, up, cores = load_case(name)
    emb = E.TTEmbedding(cfg)
    emb.set_cores(cores)
    emb.set_path(path)
    out = E.lookup_batch(emb, idx)
    assert np.all(np.abs(out - z["out"]) <= 1e-5 * z["out_abs"] + 1e-30)
    g = E.backward_lookup(emb, idx, up).grads
    for k in range(cfg.d):
        assert np.all(np.abs(g[k] - z[f"grad{k}"]) <= 1e-5 * z[f"grad_abs{k}"] + 1e-30)


@pytest.mark.gpu
@pytest.mark.parametrize("name", NAMES)
def test_engine_digits_golden(name):
    import torch
    from paper_2206_10581_b200 import engine as E
    cfg = cfg_of(name)
    rows = REF[f"{name}_rows"]
    rows = rows[rows < cfg.num_nodes]
    emb = E.TTEmbedding(cfg)
    emb.forward(torch.tensor(rows, device="cuda"))
    emb.sync()
    ids, dig = emb.plan_digits()
    want = {int(r): list(w) for r, w in zip(REF[f"{name}_rows"], REF[f"{name}_digits"])}
    for i, dgt in zip(ids, dig):
        assert list(dgt) == want[int(i)]
