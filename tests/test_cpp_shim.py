"""A C++ host on the C-ABI (include/tt_engine.hpp, tests/cpp/shim_test.cpp).

The reference is C++ and its training loop calls lookup_batch /
backward_lookup / OptimizerState::make / apply_update (gnn.cpp:89-128,
313-411).  This compiles a C++ program against include/tt_engine.hpp and
libtt_b200.so (CPU test: the header compiles and every call links), and on
the GPU runs it on the golden fixture (small, SGD) and on a products-shaped
batch (the fused path, Adagrad): its rows, CoreGradients and updated cores
are compared with the oracle, its exceptions are checked inside the program
(std::out_of_range with the first bad position, std::invalid_argument for a
shape mismatch and for a non-finite gradient with cores and step untouched),
and one step on an engine with a 1-rank NCCL communicator (device path +
tt_allreduce_grads) must equal the host-path step bit for bit."""
import os
import subprocess

import numpy as np
import pytest

import oracle
from paper_2206_10581_b200 import _build
from paper_2206_10581_b200 import config as C
from paper_2206_10581_b200 import synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "shim_test.cpp")
BIN = os.path.join(ROOT, "tests", "cpp", "shim_test")
CUDA = "/usr/local/cuda"


def build_shim():
    _build.build()  # no-op when the library is current
    libdir = os.path.dirname(_build.LIB)
    cmd = ["g++", "-std=c++17", "-O1", "-Wall", "-I", os.path.join(ROOT, "include"), "-I", f"{CUDA}/include",
           SRC, "-o", BIN, f"-L{libdir}", "-ltt_b200", f"-L{CUDA}/lib64", "-lcudart",
           f"-Wl,-rpath,{libdir}:{CUDA}/lib64"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-3000:]
    return BIN


def test_cpp_shim_compiles_and_links():
    assert os.path.exists(build_shim())
    out = subprocess.run(["nm", "-u", BIN], capture_output=True, text=True).stdout
    for sym in ("tt_engine_create", "tt_lookup_batch", "tt_backward_lookup", "tt_apply_update",
                "tt_comm_init_rank", "tt_allreduce_grads", "tt_opt_init"):
        assert sym in out


def _write_case(d, cfg, cores, idx, up):
    with open(os.path.join(d, "cfg.txt"), "w") as f:
        f.write(f"{cfg.num_nodes} {cfg.emb_dim} {cfg.d}\n")
        f.write(" ".join(map(str, cfg.m)) + "\n" + " ".join(map(str, cfg.n)) + "\n" + " ".join(map(str, cfg.R)) + "\n")
    for k, c in enumerate(cores):
        np.ascontiguousarray(c, np.float64).tofile(os.path.join(d, f"core{k}.f64"))
    np.ascontiguousarray(idx, np.int64).tofile(os.path.join(d, "idx.i64"))
    np.ascontiguousarray(up, np.float32).tofile(os.path.join(d, "up.f32"))


def _cases():
    from test_golden import load_case
    cfg, z, idx, up, cores = load_case("small")
    yield "golden-small", cfg, idx, up, cores, z
    cfg = C.WORKLOADS["products"]["cfg"]()
    idx = synth.zipf_ids(5, 2048, 1.1, cfg.num_nodes)
    up = synth.normal(6, 1, 2048 * cfg.emb_dim).reshape(2048, cfg.emb_dim)
    yield "products", cfg, idx, up, synth.gaussian_cores(cfg, 7), None


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["golden-small", "products"])
def test_cpp_shim_against_oracle(tmp_path, case):
    name, cfg, idx, up, cores, z = next(c for c in _cases() if c[0] == case)
    build_shim()
    d = str(tmp_path)
    _write_case(d, cfg, cores, idx, up)
    r = subprocess.run([BIN, d], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    B = len(idx)
    rows = np.fromfile(os.path.join(d, "rows.f32"), np.float32).reshape(B, cfg.emb_dim)
    c64 = [c.astype(np.float64) for c in cores]
    ref, _ = oracle.lookup_batch(cfg, c64, idx, 0)
    aref, _ = oracle.lookup_batch(cfg, [np.abs(c) for c in c64], idx, 0)
    assert np.all(np.abs(rows - ref) <= 1e-5 * aref + 1e-30)
    if z is not None:  # the committed golden rows (first 48 positions)
        n = z["out"].shape[0]
        assert np.all(np.abs(rows[:n] - z["out"]) <= 1e-5 * z["out_abs"] + 1e-30)
    gref, _ = oracle.backward_lookup(cfg, c64, idx, up, 0)
    garef, _ = oracle.backward_lookup(cfg, [np.abs(c) for c in c64], idx, np.abs(up.astype(np.float64)), 0)
    g = [np.fromfile(os.path.join(d, f"grad{k}.f64")).reshape(cfg.core_shape(k)) for k in range(cfg.d)]
    for k in range(cfg.d):
        assert np.all(np.abs(g[k] - gref[k]) <= 1e-5 * garef[k] + 1e-30), f"grad {k}"
        if z is not None:
            assert np.all(np.abs(g[k] - z[f"grad{k}"]) <= 1e-5 * z[f"grad_abs{k}"] + 1e-30)
    # Adagrad step 1 on the engine's own gradient g (fp32): the oracle's update
    p64 = [c.copy() for c in c64]
    ost = oracle.OptState(cfg, oracle.ADAGRAD, 0.01)
    g32 = [x.astype(np.float32).astype(np.float64) for x in g]
    assert oracle.apply_update(cfg, p64, g32, ost) == -1
    for k in range(cfg.d):
        got = np.fromfile(os.path.join(d, f"adagrad{k}.f64")).reshape(cfg.core_shape(k))
        assert np.all(np.abs(got - p64[k]) <= 1e-6 * (np.abs(p64[k]) + 0.01)), f"adagrad core {k}"
        comm = np.fromfile(os.path.join(d, f"comm{k}.f64")).reshape(cfg.core_shape(k))
        np.testing.assert_array_equal(comm, got)  # 1-rank all-reduce path == host path, bitwise
