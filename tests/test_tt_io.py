"""TTE1 core files (tt_io.hpp:20-35): the reference's own test cases
(proj/tests/test_tt_io.cpp) restated, plus malformed-file rejections."""
import struct

import numpy as np
import pytest

from paper_2206_10581_b200 import config as C
from paper_2206_10581_b200 import synth
from paper_2206_10581_b200.tt_io import CoreFileError, load_tt, save_tt


def _random_cores(cfg, seed):
    return [synth.normal(seed, k, cfg.core_size(k), 1.0, np.float64).reshape(cfg.core_shape(k)) for k in range(cfg.d)]


def test_round_trip_is_bit_exact(tmp_path):  # test_tt_io.cpp "core file round trip is bit exact"
    cfg = C.plan_factorization(12, 6, [2, 3, 2], [2, 3, 1], [1, 3, 2, 1])
    cores = _random_cores(cfg, 2024)
    p = str(tmp_path / "rt.tte")
    save_tt(cfg, cores, p)
    cfg2, cores2 = load_tt(p)
    assert cfg2 == cfg
    for a, b in zip(cores, cores2):
        assert a.tobytes() == b.tobytes()


def test_header_layout_is_little_endian_sequence(tmp_path):  # "header layout is the documented ..."
    cfg = C.plan_factorization(4, 4, [2, 2], [2, 2], [1, 3, 1])
    cores = [np.zeros(cfg.core_shape(k)) for k in range(cfg.d)]
    p = str(tmp_path / "h.tte")
    save_tt(cfg, cores, p)
    head = open(p, "rb").read(4 + 4 + 2 * 16)
    assert head[:4] == b"TTE1"
    u = struct.unpack("<9I", head[4:])
    assert u == (2, 2, 2, 1, 3, 2, 2, 3, 1)  # d; (m, n, R_prev, R_next) per core


def test_without_sidecar_falls_back_to_padded(tmp_path):  # "loading without the sidecar ..."
    cfg = C.plan_factorization(7, 3, [4, 2], [2, 2], [1, 2, 1])
    cores = _random_cores(cfg, 9)
    p = tmp_path / "ns.tte"
    save_tt(cfg, cores, str(p))
    (tmp_path / "ns.tte.json").unlink()
    cfg2, cores2 = load_tt(str(p))
    assert cfg2.num_nodes == 8 and cfg2.emb_dim == 4
    for a, b in zip(cores, cores2):
        np.testing.assert_array_equal(a, b)


def test_wrong_magic_rejected(tmp_path):  # "a wrong magic is rejected"
    p = tmp_path / "bad.tte"
    p.write_bytes(b"NOPE")
    with pytest.raises(CoreFileError, match="TTE1"):
        load_tt(str(p))


@pytest.mark.parametrize("cut,msg", [(6, "truncated in header"), (40, "truncated core data")])
def test_truncated_files_rejected(tmp_path, cut, msg):
    cfg = C.plan_factorization(4, 4, [2, 2], [2, 2], [1, 3, 1])
    p = tmp_path / "t.tte"
    save_tt(cfg, _random_cores(cfg, 1), str(p))
    p.write_bytes(p.read_bytes()[:cut])
    with pytest.raises(CoreFileError, match=msg):
        load_tt(str(p))


def test_inconsistent_ranks_rejected(tmp_path):
    p = tmp_path / "r.tte"
    p.write_bytes(b"TTE1" + struct.pack("<9I", 2, 2, 2, 1, 3, 2, 2, 4, 1))
    with pytest.raises(CoreFileError, match="inconsistent ranks"):
        load_tt(str(p))


def test_workload_config_round_trip(tmp_path):
    cfg = C.WORKLOADS["products"]["cfg"]()
    cores = [c.astype(np.float64) for c in synth.gaussian_cores(cfg, 4)]
    p = str(tmp_path / "w.tte")
    save_tt(cfg, cores, p)
    cfg2, cores2 = load_tt(p)
    assert cfg2 == cfg
    for a, b in zip(cores, cores2):
        np.testing.assert_array_equal(a, b)
