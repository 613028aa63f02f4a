"""Pins the oracle's (and the host mirror's) index arithmetic bit-exactly
against the reference's OWN tt_config.cpp, compiled in place into
oracle/_ref/libttref.so by oracle/Makefile.  Skipped where the reference is
not present (e.g. the GPU box); the committed golden fixtures under
tests/golden/ carry the same pins there."""
import numpy as np
import pytest

import oracle
from paper_2206_10581_b200 import config as C
from paper_2206_10581_b200 import synth

pytestmark = pytest.mark.skipif(oracle.ref() is None, reason="oracle/_ref not built (no /root/reference)")

CFGS = [
    C.plan_factorization(48, 8, [3, 4, 4], [2, 2, 2], [1, 2, 2, 1]),
    C.WORKLOADS["small"]["cfg"](),
    C.WORKLOADS["products"]["cfg"](),
    C.WORKLOADS["papers"]["cfg"](),
    C.WORKLOADS["billion"]["cfg"](),
    C.plan_factorization(99 * 101, 4, [99, 101], [2, 2], [1, 3, 1]),
    C.plan_factorization(7 * 3 * 9 * 11, 4, [7, 3, 9, 11], [1, 2, 2, 1], [1, 2, 2, 2, 1]),
]


@pytest.mark.parametrize("cfg", CFGS, ids=lambda c: "x".join(map(str, c.m)))
def test_digits_bit_exact_vs_reference(cfg):
    rows = np.concatenate([np.arange(min(cfg.padded_rows(), 2000)),
                           synth.bounded(1, 1, 20000, min(cfg.padded_rows(), 1 << 32))])
    want, bad = oracle.ref_digits(cfg, rows)
    assert bad == -1
    got = np.array([oracle.index_to_coordinate(cfg, int(r)) for r in rows[:3000]])
    np.testing.assert_array_equal(got, want[:3000])
    host = np.array([C.index_to_coordinate(cfg, int(r)) for r in rows[:3000]])
    np.testing.assert_array_equal(host, want[:3000])
    # out of range exactly at prod(m)
    _, bad = oracle.ref_digits(cfg, [0, cfg.padded_rows()])
    assert bad == 1 and oracle.index_to_coordinate(cfg, cfg.padded_rows()) is None


@pytest.mark.parametrize("cfg", CFGS, ids=lambda c: "x".join(map(str, c.m)))
def test_count_params_vs_reference(cfg):
    assert oracle.count_params(cfg) == oracle.ref_count_params(cfg) == C.count_params(cfg)


def test_validate_vs_reference():
    bad = [C.TTConfig(8, 8, [2, 2, 2], [2, 2, 2], [2, 2, 2, 2]),
           C.TTConfig(9, 8, [2, 2, 2], [2, 2, 2], [1, 2, 2, 1]),
           C.TTConfig(8, 9, [2, 2, 2], [2, 2, 2], [1, 2, 2, 1]),
           C.TTConfig(8, 8, [2, 2, 2], [2, 2, 2], [1, 0, 2, 1]),
           C.TTConfig(8, 8, [8], [8], [1, 1])]
    for cfg in bad + CFGS:
        want = oracle.ref_validate(cfg)
        assert (oracle.validate(cfg) != 0) == (want != 0)
        try:
            cfg.validate()
            host = 0
        except C.InvalidArgument:
            host = 1
        assert host == want


@pytest.mark.parametrize("M,N,d", [(169363, 128, 3), (8, 8, 3), (2449029, 100, 3), (1000, 64, 2),
                                   (97, 10, 3), (100000, 256, 4)])
def test_auto_planner_vs_reference(M, N, d):
    R = [1] + [4] * (d - 1) + [1]
    for ortho in (True, False):
        want = oracle.ref_plan_auto(M, N, d, R, ortho)
        cfg = C.plan_factorization(M, N, d, R, ortho_friendly=ortho)
        assert (cfg.m, cfg.n) == (want[0], want[1])
