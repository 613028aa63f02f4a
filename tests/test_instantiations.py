"""Every compiled kernel instantiation has a GPU parity case (CPU check).

The fused FFMA kernels are compiled for a fixed list of (K, BN, RP, NL)
tuples (TT_FUSED_SHAPES, csrc/kernels_fused.cuh) and the tcgen05 kernels for
TT_TC_SHAPES (csrc/kernels_tcgen05.cuh).  This test parses both lists and
restates the host's shape admission (fused_plan_shape / wide_shape /
tc_plan_shape) for every config in tests/test_gpu_parity.py SHAPES, and
fails if a compiled tuple is reached by none of them -- i.e. if a kernel
could produce a bench line without ever being compared with the oracle.
"""
import os
import re

from test_gpu_parity import FUSED_SHAPES, SHAPES, TC_SHAPES

CSRC = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2206_10581_b200", "csrc")


def _macro_tuples(fname, macro):
    src = open(os.path.join(CSRC, fname)).read()
    m = re.search(r"#define\s+" + macro + r"\(X\)((?:[^\n]*\\\n)*[^\n]*)", src)
    assert m, f"{macro} not found in {fname}"
    return {tuple(int(v) for v in t) for t in re.findall(r"X\((\d+),\s*(\d+),\s*(\d+),\s*(\d+)\)", m.group(1))}


def _block(K, NC, wide=False):
    """Column block of the backward (fused_plan_shape / wide_shape)."""
    if K == 8 and NC % 32 == 0 and not wide:
        return 32
    if K == 16 and NC % 64 == 0:
        return 64
    if K in (32, 64) and NC % 128 == 0:
        return 128
    if K == 128:
        if wide and NC % 128 == 0:
            return 128
        if not wide and NC % 64 == 0:
            return 64
    if not wide and K in (32, 64) and NC % K == 0:
        return K
    return 0


def reached(cfg):
    """(FFMA tuples, tcgen05 tuples) the engine launches for cfg."""
    d = cfg.d
    m, n, R = cfg.m, cfg.n, cfg.R
    rows = [1] * d
    for k in range(1, d):
        rows[k] = rows[k - 1] * n[k - 1]
    cols = [n[k] * R[k + 1] for k in range(d)]
    ffma, tc = set(), set()
    if d < 3:
        return ffma, tc
    F = d - 2
    K, NC, RP, NL = R[F], cols[F], rows[F], n[d - 1]
    BN = _block(K, NC)
    if R[F + 1] != K or not BN:
        return ffma, tc
    BNf = 128 if (K == 128 and NC % 128 == 0) else min(BN, 128)
    ffma |= {(K, BN, RP, NL), (K, BNf, RP, NL)}
    if K in (32, 64) and NC % 128 == 0:
        tc.add((K, 128, RP, NL))
    if K == 128 and NC % 64 == 0:
        tc.add((RP, NL))  # k_tc_bwd128 (TT_TC128_SHAPES)
    for k in range(1, F):  # wide levels on the fused kernels
        Kw, NCw, RPw = R[k], cols[k], rows[k]
        BNw = _block(Kw, NCw, wide=True)
        if BNw and RPw <= 64 and 64 % RPw == 0 and R[k + 1] == Kw:
            ffma.add((Kw, BNw, RPw, "*"))
    return ffma, tc


def test_every_ffma_instantiation_has_a_parity_case():
    compiled = _macro_tuples("kernels_fused.cuh", "TT_FUSED_SHAPES")
    assert len(compiled) >= 9
    covered = set()
    for name in FUSED_SHAPES:
        ffma, _ = reached(SHAPES[name][0]())
        covered |= ffma
    exact = {t for t in covered if t[3] != "*"}
    missing = sorted(t for t in compiled if t not in exact)
    assert not missing, f"compiled FFMA instantiations with no parity case: {missing}"


def test_every_fwd8_instantiation_has_a_parity_case():
    src = open(os.path.join(CSRC, "kernels_fused.cuh")).read()
    m = re.search(r"#define\s+TT_FWD8_SHAPES\(X\)([^\n]*)", src)
    compiled = {tuple(int(v) for v in t) for t in re.findall(r"X\((\d+),\s*(\d+)\)", m.group(1))}
    covered = set()
    for name in FUSED_SHAPES:
        ffma, _ = reached(SHAPES[name][0]())
        covered |= {(t[0], t[2]) for t in ffma if t[1] == 128}
    missing = sorted(t for t in compiled if t not in covered)
    assert not missing, f"compiled 8x8-tile forward instantiations with no parity case: {missing}"


def test_every_bwdk32_instantiation_has_a_parity_case():
    src = open(os.path.join(CSRC, "kernels_fused.cuh")).read()
    m = re.search(r"#define\s+TT_BWDK32_SHAPES\(X\)([^\n]*)", src)
    compiled = {tuple(int(v) for v in t) for t in re.findall(r"X\((\d+),\s*(\d+)\)", m.group(1))}
    covered = set()
    for name in FUSED_SHAPES:
        ffma, _ = reached(SHAPES[name][0]())
        covered |= {(t[2], t[3]) for t in ffma if t[0] == 32 and t[1] == 128 and t[3] != "*"}
    missing = sorted(t for t in compiled if t not in covered)
    assert not missing, f"compiled rank-32 backward instantiations with no parity case: {missing}"


def test_every_lowrank_backward_instantiation_has_a_parity_case():
    # k_lowrank_bwd<K, RP, NL, CPL> (TT_LOWRANK_SHAPES): one column block of NC = 32 CPL
    src = open(os.path.join(CSRC, "kernels_fused.cuh")).read()
    m = re.search(r"#define\s+TT_LOWRANK_SHAPES\(X\)([^\n]*)", src)
    compiled = {tuple(int(v) for v in t) for t in re.findall(r"X\((\d+),\s*(\d+),\s*(\d+),\s*(\d+)\)", m.group(1))}
    assert compiled
    covered = set()
    for name in FUSED_SHAPES:
        ffma, _ = reached(SHAPES[name][0]())
        covered |= {(t[0], t[2], t[3], t[1] // 32) for t in ffma if t[0] <= 16 and t[3] != "*" and t[1] % 32 == 0}
    missing = sorted(t for t in compiled if t not in covered)
    assert not missing, f"compiled low-rank backward instantiations with no parity case: {missing}"


def test_every_lowrank_forward_instantiation_has_a_parity_case():
    # k_lowrank_fwd<K, RP, NL, CPL> (TT_LOWRANK_FWD_SHAPES): one block of NC = 32 CPL columns
    src = open(os.path.join(CSRC, "kernels_fused.cuh")).read()
    m = re.search(r"#define\s+TT_LOWRANK_FWD_SHAPES\(X\)([^\n]*)", src)
    compiled = {tuple(int(v) for v in t) for t in re.findall(r"X\((\d+),\s*(\d+),\s*(\d+),\s*(\d+)\)", m.group(1))}
    assert compiled
    covered = set()
    for name in FUSED_SHAPES:
        ffma, _ = reached(SHAPES[name][0]())
        covered |= {(t[0], t[2], t[3], t[1] // 32) for t in ffma if t[0] <= 16 and t[1] % 32 == 0 and t[3] != "*"}
    missing = sorted(t for t in compiled if t not in covered)
    assert not missing, f"compiled low-rank forward instantiations with no parity case: {missing}"


def test_every_rank128_tcgen05_instantiation_has_a_parity_case():
    src = open(os.path.join(CSRC, "kernels_tcgen05.cuh")).read()
    m = re.search(r"#define\s+TT_TC128_SHAPES\(X\)([^\n]*)", src)
    compiled = {tuple(int(v) for v in t) for t in re.findall(r"X\((\d+),\s*(\d+)\)", m.group(1))}
    covered = set()
    for name in TC_SHAPES:
        _, tc = reached(SHAPES[name][0]())
        covered |= {t for t in tc if len(t) == 2}
    missing = sorted(t for t in compiled if t not in covered)
    assert not missing, f"compiled rank-128 tcgen05 instantiations with no parity case: {missing}"


def test_every_tcgen05_instantiation_has_a_parity_case():
    compiled = _macro_tuples("kernels_tcgen05.cuh", "TT_TC_SHAPES")
    covered = set()
    for name in TC_SHAPES:
        _, tc = reached(SHAPES[name][0]())
        assert tc, f"{name} is listed as a tensor-core parity shape but admits no tcgen05 kernel"
        covered |= {t for t in tc if len(t) == 4}
    missing = sorted(t for t in compiled if t not in covered)
    assert not missing, f"compiled tcgen05 instantiations with no parity case: {missing}"


def test_every_baseline_workload_is_a_parity_case():
    from paper_2206_10581_b200.config import WORKLOADS
    for w in WORKLOADS:
        assert w in SHAPES and w in FUSED_SHAPES, f"BASELINE workload {w} has no fused parity case"
