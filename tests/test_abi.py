"""CPU-side checks of the C-ABI boundary: the library builds/loads, exports
every symbol include/tt_engine.h declares, and its host-only entry points
(config validation, parameter counting) agree with the oracle.  No compute
calls are made here (no GPU in this container)."""
import os
import re
import subprocess

import pytest

import oracle
from paper_2206_10581_b200 import config as C
from paper_2206_10581_b200 import engine, _build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "tt_engine.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(tt_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = engine.load_library()
    out = subprocess.run(["nm", "-D", "--defined-only", _build.LIB], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (tt_[a-z0-9_]+)", out))
    declared = header_symbols()
    assert declared, "no declarations parsed"
    missing = [s for s in declared if s not in exported]
    assert not missing, missing
    assert sorted(engine.SYMBOLS) == declared
    for s in declared:
        assert hasattr(lib, s)


def test_built_for_sm100a():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _build.LIB], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


@pytest.mark.parametrize("cfg", [C.WORKLOADS[w]["cfg"]() for w in ("small", "products", "papers", "billion")] +
                         [C.plan_factorization(12, 8, [2, 3, 2], [2, 2, 2], [1, 3, 2, 1])])
def test_count_params_matches_oracle(cfg):
    lib = engine.load_library()
    cc = engine.to_cconfig(cfg)
    assert lib.tt_config_validate(engine.C.byref(cc)) == 0
    assert lib.tt_count_params(engine.C.byref(cc)) == oracle.count_params(cfg)


def test_validate_rejects_like_reference():
    lib = engine.load_library()
    bad = [C.TTConfig(8, 8, [2, 2, 2], [2, 2, 2], [2, 2, 2, 2]),
           C.TTConfig(9, 8, [2, 2, 2], [2, 2, 2], [1, 2, 2, 1]),
           C.TTConfig(8, 9, [2, 2, 2], [2, 2, 2], [1, 2, 2, 1]),
           C.TTConfig(0, 8, [2, 2, 2], [2, 2, 2], [1, 2, 2, 1]),
           C.TTConfig(8, 8, [2, 2, 2], [2, 2, 2], [1, -1, 2, 1])]
    for cfg in bad:
        cc = engine.to_cconfig(cfg)
        assert lib.tt_config_validate(engine.C.byref(cc)) == engine.TT_ERR_ARG
        assert oracle.validate(cfg) != 0
        assert b"TTConfig" in lib.tt_last_error()
