"""In-tree build of the CUDA engine (sm_100a) into paper_2206_10581_b200/libtt_b200.so."""
from __future__ import annotations

import os
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libtt_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
         "-Xcompiler", "-fPIC,-O2", "-shared", "-Xptxas", "-v"]


def sources():
    return sorted(os.path.join(SRC, f) for f in os.listdir(SRC) if f.endswith((".cu", ".cuh")))


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    hdr = os.path.join(os.path.dirname(PKG), "include", "tt_engine.h")
    return any(os.path.getmtime(s) > t for s in sources() + [hdr])


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not stale():
        return LIB
    extra = os.environ.get("TT_NVCC_EXTRA", "").split()  # diagnostics only, e.g. -DTT_BWD3_TRACE
    out = os.environ.get("TT_BUILD_OUT", LIB)  # A/B variants (with TT_NVCC_EXTRA=-D...) go elsewhere
    cmd = [NVCC, *FLAGS, *extra, "-o", out, os.path.join(SRC, "engine.cu"), "-ldl"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    log = os.path.join(PKG, "build.log")
    with open(log, "w") as f:
        f.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed ({r.returncode}); see {log}\n{r.stderr[-4000:]}")
    if verbose:
        print(r.stderr)
    return LIB


if __name__ == "__main__":
    build(force=True)
    print(LIB)
