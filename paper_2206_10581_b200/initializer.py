"""Core initializers (initializer.hpp:54-69).

* `init_gaussian(cfg, seed, std)`: i.i.d. N(0, std^2) cores
  (initializer.cpp:91-101). The reference draws them from std::mt19937_64 +
  std::normal_distribution, which is not portable, so the seeded portable
  generator (synth.gaussian_cores) stands in. Every BASELINE config is
  initialised this way.
* `init_ortho_core(cfg, seed, target_scale=None, device=0)`: the ortho-core
  init (initializer.cpp:103-132), computed on the GPU in fp64
  (tt_ortho_cores_f64, csrc/kernels_init.cuh). Core k's n_k R_{k-1} slice
  vectors are orthonormal (length m_k R_k), so the materialised table is
  semi-orthogonal (W^T W = alpha I, the paper's Claim 1). It returns fp64
  cores in the reference layout, like the reference's TTEmbedding; set them
  into an engine with TTEmbedding.set_cores.
"""
from __future__ import annotations

import ctypes as C
from typing import List, Optional

import numpy as np

from . import synth
from .config import InvalidArgument, TTConfig


class InfeasibleRanksError(InvalidArgument):
    """InfeasibleRanksError (initializer.hpp): core k needs more orthonormal
    vectors (n_k R_{k-1}) than their length (m_k R_k) allows."""

    def __init__(self, core: int, needed: int, available: int):
        super().__init__(f"ortho-core init infeasible at core {core}: needs {needed} orthonormal vectors of length "
                         f"{available} (require n_k*R_{{k-1}} <= m_k*R_k)")
        self.core_index, self.num_vectors, self.vector_dim = core, needed, available


def init_gaussian(cfg: TTConfig, seed: int, std: float) -> List[np.ndarray]:
    if std < 0:
        raise InvalidArgument("gaussian_std must be nonnegative")
    return [c.astype(np.float64) for c in synth.gaussian_cores(cfg, seed, std)]


def init_ortho_core(cfg: TTConfig, seed: int, target_scale: Optional[float] = None,
                    device: int = 0) -> List[np.ndarray]:
    from .engine import _raise, load_library, to_cconfig
    cfg.validate()
    if target_scale is not None and target_scale <= 0.0:
        raise InvalidArgument("target_scale must be positive")
    lib = load_library()
    cores = [np.zeros(cfg.core_shape(k), np.float64) for k in range(cfg.d)]
    ptrs = (C.c_void_p * cfg.d)(*[c.ctypes.data for c in cores])
    bad = np.full(3, -1, np.int64)
    cc = to_cconfig(cfg)
    rc = lib.tt_ortho_cores_f64(C.byref(cc), device, int(seed) & 0xFFFFFFFFFFFFFFFF,
                                float(target_scale or 0.0), ptrs, bad.ctypes.data)
    if rc != 0 and bad[0] >= 0:
        raise InfeasibleRanksError(int(bad[0]), int(bad[1]), int(bad[2]))
    _raise(rc, "tt_ortho_cores_f64")
    return cores
