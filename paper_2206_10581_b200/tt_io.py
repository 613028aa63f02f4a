"""TTE1 core files and training checkpoints.

`save_tt` / `load_tt` follow the reference's format (tt_io.hpp:20-35,
tt_io.cpp:48-124):

* magic "TTE1";
* u32 d;
* per core the u32 (m_k, n_k, R_{k-1}, R_k);
* the cores in order as little-endian f64, row-major over (R_{k-1}, m_k, n_k, R_k);
* a JSON sidecar `path + ".json"` holding num_nodes, emb_dim, row_factors,
  col_factors and ranks. Without it, load falls back to the padded dimensions.

Errors follow the reference's std::runtime_error messages ("not a TTE1 core
file", "core file truncated in header", "implausible core count",
"R_0 != 1", "inconsistent ranks between cores", "R_d != 1",
"truncated core data").

`save_checkpoint` / `load_checkpoint` add what the reference lacks (resume,
SPEC.md:102). They write the TTE1 file of a device-resident TTEmbedding plus a
"TTO1" optimizer file next to it (`path + ".opt"`):

* magic "TTO1";
* u32 kind, u32 has_s1, u32 has_s2;
* f64 lr, beta1, beta2, eps;
* i64 step;
* then s1 and s2, in the core layout above (f64).

A checkpointed engine resumes bit-exactly.
"""
from __future__ import annotations

import json
import os
import struct
from typing import List, Sequence, Tuple

import numpy as np

from .config import TTConfig, plan_factorization

MAGIC = b"TTE1"
OPT_MAGIC = b"TTO1"


class CoreFileError(RuntimeError):
    """std::runtime_error of the reference's core-file reader/writer."""


def _core_shapes(cfg: TTConfig):
    return [cfg.core_shape(k) for k in range(cfg.d)]


def save_tt(cfg: TTConfig, cores: Sequence[np.ndarray], path: str) -> None:
    """save_tt (tt_io.cpp:48-80) for host cores in the reference layout."""
    cfg.validate()
    shapes = _core_shapes(cfg)
    arrs = []
    for k, c in enumerate(cores):
        a = np.ascontiguousarray(c, dtype="<f8")
        if tuple(a.shape) != tuple(shapes[k]):
            raise CoreFileError(f"core {k} has shape {a.shape}, expected {shapes[k]}")
        arrs.append(a)
    try:
        with open(path, "wb") as f:
            f.write(MAGIC)
            f.write(struct.pack("<I", cfg.d))
            for (r0, m, n, r1) in shapes:
                f.write(struct.pack("<4I", m, n, r0, r1))
            for a in arrs:
                f.write(a.tobytes())
    except OSError as e:
        raise CoreFileError(f"cannot open {path} for writing") from e
    side = {"num_nodes": cfg.num_nodes, "emb_dim": cfg.emb_dim, "row_factors": list(cfg.m),
            "col_factors": list(cfg.n), "ranks": list(cfg.R)}
    try:
        with open(path + ".json", "w") as js:
            js.write(json.dumps(side, indent=2) + "\n")
    except OSError as e:
        raise CoreFileError(f"cannot open {path}.json for writing") from e


def _u32(f) -> int:
    b = f.read(4)
    if len(b) != 4:
        raise CoreFileError("core file truncated in header")
    return struct.unpack("<I", b)[0]


def load_tt(path: str) -> Tuple[TTConfig, List[np.ndarray]]:
    """load_tt (tt_io.cpp:82-124): (config, cores f64 in the reference layout)."""
    try:
        f = open(path, "rb")
    except OSError as e:
        raise CoreFileError(f"cannot open {path}") from e
    with f:
        if f.read(4) != MAGIC:
            raise CoreFileError(f"{path}: not a TTE1 core file")
        d = _u32(f)
        if d < 2 or d > 64:
            raise CoreFileError(f"{path}: implausible core count")
        m, n, R = [], [], [1] * (d + 1)
        for k in range(d):
            mk, nk, rp, rn = _u32(f), _u32(f), _u32(f), _u32(f)
            if k == 0 and rp != 1:
                raise CoreFileError(f"{path}: R_0 != 1")
            if k > 0 and rp != R[k]:
                raise CoreFileError(f"{path}: inconsistent ranks between cores")
            m.append(mk)
            n.append(nk)
            R[k + 1] = rn
        if R[-1] != 1:
            raise CoreFileError(f"{path}: R_d != 1")
        num_nodes, emb_dim = int(np.prod(m)), int(np.prod(n))  # padded fallback
        if os.path.exists(path + ".json"):
            with open(path + ".json") as js:
                side = json.load(js)
            num_nodes, emb_dim = int(side["num_nodes"]), int(side["emb_dim"])
        cfg = plan_factorization(num_nodes, emb_dim, m, n, R)
        cores = []
        for k in range(d):
            shape = cfg.core_shape(k)
            cnt = int(np.prod(shape))
            raw = f.read(cnt * 8)
            if len(raw) != cnt * 8:
                raise CoreFileError(f"{path}: truncated core data")
            cores.append(np.frombuffer(raw, dtype="<f8").reshape(shape).copy())
    return cfg, cores


def save_checkpoint(emb, path: str) -> None:
    """Cores (TTE1) + optimizer state (TTO1, path + '.opt') of a device TTEmbedding."""
    from .engine import OptimizerState
    cfg = emb.config
    save_tt(cfg, emb.get_cores(np.float64), path)
    opt = emb._opt if emb._opt is not None else OptimizerState(kind=0)
    s1, s2, step = emb.get_opt_state()
    with open(path + ".opt", "wb") as f:
        f.write(OPT_MAGIC)
        f.write(struct.pack("<3I", opt.kind, s1 is not None, s2 is not None))
        f.write(struct.pack("<4d", opt.learning_rate, opt.beta1, opt.beta2, opt.epsilon))
        f.write(struct.pack("<q", step))
        for arrs in (s1, s2):
            if arrs is not None:
                for a in arrs:
                    f.write(np.ascontiguousarray(a, dtype="<f8").tobytes())


def load_checkpoint(path: str, device: int = 0):
    """A device TTEmbedding with the checkpoint's cores, optimizer and step."""
    from .engine import OptimizerState, TTEmbedding
    cfg, cores = load_tt(path)
    emb = TTEmbedding(cfg, device)
    emb.set_cores(cores)
    with open(path + ".opt", "rb") as f:
        if f.read(4) != OPT_MAGIC:
            raise CoreFileError(f"{path}.opt: not a TTO1 optimizer file")
        kind, has1, has2 = struct.unpack("<3I", f.read(12))
        lr, b1, b2, eps = struct.unpack("<4d", f.read(32))
        (step,) = struct.unpack("<q", f.read(8))
        opt = OptimizerState(kind=kind, learning_rate=lr, beta1=b1, beta2=b2, epsilon=eps)
        emb.configure_optimizer(opt)

        def read_state():
            out = []
            for k in range(cfg.d):
                shape = cfg.core_shape(k)
                cnt = int(np.prod(shape))
                raw = f.read(cnt * 8)
                if len(raw) != cnt * 8:
                    raise CoreFileError(f"{path}.opt: truncated optimizer state")
                out.append(np.frombuffer(raw, dtype="<f8").reshape(shape))
            return out

        s1 = read_state() if has1 else None
        s2 = read_state() if has2 else None
    emb.set_opt_state(s1, s2, step)
    return emb
