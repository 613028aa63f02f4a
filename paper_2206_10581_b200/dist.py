"""Data parallelism over the index batch: one process per GPU,
cores replicated, the batch sharded by position, and exactly one exchange
step -- a sum all-reduce (NCCL over NVLink/NVSwitch via torch.distributed) of
the single contiguous gradient buffer between backward and update.

The buffer holds every core's gradient in the engine's device layout
([m_k][R_{k-1}][n_k][R_k]) followed by one touch counter per core slice, so
the same all-reduce yields the global gradient and the union of the slices
any rank touched; the update then runs on that union (exactly the dense
SGD/Adagrad update, see kernels_update.cuh).  The host-side helpers below
(shard bounds, buffer layout) are shared with the CPU gloo tests.
"""
from __future__ import annotations

from typing import List, Sequence

import numpy as np

from .config import TTConfig


def shard_bounds(B: int, rank: int, world: int):
    """Contiguous position shard [lo, hi) of a global batch of B."""
    return B * rank // world, B * (rank + 1) // world


def grad_buffer_len(cfg: TTConfig) -> int:
    return sum(cfg.core_size(k) for k in range(cfg.d)) + sum(cfg.m)


def pack_grad_buffer(cfg: TTConfig, grads: Sequence[np.ndarray], touched: Sequence[np.ndarray],
                     dtype=np.float64) -> np.ndarray:
    """Reference-layout gradients (R,m,n,R) + per-slice touch counts -> the
    engine's flat buffer layout."""
    parts: List[np.ndarray] = []
    for k in range(cfg.d):
        g = np.asarray(grads[k], dtype).reshape(cfg.core_shape(k))
        parts.append(np.ascontiguousarray(g.transpose(1, 0, 2, 3)).ravel())  # -> [m][R][n][R]
    parts += [np.asarray(t, dtype).ravel() for t in touched]
    return np.concatenate(parts)


def unpack_grad_buffer(cfg: TTConfig, buf: np.ndarray):
    grads, off = [], 0
    for k in range(cfg.d):
        R0, m, n, R1 = cfg.core_shape(k)
        g = buf[off: off + cfg.core_size(k)].reshape(m, R0, n, R1).transpose(1, 0, 2, 3)
        grads.append(np.ascontiguousarray(g))
        off += cfg.core_size(k)
    touched = []
    for k in range(cfg.d):
        touched.append(buf[off: off + cfg.m[k]].copy())
        off += cfg.m[k]
    return grads, touched


def touch_counts(cfg: TTConfig, idx: np.ndarray) -> List[np.ndarray]:
    """Per core k, the number of distinct prefixes (i_1..i_{k+1}) of the batch
    whose digit i_{k+1} equals v (what the engine writes as touch counters)."""
    idx = np.unique(np.asarray(idx, np.int64))
    out = []
    suffix = [int(np.prod(cfg.m[k + 1:])) for k in range(cfg.d)]
    for k in range(cfg.d):
        prefixes = np.unique(idx // suffix[k])
        out.append(np.bincount(prefixes % cfg.m[k], minlength=cfg.m[k]).astype(np.float64))
    return out


class DataParallelTT:
    """Wraps a TTEmbedding for one rank of a torch.distributed job: binds the
    gradient buffer to a torch tensor, turns on dense gradients and
    all-reduces before every update."""

    def __init__(self, emb, group=None):
        import torch
        import torch.distributed as dist
        self.emb = emb
        self.group = group
        self.dist = dist
        n = grad_buffer_len(emb.config)
        self.buf = torch.zeros(n, dtype=torch.float32, device=f"cuda:{emb.device}")
        emb.bind_grad_buffer(self.buf)
        emb.set_dense_grads(True)

    def forward(self, indices, out=None):
        return self.emb.forward(indices, out)

    def backward(self, grad_out, indices=None):
        self.emb.backward(grad_out, indices)

    def allreduce(self):
        if self.dist.is_initialized() and self.dist.get_world_size() > 1:
            self.dist.all_reduce(self.buf, group=self.group)

    def step(self):
        self.allreduce()
        self.emb.step()
