"""Data parallelism over the index batch: one process per GPU.

Two schemes share the engine's single contiguous gradient buffer:

* position sharding (DataParallelTT): cores replicated, the batch sharded by
  position, and exactly one exchange step -- a sum all-reduce (NCCL over
  NVLink/NVSwitch via torch.distributed) of the whole buffer between backward
  and update.  Cross-shard duplicates of a prefix are computed on every rank
  that sees them (a ~5.3x ceiling at papers on 8 GPUs).
* ID-owner sharding (OwnerShardedTT): the level-F core (F = d-2, the core of
  the fused GEMMs -- 63 MB of the 64 MB at papers) is sharded by its digit
  i_{d-1}: rank r owns the digit range [v_r, v_{r+1}) and so every ID, every
  level-F prefix and every G_F slice with such a digit.  Each step routes the
  IDs and their upstream rows to their owners (all-to-all), every prefix is
  computed exactly once in the job, output rows travel back (all-to-all), and
  only the small replicated cores' gradients are all-reduced.  The owned G_F
  slices (and their optimizer state) are only ever read and updated by their
  owner, so they never cross NVLink.

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


def native_enabled() -> bool:
    """TT_DIST_NATIVE=0: torch.distributed collectives on the data plane even
    under NCCL (the engine's own communicator is the default)."""
    import os
    return os.environ.get("TT_DIST_NATIVE", "1") != "0"


def _native_init(emb, dist, rank: int, world: int) -> bool:
    """The engine's NCCL communicator over the torch process group; every rank
    agrees on the outcome, and on failure the wrappers keep the
    torch.distributed (NCCL) data plane."""
    import sys
    import torch
    ok = 1
    try:
        obj = [emb_nccl_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        emb.comm_init_rank(obj[0], rank, world)
    except Exception as e:  # noqa: BLE001 -- reported, then the torch data plane
        print(f"[tt] rank {rank}: engine NCCL communicator unavailable ({e}); torch.distributed data plane",
              file=sys.stderr)
        ok = 0
    flag = torch.tensor([ok], dtype=torch.int32, device=f"cuda:{emb.device}")
    dist.all_reduce(flag, op=dist.ReduceOp.MIN)
    return bool(flag.item())


class DataParallelTT:
    """Wraps a TTEmbedding for one rank of a torch.distributed job (position
    sharding).

    Under the NCCL backend the data plane is the engine's own: rank 0 draws an
    NCCL unique id (tt_nccl_unique_id), torch.distributed only ships those 128
    bytes to the other ranks (control plane), every engine creates its
    communicator (tt_comm_init_rank), and each step's gradient all-reduce is
    tt_allreduce_grads -- the level-F core's gradient is reduced as soon as
    the GEMM kernel that writes it ends, overlapping the rest of the backward.
    Under gloo (CPU tests) the gradient buffer is bound to a torch tensor and
    all-reduced by torch.distributed."""

    def __init__(self, emb, group=None):
        import torch
        import torch.distributed as dist
        self.emb = emb
        self.group = group
        self.dist = dist
        self.native = (dist.is_initialized() and dist.get_backend(group) == "nccl" and group is None
                       and native_enabled())
        if self.native:
            self.native = _native_init(emb, dist, dist.get_rank(), dist.get_world_size())
        if self.native:
            self.buf = None
            return
        n = grad_buffer_len(emb.config)
        self.buf = torch.zeros(n, dtype=torch.float32, device=f"cuda:{emb.device}")
        emb.bind_grad_buffer(self.buf)
        emb.set_dense_grads(True)

    def forward(self, indices, out=None):
        return self.emb.forward(indices, out)

    def backward(self, grad_out, indices=None):
        self.emb.backward(grad_out, indices)

    def allreduce(self):
        if self.native:
            self.emb.allreduce_grads()
        elif self.dist.is_initialized() and self.dist.get_world_size() > 1:
            self.dist.all_reduce(self.buf, group=self.group)

    def step(self):
        self.allreduce()
        self.emb.step()


def emb_nccl_id() -> bytes:
    from .engine import nccl_unique_id
    return nccl_unique_id()


# ---------------------------------------------------------------------------
# ID-owner sharding

def owner_bounds(cfg: TTConfig, world: int) -> List[int]:
    """Digit boundaries v_0 = 0 < ... < v_world = m_F of the level-F core
    (F = d-2; the first core when d = 2): rank r owns digits [v_r, v_{r+1})."""
    F = max(cfg.d - 2, 0)
    m = cfg.m[F]
    return [m * r // world for r in range(world + 1)]


def owner_of(cfg: TTConfig, idx, world: int):
    """Owner rank of every ID (torch int64 tensor, any device): the rank whose
    digit range holds the ID's level-F digit (tt_config.cpp:176-189 radix)."""
    import torch
    F = max(cfg.d - 2, 0)
    suffix = int(np.prod(cfg.m[F + 1:])) if F + 1 < cfg.d else 1
    digit = torch.div(idx, suffix, rounding_mode="floor") % cfg.m[F]
    b = torch.tensor(owner_bounds(cfg, world)[1:-1], dtype=torch.int64, device=idx.device)
    return torch.bucketize(digit, b, right=True)


class Route:
    """One all-to-all exchange plan: local positions sorted by owner rank."""

    def __init__(self, order, send_counts: List[int], recv_counts: List[int]):
        self.order, self.send_counts, self.recv_counts = order, send_counts, recv_counts


def _a2a(dist, out, inp, out_splits, in_splits, group):
    """all_to_all_single; under gloo (CPU collectives, smoke tests) CUDA
    tensors hop through host memory."""
    if inp.is_cuda and hasattr(dist, "get_backend") and dist.is_initialized() and dist.get_backend(group) == "gloo":
        o = out.cpu()
        dist.all_to_all_single(o, inp.cpu(), out_splits, in_splits, group=group)
        out.copy_(o)
    else:
        dist.all_to_all_single(out, inp, out_splits, in_splits, group=group)


def route_to_owners(cfg: TTConfig, idx, group=None, comm=None):
    """Send every local ID to its owner.  Returns (received IDs, Route).
    `comm` is torch.distributed (default) or an object with the same
    collective calls (tests)."""
    import torch
    dist = comm or __import__("torch.distributed", fromlist=["x"])
    world = dist.get_world_size(group)
    own = owner_of(cfg, idx, world)
    order = torch.argsort(own, stable=True)
    counts = torch.bincount(own, minlength=world)
    rc = torch.empty_like(counts)
    _a2a(dist, rc, counts, None, None, group)
    send, recv = counts.tolist(), rc.tolist()
    out = torch.empty(sum(recv), dtype=idx.dtype, device=idx.device)
    _a2a(dist, out, idx[order].contiguous(), recv, send, group)
    return out, Route(order, send, recv)


def route_rows(rows, r: Route, group=None, comm=None):
    """Local rows (one per local ID) -> the owners, in received-ID order."""
    import torch
    dist = comm or __import__("torch.distributed", fromlist=["x"])
    out = torch.empty((sum(r.recv_counts),) + tuple(rows.shape[1:]), dtype=rows.dtype, device=rows.device)
    _a2a(dist, out, rows[r.order].contiguous(), r.recv_counts, r.send_counts, group)
    return out


def route_back(rows, r: Route, out=None, group=None, comm=None):
    """Owner rows (received-ID order) -> back to the local positions."""
    import torch
    dist = comm or __import__("torch.distributed", fromlist=["x"])
    tmp = torch.empty((sum(r.send_counts),) + tuple(rows.shape[1:]), dtype=rows.dtype, device=rows.device)
    _a2a(dist, tmp, rows.contiguous(), r.send_counts, r.recv_counts, group)
    if out is None:
        out = torch.empty_like(tmp)
    out[r.order] = tmp
    return out


def replicated_segments(cfg: TTConfig) -> List[tuple]:
    """(offset, length) ranges of the gradient buffer that are all-reduced
    under owner sharding: every core but the sharded level-F core, and their
    touch counters (merged where adjacent)."""
    F = max(cfg.d - 2, 0)
    spans, off = [], 0
    sizes = [cfg.core_size(k) for k in range(cfg.d)]
    for k in range(cfg.d):
        if k != F:
            spans.append((off, sizes[k]))
        off += sizes[k]
    for k in range(cfg.d):
        if k != F:
            spans.append((off, cfg.m[k]))
        off += cfg.m[k]
    merged: List[list] = []
    for o, n in spans:
        if merged and merged[-1][0] + merged[-1][1] == o:
            merged[-1][1] += n
        else:
            merged.append([o, n])
    return [tuple(x) for x in merged]


class OwnerShardedTT:
    """One rank of an ID-owner-sharded TT embedding (see the module docstring).

    forward(indices) takes this rank's local batch (any IDs), returns their
    rows in local order; backward(grad_out) takes the local upstream rows;
    step() all-reduces the replicated cores' gradients and updates.  Every
    rank must hold the same initial cores; the level-F slices a rank does not
    own are never read or written by it (gather_level_core() assembles them).
    """

    def __init__(self, emb, group=None, comm=None):
        import torch
        dist = comm or __import__("torch.distributed", fromlist=["x"])
        self.emb, self.group, self.dist = emb, group, dist
        cfg = emb.config
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.bounds = owner_bounds(cfg, self.world)
        self.segments = replicated_segments(cfg)
        # Under the NCCL backend the data plane is the engine's own
        # (tt_owner_forward / _backward / _step over its communicator): no torch
        # ops on the rows; torch.distributed ships only the 128-byte NCCL id
        self.native = (comm is None and group is None and dist.is_initialized()
                       and dist.get_backend() == "nccl" and native_enabled())
        if self.native:
            self.native = _native_init(emb, dist, self.rank, self.world)
        if self.native:
            self.buf = None
            return
        self.buf = torch.zeros(grad_buffer_len(cfg), dtype=torch.float32, device=f"cuda:{emb.device}")
        emb.bind_grad_buffer(self.buf)
        emb.set_dense_grads(True)
        self._route = None
        self._recv_idx = None
        # the replicated segments travel as one packed all-reduce (one NCCL call
        # per step instead of one per segment)
        if len(self.segments) > 1:
            pos = np.concatenate([np.arange(o, o + n, dtype=np.int64) for o, n in self.segments])
            self._pack_idx = torch.from_numpy(pos).to(self.buf.device)
            self._pack = torch.empty(len(pos), dtype=torch.float32, device=self.buf.device)
        else:
            self._pack_idx = None

    def forward(self, indices, out=None):
        import torch
        if self.native:
            return self.emb.owner_forward(indices, out)
        cfg = self.emb.config
        recv, self._route = route_to_owners(cfg, indices, self.group, self.dist)
        self._recv_idx = recv
        rows = self.emb.forward(recv) if recv.numel() else \
            torch.empty((0, cfg.emb_dim), dtype=torch.float32, device=indices.device)
        return route_back(rows, self._route, out, self.group, self.dist)

    def backward(self, grad_out):
        if self.native:
            self.emb.owner_backward(grad_out)
            return
        if self._route is None:
            raise RuntimeError("OwnerShardedTT.backward: no forward on this rank")
        up = route_rows(grad_out, self._route, self.group, self.dist)
        if self._recv_idx.numel():
            self.emb.backward(up)
        else:  # nothing owned this step: zero gradients (CoreGradients::zeros)
            self.emb.backward(up, self._recv_idx)

    def allreduce(self):
        if self._pack_idx is None:
            for o, n in self.segments:
                self.dist.all_reduce(self.buf[o: o + n], group=self.group)
            return
        import torch
        torch.index_select(self.buf, 0, self._pack_idx, out=self._pack)
        self.dist.all_reduce(self._pack, group=self.group)
        self.buf.index_copy_(0, self._pack_idx, self._pack)

    def step(self):
        if self.native:
            self.emb.owner_step()
            return
        self.allreduce()
        self.emb.step()

    def gather_level_core(self):
        """Full level-F core (reference layout) assembled from the owners' slices."""
        import torch
        cfg = self.emb.config
        F = max(cfg.d - 2, 0)
        mine = torch.from_numpy(np.ascontiguousarray(self.emb.get_cores(np.float32)[F])).to(self.buf.device)
        parts = [torch.empty_like(mine) for _ in range(self.world)]
        self.dist.all_gather(parts, mine, group=self.group)
        full = mine.clone()
        for r in range(self.world):
            lo, hi = self.bounds[r], self.bounds[r + 1]
            full[:, lo:hi] = parts[r][:, lo:hi]
        return full.cpu().numpy()
