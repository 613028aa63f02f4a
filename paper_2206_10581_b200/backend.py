"""EmbeddingBackend: the reference's trainable node-embedding
source for its GNN harness (gnn.hpp:38-72, gnn.cpp:37-128), with the
tensor-train kind served by the B200 engine.

* kind `tt`: cores on the device (engine.TTEmbedding).
  * `lookup_all` / `lookup` run the CUDA forward.
  * `apply_gradients(grad_rows)` runs the CUDA backward over all rows plus one
    update on the device. This is the reference's backward_lookup over
    iota(num_nodes) followed by apply_update (gnn.cpp:123-127).
* kind `full`: the dense M x N table the reference compares against. It stays
  a host fp64 table with the reference's own arithmetic (SGD, or Adam via
  adam_step, autodiff.cpp:135-145). It is the baseline of the paper's
  experiments, not the TT hot path, so no device kernel serves it.

Errors and messages follow gnn.cpp:
* lookup out of range -> OutOfRange;
* wrong gradient shape -> InvalidArgument("apply_gradients: bad gradient shape");
* non-finite table gradient -> InvalidArgument;
* tt() / table() on the wrong kind -> LogicError.
"""
from __future__ import annotations

import numpy as np

from . import synth
from .config import InvalidArgument, OutOfRange


class BackendKind:
    full = 0
    tt = 1


class EmbeddingBackend:
    def __init__(self):
        self._kind = BackendKind.full
        self._table = None
        self._m = self._v = None
        self._step = 0
        self._tt = None
        self._opt_kind = 1  # OptKind.adam
        self._lr = 1e-3

    # ---- construction (gnn.cpp:40-77) -------------------------------------
    @staticmethod
    def full_table(num_nodes: int, emb_dim: int, seed: int, init_std: float, opt: int, lr: float):
        """Dense table of init_std x N(0, 1) entries.

        The reference draws them from std::mt19937_64 + std::normal_distribution.
        That pairing is not portable across standard libraries, so the seeded
        portable generator (synth.normal) stands in, as for the cores.
        """
        table = init_std * synth.normal(seed, 0, num_nodes * emb_dim, 1.0, np.float64).reshape(num_nodes, emb_dim)
        return EmbeddingBackend.full_table_from(table, opt, lr)

    @staticmethod
    def full_table_from(table, opt: int, lr: float):
        from .engine import OptKind
        b = EmbeddingBackend()
        b._kind = BackendKind.full
        b._table = np.array(table, dtype=np.float64, copy=True)
        b._opt_kind, b._lr = opt, lr
        if opt == OptKind.adam:
            b._m = np.zeros_like(b._table)
            b._v = np.zeros_like(b._table)
        return b

    @staticmethod
    def tensor_train(emb, opt: int, lr: float):
        """`emb` is a device engine.TTEmbedding (cores already set)."""
        from .engine import OptimizerState
        emb.config.validate()
        b = EmbeddingBackend()
        b._kind = BackendKind.tt
        b._tt = emb
        b._opt_kind, b._lr = opt, lr
        emb.configure_optimizer(OptimizerState.make(emb.config, opt, lr))
        return b

    # ---- shape ---------------------------------------------------------------
    def kind(self) -> int:
        return self._kind

    def num_nodes(self) -> int:
        return self._table.shape[0] if self._kind == BackendKind.full else self._tt.config.num_nodes

    def emb_dim(self) -> int:
        return self._table.shape[1] if self._kind == BackendKind.full else self._tt.config.emb_dim

    def param_count(self) -> int:
        if self._kind == BackendKind.full:
            return int(self._table.size)
        cfg = self._tt.config
        return int(sum(cfg.core_size(k) for k in range(cfg.d)))

    # ---- lookups (gnn.cpp:89-105) -------------------------------------------
    def lookup_all(self) -> np.ndarray:
        if self._kind == BackendKind.full:
            return self._table.copy()
        return self.lookup(np.arange(self._tt.config.num_nodes, dtype=np.int64))

    def lookup(self, indices) -> np.ndarray:
        idx = np.ascontiguousarray(indices, dtype=np.int64)
        if self._kind == BackendKind.tt:
            from .engine import lookup_batch
            return lookup_batch(self._tt, idx).astype(np.float64)
        bad = np.flatnonzero((idx < 0) | (idx >= self._table.shape[0]))
        if bad.size:
            b = int(bad[0])
            raise OutOfRange(f"lookup: index {int(idx[b])} at batch position {b} out of range")
        return self._table[idx].copy()

    # ---- training (gnn.cpp:107-128) -----------------------------------------
    def apply_gradients(self, grad_rows) -> None:
        """One optimizer step from dLoss/dH0 over all rows."""
        from .engine import OptKind
        g = np.asarray(grad_rows)
        if g.shape != (self.num_nodes(), self.emb_dim()):
            raise InvalidArgument("apply_gradients: bad gradient shape")
        if self._kind == BackendKind.full:
            g = g.astype(np.float64)
            if not np.all(np.isfinite(g)):
                raise InvalidArgument("apply_gradients: non-finite table gradient")
            self._step += 1
            if self._opt_kind == OptKind.sgd:
                self._table -= self._lr * g
            else:  # adam_step (autodiff.cpp:135-145)
                b1, b2, eps = 0.9, 0.999, 1e-8
                bc1 = 1.0 - b1 ** self._step
                bc2 = 1.0 - b2 ** self._step
                self._m = b1 * self._m + (1.0 - b1) * g
                self._v = b2 * self._v + (1.0 - b2) * g * g
                self._table -= self._lr * (self._m / bc1) / (np.sqrt(self._v / bc2) + eps)
            return
        import torch
        dev = f"cuda:{self._tt.device}"
        n = self._tt.config.num_nodes
        idx = torch.arange(n, dtype=torch.int64, device=dev)
        up = torch.tensor(np.ascontiguousarray(g, dtype=np.float32), device=dev)
        self._tt.backward(up, idx)
        self._tt.step()
        self._tt.sync()

    # ---- accessors --------------------------------------------------------------
    def tt(self):
        if self._kind != BackendKind.tt:
            from .engine import LogicError
            raise LogicError("backend is not tensor-train")
        return self._tt

    def table(self) -> np.ndarray:
        if self._kind != BackendKind.full:
            from .engine import LogicError
            raise LogicError("backend is not a full table")
        return self._table
