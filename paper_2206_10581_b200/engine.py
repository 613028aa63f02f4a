"""Python mirror of the reference's TT-embedding operator API over the C-ABI.

Same names, argument meaning and error behaviour as namespace ttgnn
(tt_embedding.hpp:26-59, autodiff.hpp:29-66), backed by the CUDA engine in
libtt_b200.so (include/tt_engine.h).  There is no CPU fallback: importing
this module fails loudly when the extension is missing or no CUDA device is
usable.

  TTEmbedding          device-resident cores (TTEmbedding, tt_embedding.hpp:30-42)
  lookup_batch         tt_embedding.cpp:110-125  (host buffers)
  reconstruct_row      tt_embedding.cpp:103-108
  backward_lookup      autodiff.cpp:48-118        -> CoreGradients
  OptimizerState.make  autodiff.cpp:120-133 (+ Adagrad)
  apply_update         autodiff.cpp:147-173

plus the device-tensor path a GNN training loop uses
(`TTEmbedding.forward / backward / step` on torch CUDA tensors, stream-ordered,
no host synchronisation).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import _build
from .config import InvalidArgument, OutOfRange, TTConfig

MAX_CORES = 8
TT_OK, TT_ERR_ARG, TT_ERR_INDEX, TT_ERR_NONFINITE, TT_ERR_CUDA, TT_ERR_STATE, TT_ERR_NOMEM = range(7)


class LogicError(RuntimeError):
    """API misuse the reference would report as std::logic_error."""


class CudaError(RuntimeError):
    pass


class CConfig(C.Structure):
    _fields_ = [("num_nodes", C.c_int64), ("emb_dim", C.c_int64), ("d", C.c_int32), ("reserved_", C.c_int32),
                ("row_factors", C.c_int64 * MAX_CORES), ("col_factors", C.c_int64 * MAX_CORES),
                ("ranks", C.c_int64 * (MAX_CORES + 1))]


_lib = None

# every symbol include/tt_engine.h declares (tests/test_abi.py checks the .so)
SYMBOLS = [
    "tt_config_validate", "tt_count_params", "tt_engine_create", "tt_engine_destroy", "tt_set_cores_f64",
    "tt_set_cores_f32", "tt_get_cores_f64", "tt_get_cores_f32", "tt_opt_init", "tt_opt_get_step", "tt_forward",
    "tt_backward", "tt_step", "tt_sync", "tt_lookup_batch", "tt_backward_lookup", "tt_apply_update",
    "tt_train_step_host", "tt_get_core_grads_f64", "tt_set_core_grads_f64", "tt_grad_buffer", "tt_set_dense_grads", "tt_bind_grad_buffer",
    "tt_cores_snapshot", "tt_cores_restore", "tt_plan_stats", "tt_plan_digits", "tt_plan_sorted", "tt_launch_count", "tt_set_profiling", "tt_profile_read", "tt_set_path", "tt_last_path",
    "tt_last_error_position", "tt_last_error_value", "tt_last_error", "tt_ffma_peak_tflops", "tt_ffma_outer_tflops",
    "tt_opt_state_get_f64", "tt_opt_state_set_f64", "tt_opt_set_hparams", "tt_debug_trace", "tt_set_permutation",
    "tt_ortho_cores_f64", "tt_nccl_unique_id", "tt_comm_init_rank", "tt_comm_init", "tt_allreduce_grads",
    "tt_train_step_submit", "tt_train_step_wait", "tt_engine_stream",
    "tt_owner_forward", "tt_owner_backward", "tt_owner_step", "tt_owner_rows", "tt_main_kernel",
]


def load_library(build_if_missing: bool = True):
    """Load libtt_b200.so (building it in-tree with nvcc if absent)."""
    global _lib
    if _lib is not None:
        return _lib
    path = os.environ.get("TT_LIB_VARIANT") or _build.LIB  # A/B builds of compile-time switches only
    if not os.path.exists(path):
        if not build_if_missing:
            raise ImportError(f"{path} missing: run `python -m paper_2206_10581_b200._build`")
        _build.build()
    lib = C.CDLL(path)
    vp, i64, i32, dbl = C.c_void_p, C.c_int64, C.c_int, C.c_double
    sig = {
        "tt_config_validate": (i32, [vp]), "tt_count_params": (i64, [vp]),
        "tt_engine_create": (i32, [vp, i32, vp]), "tt_engine_destroy": (None, [vp]),
        "tt_set_cores_f64": (i32, [vp, vp]), "tt_set_cores_f32": (i32, [vp, vp]),
        "tt_get_cores_f64": (i32, [vp, vp]), "tt_get_cores_f32": (i32, [vp, vp]),
        "tt_opt_init": (i32, [vp, i32, dbl, dbl, dbl, dbl]), "tt_opt_get_step": (i32, [vp, vp]),
        "tt_opt_set_hparams": (i32, [vp, dbl, dbl, dbl, dbl]),
        "tt_forward": (i32, [vp, vp, i64, vp, vp]), "tt_backward": (i32, [vp, vp, i64, vp, vp]),
        "tt_step": (i32, [vp, vp]), "tt_sync": (i32, [vp, vp]),
        "tt_lookup_batch": (i32, [vp, vp, i64, vp]), "tt_backward_lookup": (i32, [vp, vp, i64, vp]),
        "tt_apply_update": (i32, [vp]), "tt_train_step_host": (i32, [vp, vp, i64, vp, vp]),
        "tt_get_core_grads_f64": (i32, [vp, vp, vp]), "tt_set_core_grads_f64": (i32, [vp, vp, i64]),
        "tt_grad_buffer": (i32, [vp, vp, vp]), "tt_set_dense_grads": (i32, [vp, i32]),
        "tt_bind_grad_buffer": (i32, [vp, vp, i64]),
        "tt_cores_snapshot": (i32, [vp, vp]), "tt_cores_restore": (i32, [vp, vp]),
        "tt_plan_stats": (i32, [vp, vp]), "tt_plan_digits": (i64, [vp, vp, vp, i64]),
        "tt_plan_sorted": (i64, [vp, vp, vp, i64]), "tt_launch_count": (i64, [vp]),
        "tt_set_profiling": (i32, [vp, i32]), "tt_profile_read": (i32, [vp, vp, vp, i32]),
        "tt_set_path": (i32, [vp, i32]), "tt_last_path": (i32, [vp]),
        "tt_last_error_position": (i64, []), "tt_last_error_value": (i64, []),
        "tt_last_error": (C.c_char_p, []), "tt_ffma_peak_tflops": (dbl, [i32, i32]),
        "tt_ffma_outer_tflops": (dbl, [i32, i32]),
        "tt_opt_state_get_f64": (i32, [vp, vp, vp, vp]), "tt_opt_state_set_f64": (i32, [vp, vp, vp, i64]),
        "tt_debug_trace": (i64, [vp, i64]), "tt_set_permutation": (i32, [vp, vp, i64]),
        "tt_ortho_cores_f64": (i32, [vp, i32, C.c_uint64, dbl, vp, vp]),
        "tt_nccl_unique_id": (i32, [vp, i64]), "tt_comm_init_rank": (i32, [vp, vp, i32, i32]),
        "tt_comm_init": (i32, [vp, vp, i32, i32]), "tt_allreduce_grads": (i32, [vp, vp]),
        "tt_train_step_submit": (i32, [vp, vp, i64, vp, vp]), "tt_train_step_wait": (i32, [vp]),
        "tt_engine_stream": (vp, [vp]),
        "tt_owner_forward": (i32, [vp, vp, i64, vp, vp]), "tt_owner_backward": (i32, [vp, vp, vp]),
        "tt_owner_step": (i32, [vp, vp]), "tt_owner_rows": (i64, [vp]),
        "tt_main_kernel": (C.c_char_p, [vp, i32]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    _lib = lib
    return lib


def _raise(rc: int, where: str = ""):
    if rc == TT_OK:
        return
    msg = (_lib.tt_last_error() or b"").decode()
    if rc == TT_ERR_INDEX:
        e = OutOfRange(msg)
        e.position = int(_lib.tt_last_error_position())
        e.value = int(_lib.tt_last_error_value())
        raise e
    if rc in (TT_ERR_ARG, TT_ERR_NONFINITE):
        e = InvalidArgument(msg)
        e.position = int(_lib.tt_last_error_position())
        raise e
    if rc == TT_ERR_STATE:
        raise LogicError(msg)
    if rc == TT_ERR_NOMEM:
        raise MemoryError(msg)
    raise CudaError(f"{where}: {msg}")


def to_cconfig(cfg: TTConfig) -> CConfig:
    if cfg.d > MAX_CORES:
        raise InvalidArgument(f"TTConfig: at most {MAX_CORES} cores supported")
    c = CConfig()
    c.num_nodes, c.emb_dim, c.d = int(cfg.num_nodes), int(cfg.emb_dim), len(cfg.row_factors)
    for k in range(c.d):
        c.row_factors[k], c.col_factors[k] = int(cfg.row_factors[k]), int(cfg.col_factors[k])
    for k in range(len(cfg.ranks)):
        c.ranks[k] = int(cfg.ranks[k])
    return c


def _ptr_array(arrs, ctype):
    return (C.c_void_p * len(arrs))(*[a.ctypes.data for a in arrs])


def _torch():
    import torch
    return torch


class OptKind:
    sgd = 0
    adam = 1
    adagrad = 2


@dataclass
class OptimizerState:
    """OptimizerState (autodiff.hpp:43-56); moments live on the device."""
    kind: int = OptKind.adam
    learning_rate: float = 1e-3
    beta1: float = 0.9
    beta2: float = 0.999
    epsilon: float = 1e-8
    step: int = 0

    @staticmethod
    def make(config: TTConfig, kind: int, lr: float) -> "OptimizerState":
        eps = 1e-10 if kind == OptKind.adagrad else 1e-8
        return OptimizerState(kind=kind, learning_rate=lr, epsilon=eps)


@dataclass
class CoreGradients:
    """CoreGradients (autodiff.hpp:29-34).  `grads` is fetched lazily from the
    engine that produced it (reference layout, float64)."""
    grads_: Optional[List[np.ndarray]] = None
    batch_count: int = 0
    _engine: Optional["TTEmbedding"] = field(default=None, repr=False)
    _version: int = -1

    @property
    def grads(self) -> List[np.ndarray]:
        if self.grads_ is None:
            self.grads_ = self._engine._fetch_grads()
        return self.grads_

    @staticmethod
    def zeros(config: TTConfig) -> "CoreGradients":
        return CoreGradients([np.zeros(config.core_shape(k)) for k in range(config.d)], 0)


class TTEmbedding:
    """Device-resident tensor-train embedding table (one handle per GPU)."""

    def __init__(self, config: TTConfig, device: int = 0):
        config.validate()
        self.config = config
        self.device = device
        self._lib = load_library()
        self._cc = to_cconfig(config)
        h = C.c_void_p()
        _raise(self._lib.tt_engine_create(C.byref(self._cc), device, C.byref(h)), "tt_engine_create")
        self._h = h
        self._grad_version = 0
        self._opt: Optional[OptimizerState] = None
        self._opt_sig = None

    def __del__(self):
        if getattr(self, "_h", None):
            self._lib.tt_engine_destroy(self._h)
            self._h = None

    @classmethod
    def zeros(cls, config: TTConfig, device: int = 0) -> "TTEmbedding":
        return cls(config, device)

    @classmethod
    def from_cores(cls, config: TTConfig, cores, device: int = 0) -> "TTEmbedding":
        e = cls(config, device)
        e.set_cores(cores)
        return e

    # ---- cores (reference layout) ----------------------------------------
    def set_cores(self, cores) -> None:
        cfg = self.config
        if len(cores) != cfg.d:
            raise InvalidArgument("TTEmbedding: wrong number of cores")
        arrs = []
        f64 = all(np.asarray(c).dtype == np.float64 for c in cores)
        for k, c in enumerate(cores):
            a = np.ascontiguousarray(c, dtype=np.float64 if f64 else np.float32)
            if a.size != cfg.core_size(k):
                raise InvalidArgument(f"TTEmbedding: core {k} storage size mismatch")
            arrs.append(a)
        fn = self._lib.tt_set_cores_f64 if f64 else self._lib.tt_set_cores_f32
        _raise(fn(self._h, _ptr_array(arrs, None)), "tt_set_cores")

    def get_cores(self, dtype=np.float32) -> List[np.ndarray]:
        cfg = self.config
        arrs = [np.empty(cfg.core_shape(k), dtype=dtype) for k in range(cfg.d)]
        fn = self._lib.tt_get_cores_f64 if dtype == np.float64 else self._lib.tt_get_cores_f32
        _raise(fn(self._h, _ptr_array(arrs, None)), "tt_get_cores")
        return arrs

    @property
    def cores(self) -> List[np.ndarray]:
        return self.get_cores(np.float32)

    def _fetch_grads(self) -> List[np.ndarray]:
        cfg = self.config
        arrs = [np.empty(cfg.core_shape(k), dtype=np.float64) for k in range(cfg.d)]
        bc = C.c_int64()
        _raise(self._lib.tt_get_core_grads_f64(self._h, _ptr_array(arrs, None), C.byref(bc)), "tt_get_core_grads")
        return arrs

    # ---- device-tensor path (torch CUDA tensors, current stream) -----------
    def _check_device(self, t, what: str) -> None:
        if not t.is_cuda or t.device.index != self.device:
            raise InvalidArgument(f"{what} must be on cuda:{self.device}, got {t.device}")

    def _stream(self):
        torch = _torch()
        return C.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)

    def forward(self, indices, out=None):
        torch = _torch()
        if indices.dtype != torch.int64 or not indices.is_cuda or not indices.is_contiguous():
            raise InvalidArgument("forward: indices must be a contiguous int64 CUDA tensor")
        self._check_device(indices, "forward: indices")
        B = indices.numel()
        if out is None:
            out = torch.empty((B, self.config.emb_dim), dtype=torch.float32, device=indices.device)
        else:
            if out.dtype != torch.float32 or not out.is_contiguous():
                raise InvalidArgument("forward: out must be a contiguous float32 CUDA tensor")
            if tuple(out.shape) != (B, self.config.emb_dim):
                raise InvalidArgument(f"forward: out must have shape ({B}, {self.config.emb_dim}), "
                                      f"got {tuple(out.shape)}")
            self._check_device(out, "forward: out")
        _raise(self._lib.tt_forward(self._h, C.c_void_p(indices.data_ptr()), B, C.c_void_p(out.data_ptr()),
                                    self._stream()), "tt_forward")
        return out

    def backward(self, grad_out, indices=None) -> None:
        """Gradients of the last forward (indices=None) or of `indices`."""
        torch = _torch()
        if grad_out.dtype != torch.float32 or not grad_out.is_cuda or not grad_out.is_contiguous():
            raise InvalidArgument("backward: grad_out must be a contiguous float32 CUDA tensor")
        self._check_device(grad_out, "backward: grad_out")
        if indices is not None:
            if indices.dtype != torch.int64 or not indices.is_cuda or not indices.is_contiguous():
                raise InvalidArgument("backward: indices must be a contiguous int64 CUDA tensor")
            self._check_device(indices, "backward: indices")
        B = grad_out.shape[0]
        if grad_out.dim() != 2 or grad_out.shape[1] != self.config.emb_dim:
            raise InvalidArgument("backward_lookup: upstream cols != emb_dim")
        if indices is not None and indices.numel() != B:
            raise InvalidArgument("backward_lookup: upstream rows != index count")
        ip = C.c_void_p(indices.data_ptr()) if indices is not None else None
        _raise(self._lib.tt_backward(self._h, ip, B, C.c_void_p(grad_out.data_ptr()), self._stream()),
               "tt_backward")
        self._grad_version += 1

    def step(self) -> None:
        _raise(self._lib.tt_step(self._h, self._stream()), "tt_step")

    def snapshot_cores(self) -> None:
        _raise(self._lib.tt_cores_snapshot(self._h, self._stream()), "tt_cores_snapshot")

    def restore_cores(self) -> None:
        _raise(self._lib.tt_cores_restore(self._h, self._stream()), "tt_cores_restore")

    def sync(self) -> None:
        _raise(self._lib.tt_sync(self._h, self._stream()), "tt_sync")

    def configure_optimizer(self, opt: OptimizerState) -> None:
        """Binds `opt` to the engine's device-resident optimizer state.

        In the reference the moments live in the OptimizerState object
        (autodiff.hpp:43-56) and apply_update reads lr/betas/eps from it on
        every call (autodiff.cpp:147-173).  Here the moments live on the device:
        they are (re)initialised -- zero moments, step 0, as
        OptimizerState::make produces them -- only when the optimizer kind
        changes or a fresh state object (step 0) replaces the bound one.
        Otherwise the hyper-parameters are pushed as they are now (a learning
        rate schedule never resets the moments), and the device step follows
        opt.step (a state object carried across rebuilds keeps counting)."""
        fresh = self._opt is None or self._opt_sig != opt.kind or (self._opt is not opt and opt.step == 0)
        if fresh:
            _raise(self._lib.tt_opt_init(self._h, opt.kind, opt.learning_rate, opt.beta1, opt.beta2, opt.epsilon),
                   "tt_opt_init")
            opt.step = 0
        else:
            _raise(self._lib.tt_opt_set_hparams(self._h, opt.learning_rate, opt.beta1, opt.beta2, opt.epsilon),
                   "tt_opt_set_hparams")
            if self._opt is not opt and opt.step != self.opt_step():
                _raise(self._lib.tt_opt_state_set_f64(self._h, None, None, int(opt.step)), "tt_opt_state_set")
        self._opt, self._opt_sig = opt, opt.kind

    def train_step_host(self, indices: np.ndarray, upstream: np.ndarray, out: Optional[np.ndarray] = None):
        idx = np.ascontiguousarray(indices, dtype=np.int64)
        up = np.ascontiguousarray(upstream, dtype=np.float32)
        op = out.ctypes.data if out is not None else None
        _raise(self._lib.tt_train_step_host(self._h, idx.ctypes.data, len(idx), up.ctypes.data, op),
               "tt_train_step_host")

    def train_step_submit(self, indices, upstream, out=None) -> None:
        """Pipelined host-buffer step (tt_train_step_submit): returns at once;
        the buffers (numpy arrays or pinned torch CPU tensors) must stay alive
        until train_step_wait() retires the step."""
        ip = indices.ctypes.data if isinstance(indices, np.ndarray) else indices.data_ptr()
        up = upstream.ctypes.data if isinstance(upstream, np.ndarray) else upstream.data_ptr()
        op = None if out is None else (out.ctypes.data if isinstance(out, np.ndarray) else out.data_ptr())
        B = len(indices)
        _raise(self._lib.tt_train_step_submit(self._h, C.c_void_p(ip), B, C.c_void_p(up),
                                              None if op is None else C.c_void_p(op)), "tt_train_step_submit")

    def train_step_wait(self) -> None:
        _raise(self._lib.tt_train_step_wait(self._h), "tt_train_step_wait")

    def main_kernel(self, backward: bool) -> str:
        """The level-F GEMM kernel of the last forward / backward."""
        return (self._lib.tt_main_kernel(self._h, 1 if backward else 0) or b"").decode()

    def engine_stream(self) -> int:
        return self._lib.tt_engine_stream(self._h) or 0

    def restore_cores_on_engine_stream(self) -> None:
        """tt_cores_restore ordered with the host-buffer calls (the handle's stream)."""
        _raise(self._lib.tt_cores_restore(self._h, C.c_void_p(self.engine_stream())), "tt_cores_restore")

    def grad_buffer(self):
        p, n = C.c_void_p(), C.c_int64()
        _raise(self._lib.tt_grad_buffer(self._h, C.byref(p), C.byref(n)), "tt_grad_buffer")
        return p.value, n.value

    def bind_grad_buffer(self, tensor) -> None:
        """Use a caller-owned float32 CUDA tensor as the gradient buffer."""
        if tensor is None:
            _raise(self._lib.tt_bind_grad_buffer(self._h, None, 0), "tt_bind_grad_buffer")
            self._bound = None
            return
        _raise(self._lib.tt_bind_grad_buffer(self._h, C.c_void_p(tensor.data_ptr()), tensor.numel()),
               "tt_bind_grad_buffer")
        self._bound = tensor  # keep alive

    def set_dense_grads(self, on: bool) -> None:
        _raise(self._lib.tt_set_dense_grads(self._h, 1 if on else 0), "tt_set_dense_grads")

    def set_path(self, path: str) -> None:
        _raise(self._lib.tt_set_path(self._h, {"auto": 0, "generic": 1, "tc": 2}[path]), "tt_set_path")

    def last_path(self) -> str:
        return ["generic", "fused", "fused-tc"][self._lib.tt_last_path(self._h)]

    def plan_stats(self) -> List[int]:
        out = np.zeros(self.config.d, np.int64)
        _raise(self._lib.tt_plan_stats(self._h, out.ctypes.data), "tt_plan_stats")
        return [int(x) for x in out]

    def plan_digits(self):
        cap = 1
        while True:
            ids = np.zeros(cap, np.int64)
            dig = np.zeros(cap * self.config.d, np.int32)
            U = self._lib.tt_plan_digits(self._h, ids.ctypes.data, dig.ctypes.data, cap)
            if U < 0:
                raise LogicError("tt_plan_digits: no plan")
            if U <= cap:
                return ids[:U], dig[: U * self.config.d].reshape(U, self.config.d)
            cap = int(U)

    def plan_sorted(self):
        cap = 1
        while True:
            keys = np.zeros(cap, np.int64)
            pos = np.zeros(cap, np.int32)
            B = self._lib.tt_plan_sorted(self._h, keys.ctypes.data, pos.ctypes.data, cap)
            if B < 0:
                raise LogicError("tt_plan_sorted: no plan")
            if B <= cap:
                return keys[:B], pos[:B]
            cap = int(B)

    PHASES = ("plan", "fwd_main", "bwd_main", "bwd_aux", "update")

    def set_profiling(self, on: bool) -> None:
        _raise(self._lib.tt_set_profiling(self._h, 1 if on else 0), "tt_set_profiling")

    def profile_read(self):
        """{phase: (total ms, event pairs)} since the last read (synchronises)."""
        ms = np.zeros(len(self.PHASES), np.float64)
        n = np.zeros(len(self.PHASES), np.int64)
        _raise(self._lib.tt_profile_read(self._h, ms.ctypes.data, n.ctypes.data, len(self.PHASES)), "tt_profile_read")
        return {p: (float(ms[i]), int(n[i])) for i, p in enumerate(self.PHASES)}

    def launch_count(self) -> int:
        return int(self._lib.tt_launch_count(self._h))

    def set_permutation(self, perm) -> None:
        """Node relabelling of a hierarchical reorder (graph.cpp:218-252): ID v
        is served by row perm[v] from now on (None clears)."""
        if perm is None:
            _raise(self._lib.tt_set_permutation(self._h, None, 0), "tt_set_permutation")
            return
        p = np.ascontiguousarray(perm, dtype=np.int64)
        _raise(self._lib.tt_set_permutation(self._h, p.ctypes.data, len(p)), "tt_set_permutation")

    def get_opt_state(self):
        """(s1, s2, step): optimizer state in the reference core layout (fp64),
        s1 = Adagrad accumulator / Adam first moment, s2 = Adam second moment;
        None where the configured optimizer has no such state."""
        cfg = self.config
        kind = self._opt.kind if self._opt is not None else OptKind.sgd
        s1 = [np.zeros(cfg.core_shape(k)) for k in range(cfg.d)] if kind != OptKind.sgd else None
        s2 = [np.zeros(cfg.core_shape(k)) for k in range(cfg.d)] if kind == OptKind.adam else None
        st = C.c_int64()
        _raise(self._lib.tt_opt_state_get_f64(self._h, _ptr_array(s1, None) if s1 else None,
                                              _ptr_array(s2, None) if s2 else None, C.byref(st)), "tt_opt_state_get")
        return s1, s2, int(st.value)

    def set_opt_state(self, s1, s2, step: int) -> None:
        """Restores get_opt_state()'s arrays (after configure_optimizer)."""
        cfg = self.config
        a1 = [np.ascontiguousarray(x, np.float64).reshape(cfg.core_shape(k)) for k, x in enumerate(s1)] if s1 else None
        a2 = [np.ascontiguousarray(x, np.float64).reshape(cfg.core_shape(k)) for k, x in enumerate(s2)] if s2 else None
        _raise(self._lib.tt_opt_state_set_f64(self._h, _ptr_array(a1, None) if a1 else None,
                                              _ptr_array(a2, None) if a2 else None, int(step)), "tt_opt_state_set")
        if self._opt is not None:
            self._opt.step = int(step)

    # ---- NCCL data parallelism through the C-ABI (position sharding) --------
    def comm_init_rank(self, unique_id: bytes, rank: int, world: int) -> None:
        """Creates the engine's own NCCL communicator (every rank passes the
        same 128-byte id from nccl_unique_id())."""
        buf = C.create_string_buffer(bytes(unique_id), 128)
        _raise(self._lib.tt_comm_init_rank(self._h, buf, rank, world), "tt_comm_init_rank")

    def owner_forward(self, indices, out=None):
        """ID-owner-sharded forward over the NCCL communicator (tt_owner_forward):
        this rank's batch in, its rows out (in batch order)."""
        torch = _torch()
        if indices.dtype != torch.int64 or not indices.is_cuda or not indices.is_contiguous():
            raise InvalidArgument("owner_forward: indices must be a contiguous int64 CUDA tensor")
        self._check_device(indices, "owner_forward: indices")
        B = indices.numel()
        if out is None:
            out = torch.empty((B, self.config.emb_dim), dtype=torch.float32, device=indices.device)
        _raise(self._lib.tt_owner_forward(self._h, C.c_void_p(indices.data_ptr()), B, C.c_void_p(out.data_ptr()),
                                          self._stream()), "tt_owner_forward")
        return out

    def owner_backward(self, grad_out) -> None:
        torch = _torch()
        if grad_out.dtype != torch.float32 or not grad_out.is_cuda or not grad_out.is_contiguous():
            raise InvalidArgument("owner_backward: grad_out must be a contiguous float32 CUDA tensor")
        self._check_device(grad_out, "owner_backward: grad_out")
        _raise(self._lib.tt_owner_backward(self._h, C.c_void_p(grad_out.data_ptr()), self._stream()),
               "tt_owner_backward")
        self._grad_version += 1

    def owner_step(self) -> None:
        _raise(self._lib.tt_owner_step(self._h, self._stream()), "tt_owner_step")

    def owner_rows(self) -> int:
        return int(self._lib.tt_owner_rows(self._h))

    def allreduce_grads(self) -> None:
        """Sum all-reduce of the gradient buffer over the communicator,
        stream-ordered between backward and step (tt_allreduce_grads)."""
        _raise(self._lib.tt_allreduce_grads(self._h, self._stream()), "tt_allreduce_grads")

    def opt_step(self) -> int:
        s = C.c_int64()
        _raise(self._lib.tt_opt_get_step(self._h, C.byref(s)), "tt_opt_get_step")
        return s.value


# ---- reference free functions (host buffers) -------------------------------
def lookup_batch(emb: TTEmbedding, indices) -> np.ndarray:
    """tt_embedding.cpp:110-125: (B x emb_dim) float32, row b = indices[b];
    any out-of-range index raises OutOfRange naming its batch position."""
    idx = np.ascontiguousarray(indices, dtype=np.int64).reshape(-1)
    out = np.empty((len(idx), emb.config.emb_dim), np.float32)
    _raise(emb._lib.tt_lookup_batch(emb._h, idx.ctypes.data, len(idx), out.ctypes.data), "lookup_batch")
    return out


def reconstruct_row(emb: TTEmbedding, row: int) -> np.ndarray:
    if row < 0 or row >= emb.config.num_nodes:
        raise OutOfRange(f"reconstruct_row: index {row} out of [0, {emb.config.num_nodes})")
    return lookup_batch(emb, [row])[0]


def backward_lookup(emb: TTEmbedding, indices, upstream) -> CoreGradients:
    """autodiff.cpp:48-118 (sum over rows; duplicates accumulate)."""
    idx = np.ascontiguousarray(indices, dtype=np.int64).reshape(-1)
    up = np.ascontiguousarray(upstream, dtype=np.float32)
    if up.ndim != 2 or up.shape[0] != len(idx):
        raise InvalidArgument("backward_lookup: upstream rows != index count")
    if up.shape[1] != emb.config.emb_dim:
        raise InvalidArgument("backward_lookup: upstream cols != emb_dim")
    _raise(emb._lib.tt_backward_lookup(emb._h, idx.ctypes.data, len(idx), up.ctypes.data), "backward_lookup")
    emb._grad_version += 1
    return CoreGradients(None, len(idx), emb, emb._grad_version)


def apply_update(emb: TTEmbedding, grads: CoreGradients, opt: OptimizerState) -> None:
    """autodiff.cpp:147-173: all-or-nothing; raises InvalidArgument naming the
    core on a non-finite gradient with cores, moments and step untouched."""
    cfg = emb.config
    emb.configure_optimizer(opt)
    if grads._engine is not emb or grads._version != emb._grad_version:
        g = grads.grads
        if len(g) != cfg.d:
            raise InvalidArgument("apply_update: gradient core count mismatch")
        arrs = []
        for k in range(cfg.d):
            a = np.ascontiguousarray(g[k], dtype=np.float64)
            if a.size != cfg.core_size(k):
                raise InvalidArgument(f"apply_update: gradient shape mismatch at core {k}")
            arrs.append(a)
        _raise(emb._lib.tt_set_core_grads_f64(emb._h, _ptr_array(arrs, None), grads.batch_count), "set_grads")
        emb._grad_version += 1
    _raise(emb._lib.tt_apply_update(emb._h), "apply_update")
    opt.step = emb.opt_step()


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _raise(load_library().tt_nccl_unique_id(buf, 128), "tt_nccl_unique_id")
    return buf.raw


def ffma_peak_tflops(device: int = 0, iters: int = 4096) -> float:
    return float(load_library().tt_ffma_peak_tflops(device, iters))


def ffma_outer_tflops(device: int = 0, iters: int = 4096) -> float:
    return float(load_library().tt_ffma_outer_tflops(device, iters))
