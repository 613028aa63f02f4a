"""ctypes bindings for the C oracle (TEST INFRASTRUCTURE ONLY; see __init__)."""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
MAXD = 16
SGD, ADAM, ADAGRAD = 0, 1, 2


class OrCfg(C.Structure):
    _fields_ = [("num_nodes", C.c_int64), ("emb_dim", C.c_int64), ("d", C.c_int32),
                ("pad_", C.c_int32), ("m", C.c_int64 * MAXD), ("n", C.c_int64 * MAXD),
                ("R", C.c_int64 * (MAXD + 1))]


def build() -> None:
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def _load(path: str):
    return C.CDLL(path)


_lib = None
_ref = None


def lib():
    global _lib
    if _lib is None:
        path = os.path.join(HERE, "libttoracle.so")
        if not os.path.exists(path):
            build()
        _lib = _load(path)
        _lib.or_lookup_batch.restype = C.c_int64
        _lib.or_backward_lookup.restype = C.c_int64
        _lib.or_lookup_batch_f32.restype = C.c_int64
        _lib.or_backward_lookup_f32.restype = C.c_int64
        _lib.or_count_params.restype = C.c_int64
        _lib.or_padded_rows.restype = C.c_int64
        _lib.or_ttm_entry.restype = C.c_double
        _lib.or_sort_unique.restype = C.c_int64
        _lib.or_coordinate_to_index.restype = C.c_int64
    return _lib


def ref():
    """The reference's own tt_config.cpp (oracle/_ref), or None if unbuilt."""
    global _ref
    if _ref is None:
        path = os.path.join(HERE, "_ref", "libttref.so")
        if not os.path.exists(path):
            return None
        _ref = _load(path)
        _ref.ref_count_params.restype = C.c_int64
        _ref.ref_index_to_coordinate.restype = C.c_int64
        _ref.ref_coordinate_to_index.restype = C.c_int64
    return _ref


def to_c(cfg) -> OrCfg:
    c = OrCfg()
    c.num_nodes = int(cfg.num_nodes)
    c.emb_dim = int(cfg.emb_dim)
    c.d = len(cfg.row_factors)
    for k in range(c.d):
        c.m[k] = int(cfg.row_factors[k])
        c.n[k] = int(cfg.col_factors[k])
    for k in range(len(cfg.ranks)):
        c.R[k] = int(cfg.ranks[k])
    return c


def _i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _ptrs(arrs):
    return (C.POINTER(C.c_double) * len(arrs))(*[a.ctypes.data_as(C.POINTER(C.c_double)) for a in arrs])


def count_params(cfg) -> int:
    return lib().or_count_params(C.byref(to_c(cfg)))


def validate(cfg) -> int:
    return lib().or_validate(C.byref(to_c(cfg)))


def index_to_coordinate(cfg, row: int):
    parts = np.zeros(MAXD, np.int64)
    rc = lib().or_index_to_coordinate(C.byref(to_c(cfg)), C.c_int64(row), parts.ctypes.data_as(C.c_void_p))
    return None if rc != 0 else [int(x) for x in parts[: len(cfg.row_factors)]]


def coordinate_to_index(cfg, parts) -> int:
    p = _i64(parts)
    return lib().or_coordinate_to_index(C.byref(to_c(cfg)), p.ctypes.data_as(C.c_void_p))


def lookup_batch(cfg, cores, idx, nthreads: int = 1):
    """(out float64[B, emb_dim], first bad position or -1)."""
    idx = _i64(idx)
    cores = [_f64(c).ravel() for c in cores]
    out = np.zeros((len(idx), cfg.emb_dim), np.float64)
    bad = lib().or_lookup_batch(C.byref(to_c(cfg)), _ptrs(cores), idx.ctypes.data_as(C.c_void_p),
                                C.c_int64(len(idx)), out.ctypes.data_as(C.c_void_p), C.c_int(nthreads))
    return out, int(bad)


def backward_lookup(cfg, cores, idx, upstream, nthreads: int = 1):
    """(grads list of float64 arrays shaped like the cores, bad position or -1)."""
    idx = _i64(idx)
    cores = [_f64(c).ravel() for c in cores]
    up = _f64(upstream).reshape(len(idx), cfg.emb_dim)
    grads = [np.zeros(cfg.core_size(k), np.float64) for k in range(cfg.d)]
    bad = lib().or_backward_lookup(C.byref(to_c(cfg)), _ptrs(cores), idx.ctypes.data_as(C.c_void_p),
                                   C.c_int64(len(idx)), up.ctypes.data_as(C.c_void_p), _ptrs(grads),
                                   C.c_int(nthreads))
    return [g.reshape(cfg.core_shape(k)) for k, g in enumerate(grads)], int(bad)


class OptState:
    def __init__(self, cfg, kind: int, lr: float, beta1=0.9, beta2=0.999, eps=None):
        self.kind, self.lr, self.beta1, self.beta2 = kind, lr, beta1, beta2
        self.eps = eps if eps is not None else (1e-10 if kind == ADAGRAD else 1e-8)
        self.step = 0
        self.s1 = [np.zeros(cfg.core_size(k)) for k in range(cfg.d)]
        self.s2 = [np.zeros(cfg.core_size(k)) for k in range(cfg.d)]


def apply_update(cfg, cores, grads, opt: OptState) -> int:
    """In-place on float64 `cores` (list of contiguous arrays); returns -1 or
    the index of the first core with a non-finite gradient (state untouched)."""
    flat = [c.reshape(-1) for c in cores]
    for c in flat:
        assert c.dtype == np.float64 and c.flags.c_contiguous
    g = [_f64(x).ravel() for x in grads]
    step = C.c_int64(opt.step)
    rc = lib().or_apply_update(C.byref(to_c(cfg)), _ptrs(flat), _ptrs(g), C.c_int(opt.kind),
                               C.c_double(opt.lr), C.c_double(opt.beta1), C.c_double(opt.beta2),
                               C.c_double(opt.eps), C.byref(step), _ptrs(opt.s1), _ptrs(opt.s2))
    opt.step = step.value
    return rc


# ---- fp32 variant (the multithreaded fp32 CPU
# baseline; same loops as the fp64 restatement, float elements) ------------
def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def _ptrs32(arrs):
    return (C.POINTER(C.c_float) * len(arrs))(*[a.ctypes.data_as(C.POINTER(C.c_float)) for a in arrs])


def lookup_batch_f32(cfg, cores, idx, nthreads: int = 1):
    idx = _i64(idx)
    cores = [_f32(c).ravel() for c in cores]
    out = np.zeros((len(idx), cfg.emb_dim), np.float32)
    bad = lib().or_lookup_batch_f32(C.byref(to_c(cfg)), _ptrs32(cores), idx.ctypes.data_as(C.c_void_p),
                                    C.c_int64(len(idx)), out.ctypes.data_as(C.c_void_p), C.c_int(nthreads))
    return out, int(bad)


def backward_lookup_f32(cfg, cores, idx, upstream, nthreads: int = 1):
    idx = _i64(idx)
    cores = [_f32(c).ravel() for c in cores]
    up = _f32(upstream).reshape(len(idx), cfg.emb_dim)
    grads = [np.zeros(cfg.core_size(k), np.float32) for k in range(cfg.d)]
    bad = lib().or_backward_lookup_f32(C.byref(to_c(cfg)), _ptrs32(cores), idx.ctypes.data_as(C.c_void_p),
                                       C.c_int64(len(idx)), up.ctypes.data_as(C.c_void_p), _ptrs32(grads),
                                       C.c_int(nthreads))
    return [g.reshape(cfg.core_shape(k)) for k, g in enumerate(grads)], int(bad)


class OptState32(OptState):
    def __init__(self, cfg, kind: int, lr: float, beta1=0.9, beta2=0.999, eps=None):
        super().__init__(cfg, kind, lr, beta1, beta2, eps)
        self.s1 = [np.zeros(cfg.core_size(k), np.float32) for k in range(cfg.d)]
        self.s2 = [np.zeros(cfg.core_size(k), np.float32) for k in range(cfg.d)]


def apply_update_f32(cfg, cores, grads, opt: OptState32) -> int:
    flat = [c.reshape(-1) for c in cores]
    for c in flat:
        assert c.dtype == np.float32 and c.flags.c_contiguous
    g = [_f32(x).ravel() for x in grads]
    step = C.c_int64(opt.step)
    rc = lib().or_apply_update_f32(C.byref(to_c(cfg)), _ptrs32(flat), _ptrs32(g), C.c_int(opt.kind),
                                   C.c_double(opt.lr), C.c_double(opt.beta1), C.c_double(opt.beta2),
                                   C.c_double(opt.eps), C.byref(step), _ptrs32(opt.s1), _ptrs32(opt.s2))
    opt.step = step.value
    return rc


def ttm_entry(cfg, cores, row: int, col: int) -> float:
    cores = [_f64(c).ravel() for c in cores]
    return lib().or_ttm_entry(C.byref(to_c(cfg)), _ptrs(cores), C.c_int64(row), C.c_int64(col))


def sort_unique(keys):
    """(perm int64[B] -- stable, unique int64[U])."""
    keys = _i64(keys)
    B = len(keys)
    perm = np.zeros(max(B, 1), np.int64)
    uniq = np.zeros(max(B, 1), np.int64)
    U = lib().or_sort_unique(keys.ctypes.data_as(C.c_void_p), C.c_int64(B),
                             perm.ctypes.data_as(C.c_void_p), uniq.ctypes.data_as(C.c_void_p))
    return perm[:B], uniq[:U]


def prefix_counts(cfg, idx):
    idx = _i64(idx)
    counts = np.zeros(len(cfg.row_factors), np.int64)
    lib().or_prefix_counts(C.byref(to_c(cfg)), idx.ctypes.data_as(C.c_void_p), C.c_int64(len(idx)),
                           counts.ctypes.data_as(C.c_void_p))
    return [int(x) for x in counts]


def num_threads() -> int:
    return lib().or_num_threads()


# ---- the reference's own tt_config.cpp (oracle/_ref) ------------------------
def _ref_args(cfg):
    d = len(cfg.row_factors)
    m, n, R = _i64(cfg.row_factors), _i64(cfg.col_factors), _i64(cfg.ranks)
    keep = (m, n, R)
    return keep, (C.c_int64(cfg.num_nodes), C.c_int64(cfg.emb_dim), C.c_int32(d),
                  m.ctypes.data_as(C.c_void_p), n.ctypes.data_as(C.c_void_p), R.ctypes.data_as(C.c_void_p))


def ref_count_params(cfg) -> int:
    keep, a = _ref_args(cfg)
    return ref().ref_count_params(*a)


def ref_validate(cfg) -> int:
    keep, a = _ref_args(cfg)
    return ref().ref_validate(*a)


def ref_digits(cfg, rows):
    """(digits int64[count, d], first row that threw out_of_range or -1)."""
    keep, a = _ref_args(cfg)
    rows = _i64(rows)
    d = len(cfg.row_factors)
    parts = np.zeros((len(rows), d), np.int64)
    bad = ref().ref_index_to_coordinate(*a, rows.ctypes.data_as(C.c_void_p), C.c_int64(len(rows)),
                                        parts.ctypes.data_as(C.c_void_p))
    return parts, int(bad)


def ref_plan_auto(M: int, N: int, d: int, ranks, ortho_friendly: bool = True):
    R = _i64(ranks)
    m = np.zeros(d, np.int64)
    n = np.zeros(d, np.int64)
    rc = ref().ref_plan_auto(C.c_int64(M), C.c_int64(N), C.c_int32(d), R.ctypes.data_as(C.c_void_p),
                             C.c_int(1 if ortho_friendly else 0), m.ctypes.data_as(C.c_void_p),
                             n.ctypes.data_as(C.c_void_p))
    return (None if rc else ([int(x) for x in m], [int(x) for x in n]))
