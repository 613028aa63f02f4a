"""Seeded, portable synthetic inputs for the TT-embedding workloads.

BASELINE.json's configs are shaped after OGB datasets; no
dataset content is used.  Every stream here is a pure function of
(seed, stream id, counter) built on splitmix64, so the CPU oracle and the GPU
engine always receive identical host buffers on any machine, and a batch of
one million IDs is generated in a few vectorised numpy passes:

* uniforms: splitmix64(key ^ splitmix64(counter)), top 53 bits;
* normals: Box-Muller on two uniforms;
* bounded integers: Lemire's multiply-shift ((v >> 32) * n) >> 32, n <= 2^32;
* Zipf(alpha) over ranks 1..N: inverse CDF with an exact head table
  (ranks <= 2^20) and the analytic integral for the tail;
* "seeded permutation": a keyed 4-round Feistel bijection on the smallest
  even-bit power-of-two domain >= N, with cycle-walking back into [0, N),
  so no N-sized table is ever built (N = 1e9 at the billion config).

The reference draws its fixtures from std::mt19937_64 + std::normal_distribution
(initializer.cpp:91-101, ttgnn_main.cpp:203-210), whose normal stream is
implementation-defined; SURVEY 8(d) therefore makes the generator
builder-chosen and recorded.
"""
from __future__ import annotations

import math

import numpy as np

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)
_GOLD = np.uint64(0x9E3779B97F4A7C15)
_C1 = np.uint64(0xBF58476D1CE4E5B9)
_C2 = np.uint64(0x94D049BB133111EB)


def splitmix64(x: np.ndarray) -> np.ndarray:
    x = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = x + _GOLD
        z = (z ^ (z >> np.uint64(30))) * _C1
        z = (z ^ (z >> np.uint64(27))) * _C2
    return z ^ (z >> np.uint64(31))


def _key(seed: int, stream: int) -> np.uint64:
    with np.errstate(over="ignore"):
        s = np.uint64(seed & 0xFFFFFFFFFFFFFFFF) ^ (np.uint64(stream) * np.uint64(0xD1B54A32D192ED03))
    return splitmix64(np.array([s], dtype=np.uint64))[0]


def raw64(seed: int, stream: int, n: int, offset: int = 0) -> np.ndarray:
    ctr = np.arange(offset, offset + n, dtype=np.uint64)
    return splitmix64(_key(seed, stream) ^ splitmix64(ctr))


def uniform01(seed: int, stream: int, n: int) -> np.ndarray:
    """Uniform doubles in [0, 1) from the top 53 bits."""
    return (raw64(seed, stream, n) >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)


def normal(seed: int, stream: int, n: int, std: float = 1.0, dtype=np.float32) -> np.ndarray:
    """Box-Muller: z = sqrt(-2 ln u1) cos(2 pi u2), u1 in (0, 1]."""
    v = raw64(seed, stream, 2 * n)
    u1 = ((v[0::2] >> np.uint64(11)).astype(np.float64) + 1.0) * (1.0 / 9007199254740992.0)
    u2 = (v[1::2] >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)
    z = np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * math.pi * u2)
    return (z * std).astype(dtype)


def bounded(seed: int, stream: int, n: int, bound: int) -> np.ndarray:
    """Integers uniform in [0, bound) (Lemire multiply-shift), bound <= 2^32."""
    if not 0 < bound <= (1 << 32):
        raise ValueError("bound must be in (0, 2^32]")
    v = raw64(seed, stream, n) >> np.uint64(32)
    with np.errstate(over="ignore"):
        return ((v * np.uint64(bound)) >> np.uint64(32)).astype(np.int64)


class FeistelPermutation:
    """Keyed bijection of [0, n) (4-round Feistel + cycle walking)."""

    def __init__(self, n: int, seed: int, rounds: int = 4):
        if n <= 0:
            raise ValueError("n must be positive")
        self.n = n
        bits = max(2, (n - 1).bit_length())
        bits += bits & 1
        self.half = bits // 2
        self.mask = np.uint64((1 << self.half) - 1)
        self.keys = [_key(seed, 1000 + r) for r in range(rounds)]

    def _round(self, x: np.ndarray) -> np.ndarray:
        h = np.uint64(self.half)
        left, right = x >> h, x & self.mask
        for k in self.keys:
            left, right = right, left ^ (splitmix64(right ^ k) & self.mask)
        return (left << h) | right

    def __call__(self, x: np.ndarray) -> np.ndarray:
        x = self._round(np.asarray(x, dtype=np.uint64))
        bad = x >= np.uint64(self.n)
        while bad.any():
            x[bad] = self._round(x[bad])
            bad = x >= np.uint64(self.n)
        return x.astype(np.int64)


def zipf_ranks(seed: int, stream: int, n: int, alpha: float, N: int, head: int = 1 << 20) -> np.ndarray:
    """Ranks in [1, N] with P(k) proportional to k^-alpha (alpha != 1)."""
    H = min(N, head)
    k = np.arange(1, H + 1, dtype=np.float64)
    cum = np.cumsum(k ** (-alpha))
    head_mass = float(cum[-1])
    a1 = 1.0 - alpha
    tail_mass = 0.0
    if N > H:
        tail_mass = ((N + 0.5) ** a1 - (H + 0.5) ** a1) / a1
    u = uniform01(seed, stream, n) * (head_mass + tail_mass)
    out = np.empty(n, dtype=np.int64)
    in_head = u < head_mass
    out[in_head] = np.searchsorted(cum, u[in_head], side="right") + 1
    if N > H:
        ut = u[~in_head] - head_mass
        x = ((H + 0.5) ** a1 + a1 * ut) ** (1.0 / a1)
        out[~in_head] = np.clip(np.floor(x + 0.5).astype(np.int64), H + 1, N)
    np.clip(out, 1, N, out=out)
    return out


def zipf_ids(seed: int, n: int, alpha: float, num_nodes: int) -> np.ndarray:
    """Zipf(alpha) over a seeded permutation of [0, num_nodes)."""
    ranks = zipf_ranks(seed, 11, n, alpha, num_nodes)
    return FeistelPermutation(num_nodes, seed)(ranks - 1)


def uniform_ids(seed: int, n: int, num_nodes: int) -> np.ndarray:
    return bounded(seed, 12, n, num_nodes)


def locality_ids(seed: int, n: int, num_nodes: int, block: int, run: int = 1024,
                 frac_local: float = 0.8) -> np.ndarray:
    """Rank-sweep batches (BASELINE configs[3]): frac_local of the IDs come in
    runs of `run` IDs drawn uniformly inside one i_1 block of `block`
    consecutive rows (a block shares i_1); the rest are uniform."""
    n_local = int(n * frac_local) // run * run
    nruns = n_local // run
    nblocks = -(-num_nodes // block)
    blk = bounded(seed, 13, max(nruns, 1), nblocks)[:nruns]
    lo = blk * block
    size = np.minimum(lo + block, num_nodes) - lo
    off = (uniform01(seed, 14, n_local) * np.repeat(size, run)).astype(np.int64)
    local = np.repeat(lo, run) + off
    rest = bounded(seed, 15, n - n_local, num_nodes)
    return np.concatenate([local, rest]).astype(np.int64)


def gaussian_cores(cfg, seed: int, std: float = 0.1, dtype=np.float32):
    """Cores i.i.d. N(0, std^2) in the reference layout (R_{k-1}, m_k, n_k, R_k)
    (tt_embedding.hpp:28-32), one stream per core."""
    cores = []
    for k in range(cfg.d):
        shape = (cfg.R[k], cfg.m[k], cfg.n[k], cfg.R[k + 1])
        size = int(np.prod(shape))
        cores.append(normal(seed, 100 + k, size, std, dtype).reshape(shape))
    return cores


def checksum(a: np.ndarray) -> str:
    """Order-sensitive 64-bit checksum of a buffer's bytes (for run records)."""
    b = np.ascontiguousarray(a).reshape(-1).view(np.uint8)
    pad = (-len(b)) % 8
    w = np.concatenate([b, np.zeros(pad, np.uint8)]).view(np.uint64)
    h = splitmix64(w ^ splitmix64(np.arange(len(w), dtype=np.uint64)))
    return "%016x" % int(np.bitwise_xor.reduce(h) if len(h) else 0)
