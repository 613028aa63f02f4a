"""In-process stand-in for the torch.distributed calls dist.py makes, one
thread per rank.  The exchange is host-side (tensors handed between threads,
stream-ordered on the shared device), so no kernel waits on another rank --
the multi-rank data flow of OwnerShardedTT runs with the real CUDA engine on
one GPU without emulating NCCL (B200_PROFILING.md: never run ranks whose
kernels wait on one another as separate launches on one GPU)."""
import threading

import torch


class ThreadComm:
    def __init__(self, world):
        self.world = world
        self._bar = threading.Barrier(world)
        self._slots = [None] * world
        self._tls = threading.local()

    def bind(self, rank):
        self._tls.rank = rank

    def is_initialized(self):
        return True

    def get_world_size(self, group=None):
        return self.world

    def get_rank(self, group=None):
        return self._tls.rank

    def _exchange(self, obj):
        r = self._tls.rank
        self._slots[r] = obj
        self._bar.wait()
        got = list(self._slots)
        self._bar.wait()
        return got

    def all_to_all_single(self, out, inp, out_splits=None, in_splits=None, group=None):
        n = self.world
        if in_splits is None:
            in_splits = [inp.shape[0] // n] * n
        chunks = [c.clone() for c in torch.split(inp, list(in_splits))]
        got = self._exchange(chunks)
        r = self._tls.rank
        parts = [got[src][r].to(out.device) for src in range(n)]
        if out.shape[0]:
            torch.cat(parts, out=out)

    def all_reduce(self, t, group=None):
        got = self._exchange(t.clone())
        acc = got[0].to(t.device).clone()
        for x in got[1:]:  # fixed rank order: every rank gets the same bits
            acc += x.to(t.device)
        t.copy_(acc)

    def all_gather(self, lst, t, group=None):
        got = self._exchange(t.clone())
        for i, x in enumerate(got):
            lst[i].copy_(x.to(lst[i].device))


def run_ranks(world, fn):
    """Run fn(rank, comm) in `world` threads; re-raise the first failure."""
    comm = ThreadComm(world)
    errs = [None] * world

    def body(r):
        comm.bind(r)
        try:
            fn(r, comm)
        except BaseException as e:  # noqa: BLE001
            errs[r] = e
            comm._bar.abort()

    th = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for e in errs:
        if e is not None and not isinstance(e, threading.BrokenBarrierError):
            raise e
    for e in errs:
        if e is not None:
            raise e
