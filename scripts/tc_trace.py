"""Per-CTA phase timeline of the tcgen05 backward (TT_TC_TRACE=1 builds the
trace buffer): entry, batch start, prep done, per tile (planes ready / under
MMA done / MMA done), exit.  Prints where a CTA's time goes."""
import ctypes as C
import os
import sys

import numpy as np

FWD = os.environ.get("TRACE_KERNEL") == "fwd"
os.environ["TT_TC_TRACE"] = "2" if FWD else "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2206_10581_b200 import engine as E  # noqa: E402
from paper_2206_10581_b200.config import workload_inputs  # noqa: E402

cfg, idx, up, cores = workload_inputs("papers", 2026)
emb = E.TTEmbedding(cfg, 0)
emb.set_cores(cores)
emb.set_path(os.environ.get("TRACE_PATH", "tc"))
ti, tu = torch.tensor(idx, device="cuda"), torch.tensor(up, device="cuda")
for _ in range(2):
    emb.forward(ti)
    emb.backward(tu)
if FWD:
    emb.forward(ti)
emb.sync()
def fwd_report(buf):
    # per CTA 4 x 256 stamps: MMA issued, epilogue has acc, epilogue done, A handed over
    T = buf[: 256 * 1024].reshape(256, 4, 256).astype(np.float64)
    ctas = [b for b in range(256) if T[b, 0, 0] > 0]
    t0 = min(T[b, 0, 0] for b in ctas)
    gaps, epi, lag, lead = [], [], [], []
    for b in ctas:
        nt = int((T[b, 0] > 0).sum())
        mma, e1, e2, ld = T[b, 0, :nt], T[b, 1, :nt], T[b, 2, :nt], T[b, 3, :nt]
        gaps += list(np.diff(mma) / 1e3)
        epi += list((e2 - e1) / 1e3)
        lag += list((e1 - mma) / 1e3)
        lead += list((mma - ld) / 1e3)
    print(f"CTAs {len(ctas)}  tiles/CTA {np.mean([(T[b, 0] > 0).sum() for b in ctas]):.1f}  span {(max(T[b, 2][T[b, 2] > 0].max() for b in ctas) - t0) / 1e3:.1f} us")
    for nm, v in (("MMA issue -> next MMA issue", gaps), ("epilogue (acc -> done)", epi),
                  ("MMA issue -> epilogue has acc", lag), ("A handed over -> MMA issue", lead)):
        v = np.array(v)
        print(f"  {nm:32s} mean {v.mean():6.2f}  median {np.median(v):6.2f}  p90 {np.quantile(v, .9):6.2f} us")
    first = np.array([(T[b, 0, 0] - t0) / 1e3 for b in ctas])
    print(f"  first MMA after kernel start: mean {first.mean():.2f} us")


lib = E.load_library()
lib.tt_debug_trace.restype = C.c_int64
buf = np.zeros(4096 * 64, np.int64)
lib.tt_debug_trace(buf.ctypes.data_as(C.POINTER(C.c_longlong)), buf.size)
tr = buf.reshape(4096, 64)
if FWD:
    fwd_report(buf)
    sys.exit(0)
n = tr[:, 0]
live = np.flatnonzero(n > 2)
t0 = tr[live, 1].min()
dur = np.array([tr[i, n[i]] - tr[i, 1] for i in live]) / 1e3
start = (tr[live, 1] - t0) / 1e3
end = np.array([tr[i, n[i]] for i in live] - t0) / 1e3
print(f"CTAs {len(live)}  kernel span {end.max():.1f} us  CTA duration mean {dur.mean():.2f} median {np.median(dur):.2f} max {dur.max():.2f} us")
# prologue: entry -> batch start -> prep done -> first planes-ready
pro = np.array([tr[i, 4] - tr[i, 1] for i in live]) / 1e3
print(f"prologue (entry -> first tile's planes ready) mean {pro.mean():.2f} us")
# per tile: consecutive (planes ready, pre-wait, post-wait) triples
tiles = []
for i in live:
    k = 4
    while k + 3 <= n[i]:
        p = [tr[i, k + j] for j in range(4)]
        nxt = tr[i, k + 4] if k + 4 <= n[i] else p[3]
        tiles.append([(p[j + 1] - p[j]) / 1e3 for j in range(3)] + [(nxt - p[3]) / 1e3])
        k += 4
tiles = np.array(tiles)
names = ["A(t+1) loads", "dC(t+1)", "MMA wait", "epilogue(t)+planes(t+1)+sync"]
if os.environ.get("TRACE_PATH") == "auto":
    t3 = []
    for i in live:
        k = 2
        while k + 3 <= n[i]:
            p = [tr[i, k + j] for j in range(4)]
            t3.append([(p[1] - p[0]) / 1e3, (p[2] - p[1]) / 1e3, (p[3] - p[2]) / 1e3])
            k += 3
    t3 = np.array(t3)
    print("FFMA bwd tiles %d: A load + dC + sync %.2f, dG %.2f, dA + store + sync %.2f us" % ((len(t3),) + tuple(t3.mean(0))))
    sys.exit(0)
print(f"tiles {len(tiles)}: " + "; ".join(f"{nm} {tiles[:, j].mean():.2f}" for j, nm in enumerate(names)) + " us")
pre = np.array([[(tr[i, j + 1] - tr[i, j]) / 1e3 for j in (1, 2, 3)] for i in live])
print("prologue: alloc+S staging %.2f, prep %.2f, first A+dC+planes %.2f us" % tuple(pre.mean(0)))
gaps = np.sort(start)
print("CTA start quantiles (us):", np.round(np.quantile(start, [0, .1, .5, .9, 1]), 1))
