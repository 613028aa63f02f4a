"""Where a k_tc_bwd2 CTA's time goes (TT_TC_TRACE=1): thread 0's clock cycles
per phase summed per CTA, averaged over the CTAs.  usage:
  python scripts/tc_bwd2_phases.py [config] [path]"""
import ctypes as C
import os
import sys

os.environ["TT_TC_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2206_10581_b200 import engine as E  # noqa: E402
from paper_2206_10581_b200.config import workload_inputs  # noqa: E402

cfgname = sys.argv[1] if len(sys.argv) > 1 else "papers"
cfg, idx, up, cores = workload_inputs(cfgname, 2026)
emb = E.TTEmbedding(cfg, 0)
emb.set_cores(cores)
emb.set_path(sys.argv[2] if len(sys.argv) > 2 else "tc")
ti, tu = torch.tensor(idx, device="cuda"), torch.tensor(up, device="cuda")
for _ in range(3):
    emb.forward(ti)
    emb.backward(tu)
emb.sync()
lib = E.load_library()
lib.tt_debug_trace.restype = C.c_int64
buf = np.zeros(4096 * 64, np.int64)
lib.tt_debug_trace(buf.ctypes.data_as(C.POINTER(C.c_longlong)), buf.size)
ph = buf[:148 * 16].reshape(148, 16)
names = ["wait MMA(t-1)", "new item: dG drain + slice", "store planes", "barrier", "dA drain / issue",
         "advance + prep", "loads / dC(t+1)", "tiles", "prologue", "tail"]
if os.environ.get("TT_TCBWD", "4") == "4":  # k_tc_bwd3 (built with -DTT_BWD3_TRACE)
    names = ["-", "B: wait dG done", "B: write A + dC^T", "dA dst", "D: wait dA done",
             "D: stage S + write dC", "D: dA TMEM read", "tiles", "dA store + next A loads", "dG drain"]
tot = ph[:, [0, 1, 2, 3, 4, 5, 6, 8, 9]].sum(1)
print(f"{cfgname}: CTAs {int((ph[:, 7] > 0).sum())}, tiles/CTA mean {ph[:, 7].mean():.1f} "
      f"(min {ph[:, 7].min()}, max {ph[:, 7].max()}), cycles/CTA mean {tot.mean():.0f} max {tot.max():.0f}")
for k, n in enumerate(names):
    if k == 7:
        continue
    v = ph[:, k]
    print(f"  {n:28s} {v.mean():12.0f} cyc  {100 * v.mean() / tot.mean():5.1f}%  per tile {v.mean() / max(1, ph[:, 7].mean()):8.0f}")
