"""Phase clocks of the single-CTA plan (k_plan_small) at a small batch:
TT_PS_TRACE=1, thread 0's clock64 at the end of each phase.
usage: python scripts/plan_small_phases.py [config]"""
import ctypes as C
import os
import sys

os.environ["TT_PS_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2206_10581_b200 import engine as E  # noqa: E402
from paper_2206_10581_b200.config import workload_inputs  # noqa: E402

cfgname = sys.argv[1] if len(sys.argv) > 1 else "small"
cfg, idx, up, cores = workload_inputs(cfgname, 2026)
emb = E.TTEmbedding(cfg, 0)
emb.set_cores(cores)
ti = torch.tensor(idx, device="cuda")
for _ in range(3):
    emb.forward(ti)
emb.sync()
lib = E.load_library()
lib.tt_debug_trace.restype = C.c_int64
buf = np.zeros(4096 * 64, np.int64)
lib.tt_debug_trace(buf.ctypes.data_as(C.POINTER(C.c_longlong)), buf.size)
n = int(buf[15])
names = ["validate + keys", "sort", "keys out + unique", "prefix levels", "last level", "digit orders",
         "group offsets"]
t = buf[:n]
tot = t[-1] - t[0]
print(f"{cfgname}: k_plan_small {tot} cycles (~{tot / 1.9e3:.1f} us at 1.9 GHz)")
for k in range(1, n):
    print(f"  {names[k - 1] if k - 1 < len(names) else k:20s} {t[k] - t[k - 1]:8d} cyc {100 * (t[k] - t[k - 1]) / tot:5.1f}%")
