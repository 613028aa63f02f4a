"""Summarise an ncu source page exported as SASS CSV
(ncu -i X.ncu-rep --page source --csv --print-source sass --kernel-name K):
executed instructions and stall samples per opcode, and the hottest
non-FFMA instructions."""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
data = []
for r in rows[2:]:  # the first kernel's block only
    if r and r[0] == "Kernel Name":
        break
    data.append(r)
inst = Counter()
samp = Counter()
tot_i = tot_s = 0
hot = []
for r in data:
    if len(r) < len(hdr):
        continue
    src = r[ix["Source"]].strip()
    op = src.split()[0] if src else "?"
    if op.startswith("@"):
        op = src.split()[1]
    base = op.split(".")[0]
    n = float(r[ix["Instructions Executed"]] or 0)
    s = float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    inst[base] += n
    samp[base] += s
    tot_i += n
    tot_s += s
    hot.append((n, s, r[ix["Address"]], src))
print(f"total warp instructions {tot_i:.4g}, stall samples {tot_s:.4g}")
print(f"{'op':10s} {'inst%':>7s} {'samples%':>9s}")
for op, n in inst.most_common(25):
    print(f"{op:10s} {100 * n / tot_i:7.2f} {100 * samp[op] / max(tot_s, 1):9.2f}")
print("hottest non-FFMA instructions:")
for n, s, a, src in sorted((h for h in hot if not h[3].startswith("FFMA")), reverse=True)[:int(sys.argv[2]) if len(sys.argv) > 2 else 30]:
    print(f"  {n:12.0f} {s:8.0f} {a} {src}")
