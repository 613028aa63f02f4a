"""Hot SASS regions / opcodes from `ncu --page source --csv --print-source sass`."""
import csv
import re
import sys
from collections import defaultdict


def f(v):
    try:
        return float(v)
    except ValueError:
        return 0.0


def main(path, block=48, top=14):
    r = list(csv.reader(open(path)))
    hdr = [row for row in r if "Address" in row][0]
    rows = [dict(zip(hdr, x)) for x in r if len(x) == len(hdr) and "Address" not in x]
    key = "Warp Stall Sampling (All Samples)"
    tot = sum(f(x[key]) for x in rows) or 1
    ops = defaultdict(lambda: [0, 0.0])
    for x in rows:
        op = re.sub(r"^@!?U?P\w+\s+", "", x["Source"].strip()).split(" ")[0]
        ops[op][0] += int(f(x["Instructions Executed"]))
        ops[op][1] += f(x[key])
    ninst = sum(v[0] for v in ops.values())
    print(f"{path}: {len(rows)} SASS, {ninst} warp-inst executed")
    for op, (n, s) in sorted(ops.items(), key=lambda kv: -kv[1][1])[:12]:
        print(f"  {op:16s} inst {n / ninst * 100:5.1f}%  stall {100 * s / tot:5.1f}%")
    out = []
    for i in range(0, len(rows), block):
        seg = rows[i:i + block]
        s = sum(f(x[key]) for x in seg)
        n = sum(f(x["Instructions Executed"]) for x in seg)
        ff = sum(f(x["Instructions Executed"]) for x in seg if "FFMA" in x["Source"])
        reasons = defaultdict(float)
        for x in seg:
            for k2, v in x.items():
                if k2.startswith("stall_") and "Not Issued" not in k2:
                    reasons[k2] += f(v)
        rs = ",".join(f"{k2[6:]}:{v / max(s, 1) * 100:.0f}" for k2, v in sorted(reasons.items(), key=lambda kv: -kv[1])[:3])
        out.append((s / tot * 100, i, n / ninst * 100, ff / max(n, 1) * 100, rs))
    for s, i, n, ff, rs in sorted(out, reverse=True)[:top]:
        print(f"  @{i:5d} stall {s:5.1f}%  inst {n:5.1f}%  ffma {ff:3.0f}%  [{rs}]  {rows[i]['Source'].strip()[:50]}")


if __name__ == "__main__":
    main(sys.argv[1])
