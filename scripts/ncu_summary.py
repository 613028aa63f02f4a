"""Summarise an ncu --csv launch list (gpu__time_duration.sum) per kernel."""
import csv
import sys
from collections import defaultdict

UNIT = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6}


def load(path):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    return data


def summary(path, skip_regex=None, top=30):
    import re
    agg = defaultdict(lambda: [0, 0.0])
    for d in load(path):
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = d["Kernel Name"]
        if skip_regex and re.search(skip_regex, name):
            continue
        v = float(d["Metric Value"].replace(",", "")) * UNIT.get(d["Metric Unit"], 1.0)
        key = name.split("(")[0][:70]
        agg[key][0] += 1
        agg[key][1] += v
    tot = sum(v[1] for v in agg.values())
    lines = [f"{'total_us':>10} {'n':>4} {'avg_us':>9} {'share':>6}  kernel"]
    for k, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        lines.append(f"{v:10.1f} {c:4d} {v / c:9.1f} {v / tot * 100:5.1f}%  {k}")
    lines.append(f"{tot:10.1f} total")
    return "\n".join(lines)


if __name__ == "__main__":
    print(summary(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "ffma_peak|FillFunctor"))
