"""Stall samples / executed instructions of an ncu SASS source page, summed
over address ranges: python scripts/sass_regions.py page.csv name:lo-hi ..."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
data = []
for r in rows[2:]:
    if r and r[0] == "Kernel Name":
        break
    data.append(r)
tot = sum(float(r[ix["Warp Stall Sampling (All Samples)"]] or 0) for r in data)
toti = sum(float(r[ix["Instructions Executed"]] or 0) for r in data)
for spec in sys.argv[2:]:
    name, rng = spec.split(":")
    lo, hi = (int(x, 16) for x in rng.split("-"))
    s = i = 0
    st = {h: 0.0 for h in stalls}
    for r in data:
        a = int(r[ix["Address"]], 16) & 0xFFFFF
        if lo <= a < hi:
            s += float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
            i += float(r[ix["Instructions Executed"]] or 0)
            for h in stalls:
                st[h] += float(r[ix[h]] or 0)
    top = sorted(st.items(), key=lambda x: -x[1])[:4]
    print(f"{name:10s} samples {100 * s / tot:5.1f}%  inst {100 * i / toti:5.1f}%  " +
          ", ".join(f"{k[6:]} {100 * v / tot:.1f}" for k, v in top))
