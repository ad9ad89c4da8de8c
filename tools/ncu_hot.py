#!/usr/bin/env python
"""List the SASS instructions of an `ncu --page source --csv` export in
address order with their stall samples (>= threshold) and execution counts,
de-duplicated; region sums help attribute time to warp roles."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 20
hdr = rows[1]
i_s = hdr.index("Warp Stall Sampling (All Samples)")
i_src, i_addr = hdr.index("Source"), hdr.index("Address")
i_ex = hdr.index("Instructions Executed")
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]


def f(x):
    try:
        return float(x or 0)
    except ValueError:
        return None


seen, data = set(), []
for r in rows[2:]:
    if len(r) != len(hdr) or f(r[i_s]) is None or r[i_addr] in seen:
        continue
    seen.add(r[i_addr])
    data.append(r)
tot = sum(f(r[i_s]) for r in data)
print(f"total samples {tot:.0f}")
for r in data:
    v = f(r[i_s])
    if v >= thr:
        top = max(reasons, key=lambda h: f(r[hdr.index(h)]) or 0)
        print(f"{r[i_addr][-5:]} {v:7.0f} {100 * v / tot:5.1f}% {top[6:]:18s} ex={r[i_ex]:>9s} "
              f"{r[i_src][:90]}")
