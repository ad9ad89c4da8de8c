#!/usr/bin/env python
"""Summarise an `ncu --page source --csv` export: top instructions by stall
samples and the stall-reason mix (excluding samples at EXIT)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
def _num(x):
    try:
        float(x or 0)
        return True
    except ValueError:
        return False


data = [r for r in rows[2:] if len(r) == len(hdr)]
i_s = hdr.index("Warp Stall Sampling (All Samples)")
i_src = hdr.index("Source")
data = [r for r in data if _num(r[i_s])]
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = sum(float(r[i_s] or 0) for r in data if "EXIT" not in r[i_src])
mix = {h: sum(float(r[hdr.index(h)] or 0) for r in data if "EXIT" not in r[i_src]) for h in reasons}
print(f"samples (excluding EXIT): {tot:.0f}")
for h, v in sorted(mix.items(), key=lambda kv: -kv[1])[:8]:
    print(f"  {h:24s} {100 * v / max(tot, 1):5.1f}%")
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
for r in sorted(data, key=lambda r: -float(r[i_s] or 0))[:n]:
    if "EXIT" in r[i_src]:
        continue
    top = max(reasons, key=lambda h: float(r[hdr.index(h)] or 0))
    print(f"{float(r[i_s]):7.0f} {100 * float(r[i_s]) / max(tot, 1):5.1f}% {top:18s} {r[i_src][:90]}")
