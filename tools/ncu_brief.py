#!/usr/bin/env python
"""One line per kernel of an ncu report: duration, DRAM / L2 / SM throughput,
occupancy, registers.   python tools/ncu_brief.py report.ncu-rep"""
import csv
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "details", "--csv"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[0]
iI, iN, iM, iV = (hdr.index(k) for k in ("ID", "Kernel Name", "Metric Name", "Metric Value"))
want = ["Duration", "DRAM Throughput", "L2 Cache Throughput", "Compute (SM) Throughput",
        "Executed Ipc Active", "Achieved Occupancy", "Registers Per Thread"]
k = {}
for r in rows[1:]:
    if r[iM] in want:
        k.setdefault((r[iI], r[iN][:40]), {})[r[iM]] = r[iV]
print("kernel".ljust(42) + " | ".join(w[:12] for w in want))
for (i, n), d in k.items():
    print(n.ljust(42) + " | ".join(d.get(w, "-").rjust(12) for w in want))
