#!/usr/bin/env python
"""Per-kernel DRAM traffic of one training step from an ncu CSV captured with

    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
        --clock-control none --csv --log-file gpurun_out/traffic.csv \
        python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-graph

    python tools/traffic_summary.py gpurun_out/traffic.csv profiles/rNN_traffic.json

Steps are delimited by `k_scaler_finish`; the last complete step is used.
Output: {kernel family: {launches, ms, dram_bytes_per_launch, ...}} plus the
tcgen05 GEMM aggregate that bench.py reports as roofline.traffic.
"""
import collections
import csv
import json
import re
import sys


def main():
    src, out = sys.argv[1], sys.argv[2]
    rows = list(csv.reader(open(src)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr, data = rows[hi], rows[hi + 1:]
    i_id, i_name = hdr.index("ID"), hdr.index("Kernel Name")
    i_metric, i_unit, i_val = hdr.index("Metric Name"), hdr.index("Metric Unit"), \
        hdr.index("Metric Value")
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-6, "us": 1e-3,
             "ms": 1.0, "usecond": 1e-3, "nsecond": 1e-6, "msecond": 1.0}
    launches = collections.OrderedDict()
    for r in data:
        d = launches.setdefault(r[i_id], {"name": r[i_name]})
        d[r[i_metric]] = float(r[i_val].replace(",", "")) * scale.get(r[i_unit], 1.0)
    seq = list(launches.values())
    ends = [i for i, d in enumerate(seq) if "k_scaler_finish" in d["name"]]
    step = seq[ends[-2] + 1:ends[-1] + 1] if len(ends) >= 2 else seq
    fam = collections.defaultdict(lambda: {"launches": 0, "ms": 0.0, "dram_bytes": 0.0})
    for d in step:
        if "nnl::" not in d["name"]:
            continue  # e.g. bench.py's GPU-lead spins around profiled nodes
        k = re.sub(r"\(.*", "", d["name"]).replace("void ", "").replace("<unnamed>::", "")
        k = re.sub(r"<.*", "", k)
        f = fam[k]
        f["launches"] += 1
        f["ms"] += d.get("gpu__time_duration.sum", 0.0)
        f["dram_bytes"] += d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
    res = {k: {"launches": v["launches"], "ms": round(v["ms"], 4),
               "dram_bytes_per_launch": round(v["dram_bytes"] / max(v["launches"], 1)),
               "dram_GBps": round(v["dram_bytes"] / max(v["ms"], 1e-9) / 1e6, 1)}
           for k, v in sorted(fam.items(), key=lambda kv: -kv[1]["ms"])}
    json.dump({"source": src, "step_launches": len(step), "kernels": res}, open(out, "w"),
              indent=1)
    for k, v in res.items():
        print(f"{v['ms']:8.3f} ms {v['launches']:4d} {v['dram_bytes_per_launch'] / 1e6:9.1f} MB/launch "
              f"{v['dram_GBps']:8.1f} GB/s  {k}")


if __name__ == "__main__":
    main()
