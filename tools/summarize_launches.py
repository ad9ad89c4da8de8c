#!/usr/bin/env python
"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list of
`bench.py` into one training step's kernel shares.

    python tools/summarize_launches.py gpurun_out/launches.csv profiles/rNN_launches [--step K]

Steps are delimited by the solver's `k_scaler_finish` launch (one per step).
Writes <out>.txt (per-kernel time share of the chosen step) and <out>.csv (the
raw per-launch rows of that step).  ncu serialises launches and runs them
cold-cache, so compare SHARES with the bench line, not absolute times.
"""
import argparse
import collections
import csv
import re


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("out")
    ap.add_argument("--step", type=int, default=-4,
                    help="index among complete steps (bench.py ends with two profiled eager steps)")
    args = ap.parse_args()
    rows = list(csv.reader(open(args.csv)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr, data = rows[hi], rows[hi + 1:]
    i_name, i_val = hdr.index("Kernel Name"), hdr.index("Metric Value")
    ends = [i for i, r in enumerate(data) if "k_scaler_finish" in r[i_name]]
    spans = [(a + 1, b + 1) for a, b in zip(ends, ends[1:])]
    lo, hi_ = spans[args.step]
    step = data[lo:hi_]
    total = sum(float(r[i_val]) for r in step) / 1e6
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in step:
        k = re.sub(r"\(.*", "", r[i_name]).replace("void ", "")
        agg[k][0] += 1
        agg[k][1] += float(r[i_val]) / 1e6
    with open(args.out + ".txt", "w") as f:
        f.write(f"# one training step from {args.csv}: {len(step)} launches, "
                f"{total:.3f} ms serialised (ncu, cold cache)\n")
        f.write(f"{'ms':>9s} {'share':>6s} {'n':>4s}  kernel\n")
        for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
            f.write(f"{t:9.3f} {100 * t / total:5.1f}% {n:4d}  {k}\n")
    with open(args.out + ".csv", "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["Kernel Name", "Grid Size", "Block Size", "gpu__time_duration.sum (ns)"])
        for r in step:
            w.writerow([r[i_name][:160], r[hdr.index("Grid Size")], r[hdr.index("Block Size")],
                        r[i_val]])
    print(open(args.out + ".txt").read())


if __name__ == "__main__":
    main()
