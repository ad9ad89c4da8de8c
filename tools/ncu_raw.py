#!/usr/bin/env python
"""Key raw counters per kernel of an ncu --set full report (one line each):
duration, tensor-pipe activity and fp16 MMA throughput, DRAM and L2->SM bytes,
active vs elapsed cycles, and the top warp-stall reasons.

    python tools/ncu_raw.py report.ncu-rep
"""
import csv
import subprocess
import sys

KEYS = [  # (label, metric, target unit)
    ("us", "gpu__time_duration.sum", "us"),
    ("grid", "launch__grid_size", ""),
    ("tc_act%", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", ""),
    ("f16mma%", "sm__ops_path_tensor_src_fp16_dst_fp32.avg.pct_of_peak_sustained_elapsed", ""),
    ("dramRdMB", "dram__bytes_read.sum", "MB"),
    ("dramWrMB", "dram__bytes_write.sum", "MB"),
    ("l2smMB", "l1tex__m_xbar2l1tex_read_bytes.sum", "MB"),
    ("active", "smsp__cycles_active.avg", ""),
    ("elapsed", "sm__cycles_elapsed.avg", ""),
]
SCALE = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "second": 1e6, "byte": 1e-6,
         "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3, "Tbyte": 1e6}


def main():
    out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units, data = rows[0], rows[1], rows[2:]
    iname = hdr.index("Kernel Name")
    stall = [i for i, h in enumerate(hdr)
             if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio")]
    print("kernel".ljust(46) + "".join(k.rjust(10) for k, _, _ in KEYS) + "  top stalls")
    for r in data:
        vals = []
        for _, m, tgt in KEYS:
            try:
                i = hdr.index(m)
                v = float(r[i].replace(",", "")) * (SCALE.get(units[i], 1.0) if tgt else 1.0)
                vals.append(f"{v:10.3g}")
            except (ValueError, IndexError):
                vals.append("-".rjust(10))
        st = []
        for i in stall:
            try:
                st.append((float(r[i]), hdr[i].split("stalled_")[1].replace("_per_issue_active.ratio", "")))
            except ValueError:
                pass
        st.sort(reverse=True)
        print(r[iname][:46].ljust(46) + "".join(vals) + "  " +
              ", ".join(f"{n} {v:.1f}" for v, n in st[:4]))


if __name__ == "__main__":
    main()
