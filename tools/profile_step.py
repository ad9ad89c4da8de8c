#!/usr/bin/env python
"""Per-node device-time breakdown of one ResNet-50 training step.

    python tools/profile_step.py [--batch 256] [--warmup 2] [--plain]

--plain runs warm-up + one step without CUDA events (for ncu launch lists:
`ncu --metrics gpu__time_duration.sum -s <warmup launches> -c <step launches>`).
"""

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=256)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--plain", action="store_true")
    ap.add_argument("--json", default=None)
    args = ap.parse_args()
    import torch
    import paper_2102_06725_b200 as nn
    import paper_2102_06725_b200.functions as F
    from paper_2102_06725_b200 import _lib, networks
    from paper_2102_06725_b200.communicator import DataParallelTrainer
    from paper_2102_06725_b200.profiler import PROFILER

    nn.set_default_context(nn.ExecutionContext(type_config=nn.TypeConfig.HALF))
    B = args.batch

    def build(bs):
        xv = nn.Variable((bs, 3, 224, 224))
        tv = nn.Variable((bs,))
        return {"x": xv, "label": tv,
                "loss": F.softmax_cross_entropy(networks.resnet50(xv, 1000), tv)}

    tr = DataParallelTrainer(1, B, build, lr=0.1, seed=0,
                             loss_scaling=nn.DynamicLossScaler(8.0, 2.0, 2000),
                             check_sync=False, momentum=0.9, weight_decay=1e-4)
    import numpy as np
    x = nn.RngState(1).next_uniform((B, 3, 224, 224))
    lab = (np.arange(B) % 1000).astype(np.float32)
    tr.step(x, lab)
    for _ in range(args.warmup):
        tr.step_resident()
    torch.cuda.synchronize()
    n0 = _lib.lib().nnl_launch_count(0)
    if args.plain:
        tr.step_resident()
        torch.cuda.synchronize()
        print("launches per step", _lib.lib().nnl_launch_count(0) - n0)
        return
    PROFILER.reset()
    PROFILER.enabled = True
    tr.step_resident()
    PROFILER.enabled = False
    rows = PROFILER.per_node()
    total = sum(r["ms"] for r in rows)
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    pk = peaks.get("bf16_tflops_sustained", 1400.0)
    print(f"step total {total:.2f} ms over {len(rows)} node calls")
    agg = {}
    for r in rows:
        k = (r["kind"], r["phase"], r["shape"])
        a = agg.setdefault(k, {"ms": 0.0, "flops": 0.0, "n": 0})
        a["ms"] += r["ms"]
        a["flops"] += r["flops"]
        a["n"] += 1
    print(f"{'kind.phase':28s} {'shape':38s} {'n':>3s} {'ms':>8s} {'TF/s':>8s} {'%pk':>6s}")
    for (kind, ph, shape), a in sorted(agg.items(), key=lambda kv: -kv[1]["ms"])[:60]:
        tf = a["flops"] / (a["ms"] / 1e3) / 1e12 if a["ms"] > 0 and a["flops"] else 0.0
        print(f"{kind + '.' + ph:28s} {shape:38s} {a['n']:3d} {a['ms']:8.3f} {tf:8.1f} "
              f"{100 * tf / pk:6.1f}")
    if args.json:
        with open(args.json, "w") as f:
            json.dump(rows, f)


if __name__ == "__main__":
    main()
