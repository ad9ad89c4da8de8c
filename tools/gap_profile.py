#!/usr/bin/env python
"""Kernel timeline of resident ResNet-50 training steps (CUDA-graph replay or
eager) through torch.profiler/CUPTI: GPU busy time, idle gaps between
consecutive kernels, and the kernels with the largest total time.

    python tools/gap_profile.py [--config resnet50|resnet18|lenet|mlp] [--batch B]
                                [--steps 3] [--no-graph] [--full-names]
"""
import argparse
import collections
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="resnet50")
    ap.add_argument("--batch", type=int, default=0)
    ap.add_argument("--full-names", action="store_true")
    ap.add_argument("--list", action="store_true", help="every launch of the last step, in order")
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--no-graph", action="store_true")
    args = ap.parse_args()
    import numpy as np
    import torch
    from torch.profiler import ProfilerActivity, profile

    import paper_2102_06725_b200 as nn
    import paper_2102_06725_b200.functions as F
    from paper_2102_06725_b200 import networks
    from paper_2102_06725_b200.communicator import DataParallelTrainer
    import bench
    cf = bench.CONFIGS[args.config]
    tc = nn.TypeConfig.HALF if cf["half"] else nn.TypeConfig.FLOAT
    nn.set_default_context(nn.ExecutionContext(type_config=tc))
    B = args.batch or cf["batch"]
    scaler = nn.DynamicLossScaler(*cf["scaler"]) if cf["scaler"] else None
    tr = DataParallelTrainer(1, B, lambda bs: bench.build_graph(nn, F, networks, args.config, bs),
                             lr=cf["lr"], seed=0, loss_scaling=scaler, check_sync=False,
                             momentum=cf["momentum"], weight_decay=cf["wd"])
    x = nn.RngState(1).next_uniform_device((B,) + cf["shape"], 0.0, 1.0).cpu().numpy()
    lab = (np.arange(B) % cf["classes"]).astype(np.float32)
    for _ in range(3):
        tr.step(x, lab)
    if not args.no_graph:
        tr.capture_graph()
    for _ in range(2):
        tr.step_resident()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(args.steps):
            tr.step_resident()
        torch.cuda.synchronize()
    evs = [e for e in prof.events() if e.device_type.name == "CUDA" and e.device_time_total > 0
           and "Memcpy" not in e.name and "Memset" not in e.name]
    ks = sorted(((e.time_range.start, e.time_range.end, e.name) for e in evs))
    if not ks:
        print("no kernels recorded")
        return
    busy = sum(b - a for a, b, _ in ks)
    wall = ks[-1][1] - ks[0][0]
    gaps = [max(0.0, ks[i + 1][0] - ks[i][1]) for i in range(len(ks) - 1)]
    print(f"steps {args.steps}: kernels {len(ks)}, wall {wall / 1e3 / args.steps:.3f} ms/step, "
          f"busy {busy / 1e3 / args.steps:.3f} ms/step, gaps {sum(gaps) / 1e3 / args.steps:.3f} "
          f"ms/step (median gap {sorted(gaps)[len(gaps) // 2]:.2f} us)")
    if args.list:
        per = len(ks) // args.steps
        for a, b, n in ks[-per:]:
            print(f"{(b - a):9.2f} us  {n[:150]}")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for a, b, n in ks:
        k = n if args.full_names else re.sub(r"<.*", "", re.sub(r"\(.*", "", n)).replace("void ", "")
        agg[k][0] += 1
        agg[k][1] += (b - a)
    for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:30]:
        print(f"{t / 1e3 / args.steps:8.3f} ms/step {n // args.steps:5d}  {k}")


if __name__ == "__main__":
    main()
