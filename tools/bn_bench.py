#!/usr/bin/env python
"""BatchNormalization kernel bandwidth at ResNet-50 shapes.

    python tools/bn_bench.py [--once]

Algorithmic bytes: fwd (own statistics pass) 2+2+2 B/elem (read x twice, write y);
bwd 2+2 (reduction) + 2+2+2 (apply: x, dy, dx) B/elem.
"""

import argparse
import ctypes as C
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

SHAPES = [(256, 64, 112), (256, 64, 56), (256, 256, 56), (256, 512, 28), (256, 1024, 14),
          (256, 2048, 7)]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--once", action="store_true")
    ap.add_argument("--iters", type=int, default=10)
    args = ap.parse_args()
    import torch
    from paper_2102_06725_b200 import _lib
    pk = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    hbm = pk.get("hbm_gbs", 6541.5)
    dev = torch.device("cuda")
    st = torch.cuda.current_stream().cuda_stream
    print(f"{'shape':22s} {'pass':5s} {'ms':>8s} {'GB/s':>8s} {'%hbm':>6s}")
    for n, c, hw in SHAPES:
        rows = n * hw * hw
        x = torch.randn(rows, c, device=dev, dtype=torch.float16)
        dy = torch.randn_like(x)
        y = torch.empty_like(x)
        dx = torch.empty_like(x)
        g = torch.ones(c, device=dev)
        b = torch.zeros(c, device=dev)
        rm = torch.zeros(c, device=dev)
        rv = torch.ones(c, device=dev)
        sm = torch.empty(c, device=dev)
        si = torch.empty(c, device=dev)
        dg = torch.empty(c, device=dev)
        db = torch.empty(c, device=dev)
        wsn = _lib.lib().nnl_bn_workspace_size(rows, c)
        ws = torch.empty(wsn, dtype=torch.uint8, device=dev)
        fwd = lambda: _lib.call("nnl_bn_fwd_train", 1, rows, c, x.data_ptr(), g.data_ptr(),
                                b.data_ptr(), rm.data_ptr(), rv.data_ptr(), 1e-5, 0.9, None, 0,
                                None, sm.data_ptr(), si.data_ptr(), y.data_ptr(), None, 1, ws.data_ptr(), wsn,
                                st)
        bwd = lambda: _lib.call("nnl_bn_bwd", 1, rows, c, x.data_ptr(), dy.data_ptr(), 1,
                                None, None, 0, g.data_ptr(), b.data_ptr(), sm.data_ptr(), si.data_ptr(), 1,
                                dx.data_ptr(), 0, dg.data_ptr(), 0, db.data_ptr(), 0, None, 0, None,
                                ws.data_ptr(), wsn, st)
        for name, fn, nbytes in (("fwd", fwd, 6.0 * rows * c), ("bwd", bwd, 10.0 * rows * c)):
            if args.once:
                fn()
                torch.cuda.synchronize()
                continue
            fn()
            ts = []
            for _ in range(args.iters):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                fn()
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            ms = statistics.median(ts)
            gbs = nbytes / (ms / 1e3) / 1e9
            print(f"{n}x{c}x{hw}x{hw}".ljust(22) + f" {name:5s} {ms:8.3f} {gbs:8.0f} "
                  f"{100 * gbs / hbm:6.1f}", flush=True)


if __name__ == "__main__":
    main()
