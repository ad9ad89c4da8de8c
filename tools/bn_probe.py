#!/usr/bin/env python
"""Device time of the BatchNormalization passes as the training step runs them
(statistics from the convolution epilogue, fused ReLU), each call captured
20x in a CUDA graph (no host launch gaps), against the streamed bytes:

  fwd   finalize + APPLY_F                  x, y            4 B/elem
  fwdr  finalize + APPLY_F + residual       x, res, y       6 B/elem
  bwd   STATS_B + finalize + APPLY_B        x, dy | x, dy, dx    10 B/elem
  bwdg  (residual gate) STATS_B + APPLY_B   x, dy, gate, dres | x, dy, gate, dx   14 B/elem

    python tools/bn_probe.py
"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2102_06725_b200 import _lib  # noqa: E402

SHAPES = [(256, 64, 112), (256, 64, 56), (256, 256, 56), (256, 128, 28), (256, 512, 28),
          (256, 256, 14), (256, 1024, 14), (256, 512, 7), (256, 2048, 7)]


def timeit(fn, reps=20):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(2):
            fn(s.cuda_stream)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(reps):
                fn(s.cuda_stream)
        g.replay()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        for _ in range(5):
            g.replay()
        b.record(s)
        torch.cuda.synchronize()
    return a.elapsed_time(b) * 1000 / (5 * reps)


def main():
    pk = os.path.join(ROOT, "MEASURED_PEAKS.json")
    hbm = json.load(open(pk)).get("hbm_gbs", 6541.5) if os.path.exists(pk) else 6541.5
    dev = torch.device("cuda")
    lib = _lib.lib()
    print(f"{'shape':18s} {'pass':5s} {'us':>8s} {'GB/s':>7s} {'%hbm':>6s}")
    for n, c, hw in SHAPES:
        rows = n * hw * hw
        t = lambda: torch.randn(rows, c, device=dev, dtype=torch.float16)
        x, dy, res, gate, y, dx, dres = t(), t(), t(), t(), t(), t(), t()
        f = lambda v: torch.full((c,), v, device=dev)
        g, b, rm, rv, sm, si, sh = f(1.0), f(0.0), f(0.0), f(1.0), f(0.0), f(1.0), f(0.0)
        dg, db = f(0.0), f(0.0)
        R = 148
        parts = torch.zeros(R * 2 * c, device=dev)
        parts[c:2 * c] = rows  # sum (x-K)^2 = n: var 1
        wsn = lib.nnl_bn_workspace_size(rows, c)
        ws = torch.empty(wsn, dtype=torch.uint8, device=dev)
        P = lambda a: a.data_ptr()

        def fwd(st, residual=None):
            _lib.call("nnl_bn_fwd_train", 1, rows, c, P(x), P(g), P(b), P(rm), P(rv), 1e-5, 0.9,
                      P(parts), R, P(sh), P(sm), P(si), P(y),
                      P(residual) if residual is not None else None, 1, P(ws), wsn, st)

        def bwd(st, gated=False):
            _lib.call("nnl_bn_bwd", 1, rows, c, P(x), P(dy), 0 if gated else 1,
                      P(gate) if gated else None, P(dres) if gated else None, 0, P(g), P(b),
                      P(sm), P(si), 1, P(dx), 0, P(dg), 0, P(db), 0, None, 0, None, P(ws), wsn, st)

        for name, fn, bpe in (("fwd", fwd, 4), ("fwdr", lambda st: fwd(st, res), 6),
                              ("bwd", bwd, 10), ("bwdg", lambda st: bwd(st, True), 14)):
            us = timeit(fn)
            gbs = bpe * rows * c / (us * 1e-6) / 1e9
            print(f"{n}x{c}x{hw}x{hw}".ljust(18) + f" {name:5s} {us:8.1f} {gbs:7.0f} "
                  f"{100 * gbs / hbm:6.1f}", flush=True)
        del x, dy, res, gate, y, dx, dres
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
