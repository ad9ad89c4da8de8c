#!/usr/bin/env python
"""Stem-pool probe: the ResNet-50 max pooling (256x64x112x112, 3x3 s2 p1) and
the stem's space-to-depth preparation, forward + backward once each, with
CUDA-event times of the whole calls (run under ncu for per-kernel detail).

    python tools/pool_probe.py [--iters 5]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=5)
    args = ap.parse_args()
    import numpy as np
    import torch
    import paper_2102_06725_b200 as nn
    import paper_2102_06725_b200.functions as F
    nn.set_default_context(nn.ExecutionContext(type_config=nn.TypeConfig.HALF))
    B = 256
    x = nn.Variable((B, 64, 112, 112), need_grad=True)
    x.data.write_f32_device(nn.RngState(1).next_uniform_device((B, 64, 112, 112), -1, 1))
    y = F.max_pooling(x, (3, 3), (2, 2), pad=(1, 1))
    xi = nn.Variable((B, 3, 224, 224), need_grad=False)
    xi.data.write_f32_device(nn.RngState(2).next_uniform_device((B, 3, 224, 224), 0, 1))
    w = nn.Variable((64, 3, 7, 7), need_grad=True)
    w.d = np.random.default_rng(0).uniform(-0.1, 0.1, (64, 3, 7, 7)).astype(np.float32)
    b = nn.Variable((64,), need_grad=True)
    b.d = np.zeros(64, np.float32)
    c = F.convolution(xi, w, b, stride=(2, 2), pad=(3, 3))
    for name, fn in (("pool fwd", lambda: y.forward()), ("pool bwd", lambda: y.backward(1.0)),
                     ("stem fwd", lambda: c.forward()), ("stem bwd", lambda: c.backward(1.0))):
        fn()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(args.iters):
            fn()
        e.record()
        torch.cuda.synchronize()
        print(f"{name}: {s.elapsed_time(e) / args.iters:.3f} ms")


if __name__ == "__main__":
    main()
