#!/usr/bin/env python
"""One ResNet-50 stage-1 identity bottleneck (256->64->64->256 at 56x56,
batch 256) between two others, forward + backward with the engine's fusions
(clear_buffer=True): per-node device times; run under ncu for the fused
BN-backward dgrad epilogues.   python tools/bnb_probe.py [--iters 3]"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=3)
    ap.add_argument("--batch", type=int, default=256)
    args = ap.parse_args()
    import numpy as np
    import torch
    import paper_2102_06725_b200 as nn
    import paper_2102_06725_b200.functions as F
    from paper_2102_06725_b200 import networks
    from paper_2102_06725_b200.profiler import PROFILER
    nn.set_default_context(nn.ExecutionContext(type_config=nn.TypeConfig.HALF))
    B = args.batch
    with nn.registry_scope(nn.ParameterRegistry(0)):
        xv = nn.Variable((B, 256, 56, 56), need_grad=True)
        xv.data.write_f32_device(nn.RngState(1).next_uniform_device((B, 256, 56, 56), 0, 1))
        h = xv
        for i in range(3):
            with nn.parameter_scope(f"b{i}"):
                h = networks._bottleneck(h, 64, 1, False)
        h = F.global_average_pooling(h)
        tv = nn.Variable((B,))
        tv.d = (np.arange(B) % 10).astype(np.float32)
        loss = F.softmax_cross_entropy(nn.parametric.affine(h, 10, name="fc"), tv)
        for it in range(args.iters):
            PROFILER.reset()
            PROFILER.enabled = it == args.iters - 1
            loss.forward(clear_buffer=True)
            loss.backward(grad_seed=8.0, clear_buffer=True)
        torch.cuda.synchronize()
        PROFILER.enabled = False
        for r in PROFILER.per_node():
            print(f"{r['kind']:20s} {r['phase']:4s} {r['shape']:40s} {r['ms']:8.3f}")


if __name__ == "__main__":
    main()
