"""Trajectory noise of the oracle: the 3-step schedule of
tests/test_resnet_parity_gpu.py (x0, x0, x1 with lr 0.1, momentum 0.9, wd
1e-4, dynamic loss scaling) on a batch and on the same batches in reversed
order.  Prints per-step losses of both, and the normwise weight / velocity /
running-stat differences after the last step.

    python tools/noise_steps.py resnet50 8 half|float
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import nnl_oracle as O  # noqa: E402

net, B, half = sys.argv[1], int(sys.argv[2]), sys.argv[3] == "half"
hw, ncls, builder = (224, 1000, O.resnet50) if net == "resnet50" else (32, 10, O.resnet18_cifar)
shape = (B, 3, hw, hw)
x0 = O.uniform(1, 0, shape, 0.0, 1.0)
x1 = O.uniform(1, int(np.prod(shape)), shape, 0.0, 1.0)
lab = (np.arange(B) % ncls).astype(np.float32)
lab1 = ((np.arange(B) * 7 + 3) % ncls).astype(np.float32)


def run(perm):
    tr = O.Trainer(lambda m, a, t: m.sce(builder(m, a, ncls), t), 1, B, 0.1, seed=0, half=half,
                   scaler=O.Scaler(8.0, 2.0, 2000), momentum=0.9, weight_decay=1e-4)
    losses = [tr.step(x[perm], l[perm]) for x, l in ((x0, lab), (x0, lab), (x1, lab1))]
    return losses, tr


p = np.arange(B)
la, ta = run(p)
lb, tb = run(p[::-1].copy())
ma, mb = ta.models[0], tb.models[0]
dw = {k: float(np.linalg.norm(mb.params[k].value - v.value) / (np.linalg.norm(v.value) + 1e-30))
      for k, v in ma.params.items()}
dv = {k: float(np.linalg.norm(tb.opts[0].vel[k] - v) / (np.linalg.norm(v) + 1e-30))
      for k, v in ta.opts[0].vel.items()}
out = {"net": net, "batch": B, "half": half, "losses": la, "losses_reordered": lb,
       "loss_rel_diff": [abs(a - b) / abs(a) for a, b in zip(la, lb)],
       "weight_rel_worst": sorted(dw.items(), key=lambda kv: -kv[1])[:5],
       "velocity_rel_worst": sorted(dv.items(), key=lambda kv: -kv[1])[:5]}
print(json.dumps(out, indent=1))
with open(os.path.join(ROOT, "profiles", f"noise_steps_{net}_b{B}_{'f16' if half else 'f32'}.json"),
          "w") as f:
    json.dump(out, f, indent=1)
