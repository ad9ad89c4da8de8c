"""Summation-order noise floor of the oracle (test-tolerance calibration).

    python tools/noise_floor.py resnet50 8 [half|float]

Runs one oracle training step (forward + backward with the dynamic-scaler
seed) on a batch and on the same batch in reversed order -- identical math,
a different but equally valid summation order wherever a reduction crosses
the batch -- and prints the normwise per-parameter gradient differences
(the metric tests/test_resnet_parity_gpu.py checks), the loss difference and
the BN running-statistics differences.  Writes profiles/noise_floor_<net>_b<B>_<dtype>.json.
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import nnl_oracle as O  # noqa: E402

net = sys.argv[1] if len(sys.argv) > 1 else "resnet50"
B = int(sys.argv[2]) if len(sys.argv) > 2 else 8
half = (sys.argv[3] if len(sys.argv) > 3 else "half") == "half"
if net == "resnet50":
    builder, hw, ncls = O.resnet50, 224, 1000
else:
    builder, hw, ncls = O.resnet18_cifar, 32, 10
x = O.uniform(1, 0, (B, 3, hw, hw), 0, 1)
lab = (np.arange(B) % ncls).astype(np.float32)


def run(perm):
    m = O.Model(0, half)
    lo = m.sce(builder(m, O.Var(x[perm], half=half), ncls), O.Var(lab[perm], half=half))
    O.backward(lo, 8.0 if half else 1.0)
    return float(lo.value), m


t0 = time.time()
l1, m1 = run(np.arange(B))
l2, m2 = run(np.arange(B)[::-1].copy())
p1, p2 = m1.trainable(), m2.trainable()
nrm = {k: float(np.linalg.norm(v.grad)) for k, v in p1.items()}
floor = (1e-2 if half else 1e-3) * max(nrm.values())
errs = {k: float(np.linalg.norm(p2[k].grad - v.grad) / max(nrm[k], floor)) for k, v in p1.items()}
worst = sorted(errs.items(), key=lambda kv: -kv[1])[:10]
stats = {}
for k, v in m1.params.items():
    if k.endswith("/mean") or k.endswith("/var"):
        d = np.abs(m2.params[k].value - v.value).max() / (np.abs(v.value).max() + 1e-30)
        stats[k] = float(d)
out = {"net": net, "batch": B, "half": half, "loss": l1, "loss_reordered": l2,
       "loss_rel_diff": abs(l1 - l2) / abs(l1), "grad_normwise_worst": worst,
       "grad_normwise_median": float(np.median(list(errs.values()))),
       "running_stat_worst": max(stats.values()) if stats else None,
       "floor_rule": "denominator max(||g||, (1e-2 fp16 | 1e-3 fp32) * max_k ||g_k||)",
       "seconds": round(time.time() - t0, 1)}
print(json.dumps(out, indent=1))
path = os.path.join(ROOT, "profiles", f"noise_floor_{net}_b{B}_{'f16' if half else 'f32'}.json")
with open(path, "w") as f:
    json.dump(out, f, indent=1)
