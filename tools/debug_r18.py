"""Locate the first node (in backward order) whose output gradient differs
between the GPU engine and the oracle, for a ResNet-18 step (debug aid)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2102_06725_b200 as nn
import paper_2102_06725_b200.functions as F
from paper_2102_06725_b200 import networks
from paper_2102_06725_b200.graph import _ancestors
from oracle import nnl_oracle as O

half = len(sys.argv) > 1 and sys.argv[1] == "half"
nn.set_default_context(nn.ExecutionContext(
    type_config=nn.TypeConfig.HALF if half else nn.TypeConfig.FLOAT))
B = 4
x = O.uniform(1, 0, (B, 3, 32, 32), 0, 1)
lab = (np.arange(B) % 10).astype(np.float32)
reg = nn.ParameterRegistry(0)
with nn.registry_scope(reg):
    xv = nn.Variable(x.shape)
    tv = nn.Variable(lab.shape)
    loss = F.softmax_cross_entropy(networks.resnet18_cifar(xv, 10), tv)
    xv.d = x
    tv.d = lab
    loss.forward()
    loss.backward(grad_seed=8.0 if half else 1.0)
m = O.Model(0, half)
lo = m.sce(O.resnet18_cifar(m, O.Var(x, half=half), 10), O.Var(lab, half=half))
O.backward(lo, 8.0 if half else 1.0)
gn = _ancestors(loss)
on = O.ancestors(lo)
print(len(gn), len(on))
rows = []
for a, b in zip(reversed(gn), reversed(on)):
    assert a.kind == b.kind, (a.kind, b.kind)
    for i, (va, vb) in enumerate(zip(a.inputs, b.inputs)):
        if not va.need_grad and va.parent is None:
            continue
        ga, gb = va.g, vb.grad
        ref = np.abs(gb).max()
        err = np.abs(ga - gb).max() / (ref + 1e-30)
        fa, fb = va.d, vb.value
        ferr = np.abs(fa - fb).max() / (np.abs(fb).max() + 1e-30)
        rows.append((a.kind, i, va.shape, err, ref, ferr))
for r in rows:
    if r[3] < 1e-4 or r[4] < 1e-6:
        continue
    print(f"{r[0]:22s} in{r[1]} {str(r[2]):22s} gerr {r[3]:.2e} (max {r[4]:.2e}) ferr {r[5]:.2e}")
# normwise per-parameter errors (what tests/test_training_gpu.py checks)
params = m.trainable()
gpu = {k: v.g for k, v in reg.get_parameters().items()}
nrm = {k: np.linalg.norm(v.grad) for k, v in params.items()}
floor = (1e-2 if half else 1e-3) * max(nrm.values())
errs = sorted(((np.linalg.norm(gpu[k] - v.grad) / max(nrm[k], floor), k)
               for k, v in params.items()), reverse=True)
print("normwise worst:", [(round(float(e), 5), k) for e, k in errs[:6]])
# noise floor: the same oracle on the batch in reversed order (identical math,
# different summation order everywhere a reduction crosses the batch)
m2 = O.Model(0, half)
perm = np.arange(B)[::-1].copy()
lo2 = m2.sce(O.resnet18_cifar(m2, O.Var(x[perm], half=half), 10), O.Var(lab[perm], half=half))
O.backward(lo2, 8.0 if half else 1.0)
p2 = m2.trainable()
errs2 = sorted(((np.linalg.norm(p2[k].grad - v.grad) / max(nrm[k], floor), k)
                for k, v in params.items()), reverse=True)
print("oracle-vs-reordered-oracle worst:", [(round(float(e), 5), k) for e, k in errs2[:6]])
