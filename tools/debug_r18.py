"""Per-parameter gradient error of one ResNet-18 step vs the oracle (debug aid)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2102_06725_b200 as nn
import paper_2102_06725_b200.functions as F
from paper_2102_06725_b200 import networks
from oracle import nnl_oracle as O

for half in (False, True):
    for clear in (False, True):
        nn.set_default_context(nn.ExecutionContext(
            type_config=nn.TypeConfig.HALF if half else nn.TypeConfig.FLOAT))
        B = 4
        x = O.uniform(1, 0, (B, 3, 32, 32), 0, 1)
        lab = (np.arange(B) % 10).astype(np.float32)
        with nn.registry_scope(nn.ParameterRegistry(0)) as reg:
            xv = nn.Variable(x.shape)
            tv = nn.Variable(lab.shape)
            loss = F.softmax_cross_entropy(networks.resnet18_cifar(xv, 10), tv)
            xv.d = x
            tv.d = lab
            loss.forward(clear_buffer=clear)
            loss.backward(grad_seed=8.0 if half else 1.0, clear_buffer=clear)
            grads = {k: v.g for k, v in reg.get_parameters().items()}
            got = float(loss.d)
        m = O.Model(0, half)
        xo = O.Var(x, half=half)
        to = O.Var(lab, half=half)
        lo = m.sce(O.resnet18_cifar(m, xo, 10), to)
        O.backward(lo, 8.0 if half else 1.0)
        gscale = max(np.abs(v.grad).max() for v in m.trainable().values())
        print(f"half={half} clear={clear} loss {got:.6f} vs {float(lo.value):.6f}")
        worst = []
        for k, v in m.trainable().items():
            d = np.abs(grads[k] - v.grad).max() / max(np.abs(v.grad).max(), 1e-3 * gscale)
            worst.append((d, k))
        for d, k in sorted(worst, reverse=True)[:8]:
            print(f"   {d:.4f} {k}")
