"""Whole-step parity of the benchmark configurations against the oracle.

C4 (the headline): ResNet-50 v1.5 at 224x224, fp16 storage, dynamic loss
scaling (8, x2, 2000), momentum 0.9, weight decay 1e-4, lr 0.1 -- exactly the
bench.py step -- through DataParallelTrainer, against the oracle
(oracle/nnl_oracle.py Trainer: the reference's communicator.py:206-244 step +
solver.py:132-155 + the Momentum extension) on the same bytes.  C3:
ResNet-18 CIFAR at its batch of 128, same schedule.

Checked against the oracle after the first (eager) step: the loss (1e-2
relative, north_star), every parameter's gradient normwise, the updated
weights and f32 masters (1e-2 normwise), velocities, BN running statistics,
and the loss scale / counter / overflow decision exactly.  Then the CUDA
graph path (capture + replay, the bench path) must equal the eager path bit
for bit over three steps: at lr 0.1 on 8 images the trajectory is chaotic --
the oracle on the same batches in reversed order differs from itself by 4.9 %
in the step-1 loss (tools/noise_steps.py, profiles/noise_steps_*.json) -- so
later steps are compared engine-to-engine, not against the oracle.

Gradient tolerance.  Under fp16 storage with loss scale 8 many gradients sit
in or near the binary16 subnormal range, so the reference contract itself is
noisy: the oracle run on the SAME batch in reversed order (identical math, a
different but equally valid summation order) differs from the unreversed
oracle by up to 0.52 normwise at ResNet-50 batch 8 and 0.13 at ResNet-18
batch 128 (tools/noise_floor.py, profiles/noise_floor_*.json).  Each
parameter's gradient must therefore match within 3x its own measured noise
floor plus a small base -- computed in the test from that reversed-batch
oracle run, not assumed.
"""

import numpy as np
import pytest

from oracle import nnl_oracle as O

pytestmark = pytest.mark.gpu


def _nrm(a):
    return float(np.linalg.norm(np.asarray(a, np.float64)))


def _parity(nnl, net, B, half):
    import paper_2102_06725_b200.functions as F
    from paper_2102_06725_b200 import networks
    from paper_2102_06725_b200.communicator import DataParallelTrainer
    if net == "resnet50":
        hw, ncls, gbuild, obuild = 224, 1000, networks.resnet50, O.resnet50
    else:
        hw, ncls = 32, 10
        gbuild = lambda x, n: networks.resnet18_cifar(x, n)  # noqa: E731
        obuild = O.resnet18_cifar
    tc = nnl.TypeConfig.HALF if half else nnl.TypeConfig.FLOAT
    nnl.set_default_context(nnl.ExecutionContext(type_config=tc))
    shape = (B, 3, hw, hw)
    x0 = O.uniform(1, 0, shape, 0.0, 1.0)
    x1 = O.uniform(1, int(np.prod(shape)), shape, 0.0, 1.0)
    lab = (np.arange(B) % ncls).astype(np.float32)
    lab1 = ((np.arange(B) * 7 + 3) % ncls).astype(np.float32)

    def build(bs):
        xv = nnl.Variable((bs, 3, hw, hw))
        tv = nnl.Variable((bs,))
        return {"x": xv, "label": tv, "loss": F.softmax_cross_entropy(gbuild(xv, ncls), tv)}

    def trainer():
        return DataParallelTrainer(1, B, build, lr=0.1, seed=0, momentum=0.9, weight_decay=1e-4,
                                   loss_scaling=nnl.DynamicLossScaler(8.0, 2.0, 2000))

    def state(tr):
        rep = tr.rank0
        params = rep.registry.get_parameters()
        return dict(g={k: v.g for k, v in params.items()},
                    w={k: v.d for k, v in rep.registry.get_parameters(grad_only=False).items()},
                    m={k: rep.solver.master_values(k) for k in params},
                    v={k: rep.solver.velocity_values(k) for k in params},
                    sc=rep.dscaler.snapshot(), applied=rep.dscaler.last_applied(),
                    params=list(params))

    # eager trainer: x0, x0, x1; graph trainer: x0 eager, capture (its warm-up
    # is the x0 step), x1 replayed -- the bench path
    ea = trainer()
    got_loss = ea.step(x0, lab)
    s0 = state(ea)
    eager_losses = [got_loss, ea.step(x0, lab), ea.step(x1, lab1)]
    s_eager = state(ea)
    gr = trainer()
    graph_losses = [gr.step(x0, lab)]
    gr.capture_graph()
    graph_losses.append(float(gr.rank0.handles["loss"].d))
    graph_losses.append(gr.step(x1, lab1))
    s_graph = state(gr)

    otr = O.Trainer(lambda m, a, t: m.sce(obuild(m, a, ncls), t), 1, B, 0.1, seed=0, half=half,
                    scaler=O.Scaler(8.0, 2.0, 2000), momentum=0.9, weight_decay=1e-4)
    want_loss = otr.step(x0, lab)
    om = otr.models[0]
    # the oracle's own summation-order noise at step 0: the same batch reversed
    mr = O.Model(0, half)
    perm = np.arange(B)[::-1].copy()
    lo = mr.sce(obuild(mr, O.Var(x0[perm], half=half), ncls), O.Var(lab[perm], half=half))
    O.backward(lo, 8.0)
    want_g0 = {k: v.grad for k, v in om.trainable().items()}
    noise = {k: _nrm(v.grad / 8.0 - want_g0[k]) for k, v in mr.trainable().items()}
    return dict(got_loss=got_loss, want_loss=want_loss, s0=s0, om=om, opt=otr.opts[0],
                want_sc=otr.scalers[0], want_g0=want_g0, noise=noise, eager_losses=eager_losses,
                graph_losses=graph_losses, s_eager=s_eager, s_graph=s_graph)


def _check(r, half, base):
    s0 = r["s0"]
    assert s0["applied"]                                       # overflow decision: exact
    assert s0["sc"].loss_scale == r["want_sc"].loss_scale      # loss scale: exact
    assert s0["sc"].counter == r["want_sc"].counter
    assert abs(r["got_loss"] - r["want_loss"]) <= 1e-2 * abs(r["want_loss"])
    want_g0, noise = r["want_g0"], r["noise"]
    big = max(_nrm(v) for v in want_g0.values())
    floor = (1e-2 if half else 1e-3) * big
    worst = []
    for k in s0["params"]:
        den = max(_nrm(want_g0[k]), floor)
        tol = 3.0 * noise[k] / den + base  # (noise: one reordering draw)
        e0 = _nrm(s0["g"][k] - want_g0[k]) / den
        worst.append((round(e0, 5), round(tol, 5), k))
        assert e0 <= tol, (k, e0, tol)
        # velocity after one step = lr * (g + wd * w0): the gradient tolerance
        v_want = r["opt"].vel[k]
        ev = _nrm(s0["v"][k] - v_want) / max(_nrm(v_want), 0.1 * floor)
        assert ev <= tol, (k, ev, tol)
        # weights and masters after one step: w1 = w0 - lr * (g + wd * w0), so
        # they differ by exactly lr * (the gradient difference) plus storage
        # rounding.  (BN makes the preceding conv's loss scale-invariant, so
        # its gradient ~ 1/|w| is large and lr * g dominates w1: the stem's
        # weights move from ~0.1 to ~2 in this step.)
        for got, want in ((s0["w"][k], r["om"].params[k].value), (s0["m"][k], r["opt"].master[k])):
            lim = 0.1 * tol * den + 1e-3 * _nrm(want) + 1e-6
            assert _nrm(got - want) <= lim, (k, _nrm(got - want), lim)
    for k, v in r["om"].params.items():                        # BN running statistics
        if k.endswith("/mean") or k.endswith("/var"):
            assert _nrm(s0["w"][k] - v.value) <= 1e-2 * _nrm(v.value) + 1e-6, k
    # the CUDA-graph replay (the benchmark path) is the eager step, bit for bit,
    # across three steps (a trajectory that the oracle itself reproduces only to
    # a few percent at lr 0.1: reordering the batch moves its step-1 loss by 4.9 %,
    # profiles/noise_steps_resnet50_b8_f32.json)
    assert r["graph_losses"] == r["eager_losses"]
    for key in ("w", "m", "v", "g"):
        for k, v in r["s_eager"][key].items():
            assert np.array_equal(v, r["s_graph"][key][k]), (key, k)
    assert r["s_graph"]["sc"] == r["s_eager"]["sc"]
    return sorted(worst, reverse=True)[:3]


@pytest.mark.parametrize("half", [True, False])
def test_resnet50_c4_step_parity(nnl, half):
    """Batch 8 (the oracle takes several seconds per image-step on the host);
    fp16 storage is the headline configuration, fp32 pins the same graph
    where the summation noise is small."""
    r = _parity(nnl, "resnet50", 8, half)
    print("resnet50 worst normwise (err, tol, param):", _check(r, half, 0.05 if half else 2e-3))


def test_resnet18_c3_step_parity(nnl):
    """C3 at its own batch of 128 (fp16 storage, dynamic loss scaling)."""
    r = _parity(nnl, "resnet18", 128, True)
    print("resnet18 worst normwise (err, tol, param):", _check(r, True, 0.05))
