"""Engine contracts on the device: fusions chosen by forward bind backward,
operand dtypes are validated, params-only checkpoints restart the solver
state, and a replayed training graph still refuses out-of-range labels."""

import numpy as np
import pytest

from oracle import nnl_oracle as O

pytestmark = pytest.mark.gpu


def _resnet_grads(nnl, fwd_clear, bwd_clear, half=True):
    import paper_2102_06725_b200.functions as F
    from paper_2102_06725_b200 import networks
    tc = nnl.TypeConfig.HALF if half else nnl.TypeConfig.FLOAT
    nnl.set_default_context(nnl.ExecutionContext(type_config=tc))
    x = O.uniform(1, 0, (4, 3, 32, 32), 0, 1)
    lab = (np.arange(4) % 10).astype(np.float32)
    with nnl.registry_scope(nnl.ParameterRegistry(0)) as reg:
        xv = nnl.Variable(x.shape)
        tv = nnl.Variable(lab.shape)
        loss = F.softmax_cross_entropy(networks.resnet18_cifar(xv, 10), tv)
        xv.d, tv.d = x, lab
        loss.forward(clear_buffer=fwd_clear)
        loss.backward(grad_seed=8.0, clear_buffer=bwd_clear)
        return float(loss.d), {k: v.g for k, v in reg.get_parameters().items()}


@pytest.mark.parametrize("half", [False, True])
def test_fused_forward_then_plain_backward(nnl, half):
    """forward(clear_buffer=True) fuses BN->ReLU, Add2->ReLU and the residual
    tails, so the BN/Add2 outputs are never written.  A backward with the
    default clear_buffer=False must take the same fused backward:
    bitwise equal to backward(clear_buffer=True) after the same forward, and
    within summation-order noise of the fully unfused graph."""
    l_ff, g_ff = _resnet_grads(nnl, True, False, half)
    l_tt, g_tt = _resnet_grads(nnl, True, True, half)
    l_nn, g_nn = _resnet_grads(nnl, False, False, half)
    assert l_ff == l_tt
    for k in g_tt:
        assert np.array_equal(g_ff[k], g_tt[k], equal_nan=True), k
        assert np.isfinite(g_ff[k]).all(), k
    assert abs(l_ff - l_nn) <= (2e-3 if half else 1e-5) * max(1.0, abs(l_nn))
    big = max(np.linalg.norm(v) for v in g_nn.values())
    for k in g_nn:
        err = np.linalg.norm(g_ff[k] - g_nn[k]) / max(np.linalg.norm(g_nn[k]), 1e-2 * big)
        assert err < (0.3 if half else 2e-2), (k, err)


def test_operand_dtypes_are_validated(nnl):
    import paper_2102_06725_b200.functions as F
    from paper_2102_06725_b200.errors import DtypeMismatch, ShapeMismatch
    nnl.set_default_context(nnl.ExecutionContext(type_config=nnl.TypeConfig.HALF))
    x32 = nnl.Variable((2, 3, 8, 8), dtype=nnl.Dtype.F32)  # built outside the HALF scope
    w = nnl.Variable((4, 3, 3, 3), need_grad=True)
    b = nnl.Variable((4,), need_grad=True)
    with pytest.raises(DtypeMismatch):
        F.convolution(x32, w, b)
    x16 = nnl.Variable((2, 3, 8, 8))
    h = F.convolution(x16, w, b)  # fine: one storage type
    g16 = nnl.Variable((4,), need_grad=True)  # BN scale must be F32 (parametric.py:67-70)
    f32 = [nnl.Variable((4,), dtype=nnl.Dtype.F32) for _ in range(3)]
    with pytest.raises(ShapeMismatch):  # DtypeMismatch is-a ShapeMismatch
        F.batch_normalization(h, g16, *f32)
    F.batch_normalization(h, nnl.Variable((4,), dtype=nnl.Dtype.F32), *f32)
    lab32 = nnl.Variable((2,), dtype=nnl.Dtype.F32)
    with pytest.raises(DtypeMismatch):
        F.softmax_cross_entropy(nnl.Variable((2, 10)), lab32)


def _lenet_trainer(nnl, seed=0):
    import paper_2102_06725_b200.functions as F
    from paper_2102_06725_b200 import networks
    from paper_2102_06725_b200.communicator import DataParallelTrainer
    nnl.set_default_context(nnl.ExecutionContext(type_config=nnl.TypeConfig.HALF))

    def build(bs):
        xv = nnl.Variable((bs, 1, 28, 28))
        tv = nnl.Variable((bs,))
        return {"x": xv, "label": tv,
                "loss": F.softmax_cross_entropy(networks.lenet(xv, 10), tv)}

    return DataParallelTrainer(1, 16, build, lr=0.05, seed=seed, momentum=0.9,
                               weight_decay=1e-4, loss_scaling=nnl.DynamicLossScaler(8.0, 2.0, 4))


def test_params_only_checkpoint_restarts_solver_state(nnl, golden, tmp_path):
    """A file with parameters only (the reference's parameter.bin) loaded into a
    trained solver: masters restart from the loaded weights (R11) and the
    velocity from zero, exactly like a fresh trainer set up on those weights
    (the stale master used to overwrite the loaded weights)."""
    from paper_2102_06725_b200 import checkpoint as ck
    g = golden("lenet")
    src = _lenet_trainer(nnl, seed=0)
    src.step(g["lenet_x"][0], g["lenet_labels"])
    path = str(tmp_path / "params.bin")
    ck.save(path, src.rank0.registry.get_parameters(grad_only=False))  # no solver records

    a = _lenet_trainer(nnl, seed=5)
    for i in range(2):  # a's solver now holds masters/velocities of other weights
        a.step(g["lenet_x"][i], g["lenet_labels"])
    a.load_checkpoint(path)
    b = _lenet_trainer(nnl, seed=5)
    b.load_checkpoint(path)
    # a and b: same weights, masters re-derived, zero velocity; a's scaler
    # counter differs, so compare one step with a fresh b step
    for k, v in a.rank0.registry.get_parameters().items():
        assert np.array_equal(a.rank0.solver.master_values(k), v.d.astype(np.float32)), k
        assert not a.rank0.solver.velocity_values(k).any(), k
    la = a.step(g["lenet_x"][2], g["lenet_labels"])
    lb = b.step(g["lenet_x"][2], g["lenet_labels"])
    assert la == lb
    pa, pb = a.rank0.registry.get_parameters(), b.rank0.registry.get_parameters()
    for k in pa:
        assert np.array_equal(pa[k].d, pb[k].d), k


def test_graph_replay_refuses_bad_labels(nnl, golden):
    from paper_2102_06725_b200.errors import LabelOutOfRange
    g = golden("lenet")
    tr = _lenet_trainer(nnl)
    tr.step(g["lenet_x"][0], g["lenet_labels"])
    tr.capture_graph()
    bad = g["lenet_labels"].copy()
    bad[3] = 10
    with pytest.raises(LabelOutOfRange):
        tr.step(g["lenet_x"][0], bad)
    with pytest.raises(LabelOutOfRange):
        tr.step_async(g["lenet_x"][0], bad)
    tr.step(g["lenet_x"][0], g["lenet_labels"])  # valid labels replay again
