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


def _stem_run(nnl, fuse_pool, monkeypatch):
    import paper_2102_06725_b200.functions as F
    import paper_2102_06725_b200.parametric as PF
    monkeypatch.setenv("NNL_FUSE_POOL", "1" if fuse_pool else "0")
    nnl.set_default_context(nnl.ExecutionContext(type_config=nnl.TypeConfig.HALF))
    x = O.uniform(3, 0, (4, 3, 64, 64), -1, 1)
    lab = (np.arange(4) % 10).astype(np.float32)
    with nnl.registry_scope(nnl.ParameterRegistry(0)) as reg:
        xv = nnl.Variable(x.shape)
        tv = nnl.Variable(lab.shape)
        h = PF.convolution(xv, 64, (7, 7), stride=(2, 2), pad=(3, 3), name="conv1")
        z = F.relu(PF.batch_normalization(h, name="bn1"))
        pool = F.max_pooling(z, (3, 3), (2, 2), pad=(1, 1))
        h = PF.convolution(pool, 64, (3, 3), pad=(1, 1), name="conv2")
        h = F.relu(PF.batch_normalization(h, name="bn2"))
        h = F.global_average_pooling(h)
        loss = F.softmax_cross_entropy(PF.affine(h, 10, name="fc"), tv)
        xv.d, tv.d = x, lab
        loss.forward(clear_buffer=True)
        pd = pool.d.copy()
        loss.backward(grad_seed=8.0, clear_buffer=True)
        out = float(loss.d), pd, {k: v.g.copy() for k, v in reg.get_parameters().items()}
    nnl.set_default_context(nnl.ExecutionContext())
    return out


def test_bn_relu_maxpool_fusion_is_bit_identical(nnl, monkeypatch):
    """The stem's BN -> ReLU -> MaxPooling as one pass (opt-in NNL_FUSE_POOL=1;
    relu(BN(x)) never written, the pool's argmax from the fused kernel): loss,
    pooled activations and every parameter gradient bit-identical to the
    BN->ReLU pass + pool."""
    import paper_2102_06725_b200.functions as F
    calls = []
    orig = F.BatchNormalization.forward_fused_pool
    monkeypatch.setattr(F.BatchNormalization, "forward_fused_pool",
                        lambda self, *a: (calls.append(1), orig(self, *a))[1])
    l1, p1, g1 = _stem_run(nnl, True, monkeypatch)
    assert calls == [1]  # the stem's BN -> ReLU -> pool took the fused pass
    l0, p0, g0 = _stem_run(nnl, False, monkeypatch)
    assert l1 == l0
    assert np.array_equal(p1.view(np.uint32), p0.view(np.uint32))
    for k in g0:
        assert np.array_equal(g1[k].view(np.uint32), g0[k].view(np.uint32)), k
