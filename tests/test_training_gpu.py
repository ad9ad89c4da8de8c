"""End-to-end parity: whole training steps on the GPU against the reference's
golden trajectories and the oracle (same seeds, same inputs)."""

import numpy as np
import pytest

from oracle import nnl_oracle as O

pytestmark = pytest.mark.gpu


def close(a, b, rtol, atol):
    np.testing.assert_allclose(np.asarray(a, np.float64), np.asarray(b, np.float64), rtol=rtol,
                               atol=atol, equal_nan=True)


def _ctx(nn, half):
    tc = nn.TypeConfig.HALF if half else nn.TypeConfig.FLOAT
    nn.set_default_context(nn.ExecutionContext(type_config=tc))


@pytest.mark.parametrize("half", [False, True])
@pytest.mark.parametrize("clear", [False, True])
def test_lenet_steps_match_reference(nnl, golden, half, clear):
    import paper_2102_06725_b200.functions as F
    from paper_2102_06725_b200 import networks
    g = golden("lenet")
    tag = "h" if half else "f"
    _ctx(nnl, half)
    with nnl.registry_scope(nnl.ParameterRegistry(0)) as reg:
        xv = nnl.Variable((16, 1, 28, 28))
        tv = nnl.Variable((16,))
        loss = F.softmax_cross_entropy(networks.lenet(xv, 10), tv)
        params = reg.get_parameters()
        for k, v in params.items():  # R12: bit-identical initial weights
            assert np.array_equal(v.d, g[f"lenet_{tag}_init__{k}"]), k
        solver = nnl.SgdSolver(0.05).setup(params)
        sc = nnl.DynamicLossScaler(8.0, 2.0, 2000)
        losses = []
        for s in range(3):
            xv.d = g["lenet_x"][s]
            tv.d = g["lenet_labels"]
            loss.forward(clear_buffer=clear)
            loss.backward(grad_seed=sc.loss_scale if half else 1.0, clear_buffer=clear)
            if s == 0:
                tol = dict(rtol=2e-2, atol=2e-2) if half else dict(rtol=1e-4, atol=1e-5)
                for k, v in params.items():
                    close(v.g, g[f"lenet_{tag}_grad0__{k}"], **tol)
            if half:
                assert nnl.dynamic_step(sc, solver).applied
            else:
                solver.update()
            losses.append(float(loss.d))
    tol = dict(rtol=2e-3, atol=2e-3) if half else dict(rtol=1e-5, atol=1e-6)
    close(losses, g[f"lenet_{tag}_losses"], **tol)
    for k, v in params.items():
        close(v.d, g[f"lenet_{tag}_final__{k}"], rtol=1e-2 if half else 1e-5,
              atol=2e-3 if half else 1e-6)


def test_mlp_fp32_matches_reference(nnl, golden):
    import paper_2102_06725_b200.functions as F
    from paper_2102_06725_b200 import networks
    g = golden("mlp")
    _ctx(nnl, False)
    with nnl.registry_scope(nnl.ParameterRegistry(0)) as reg:
        xv = nnl.Variable((64, 784))
        tv = nnl.Variable((64,))
        loss = F.softmax_cross_entropy(networks.mlp(xv, 10, hidden=(256,)), tv)
        solver = nnl.SgdSolver(0.1).setup(reg.get_parameters())
        losses = []
        for s in range(2):
            xv.d = g["mlp_x"][s]
            tv.d = g["mlp_labels"]
            loss.forward()
            loss.backward()
            solver.update()
            losses.append(float(loss.d))
        close(losses, g["mlp_losses"], rtol=1e-5, atol=1e-6)
        for k, v in reg.get_parameters().items():
            close(v.d, g[f"mlp_final__{k}"], rtol=1e-5, atol=1e-6)


def test_dynamic_scaler_sequence_matches_reference(nnl, golden):
    g = golden("solver")
    _ctx(nnl, True)
    w = nnl.Variable((4,), need_grad=True)
    w.d = np.array([1.0, -2.0, 0.5, 3.0], np.float32)
    s = nnl.SgdSolver(0.1).setup({"w": w})
    sc = nnl.DynamicLossScaler(8.0, 2.0, 2)
    for i, gr in enumerate(g["seq_grads"]):
        w.g = gr * np.float32(sc.loss_scale)
        out = nnl.dynamic_step(sc, s)
        assert out.applied == bool(g["seq_applied"][i])          # integer decision: exact
        assert sc.loss_scale == g["seq_scales"][i]
        assert np.array_equal(w.d, g["seq_w"][i])                # bitwise


def test_device_scaler_matches_host_scaler(nnl, golden):
    """The sync-free device state machine reproduces dynamic_step exactly."""
    g = golden("solver")
    _ctx(nnl, True)
    w = nnl.Variable((4,), need_grad=True)
    w.d = np.array([1.0, -2.0, 0.5, 3.0], np.float32)
    s = nnl.SgdSolver(0.1).setup({"w": w})
    dsc = nnl.DeviceLossScaler(nnl.DynamicLossScaler(8.0, 2.0, 2))
    for i, gr in enumerate(g["seq_grads"]):
        w.g = gr * np.float32(dsc.snapshot().loss_scale)
        s.dynamic_update(dsc, check=True)
        assert dsc.last_applied() == bool(g["seq_applied"][i])
        assert dsc.snapshot().loss_scale == g["seq_scales"][i]
        assert np.array_equal(w.d, g["seq_w"][i])


def test_half_master_accumulates(nnl, golden):
    g = golden("solver")
    _ctx(nnl, True)
    w = nnl.Variable((1,), need_grad=True)
    w.d = np.array([1.0], np.float32)
    s = nnl.SgdSolver(2.0 ** -16).setup({"w": w})
    vis = []
    for _ in range(3):
        w.g = np.array([1.0], np.float32)
        s.update()
        vis.append(float(w.d[0]))
    assert vis == list(g["master_w"])
    assert np.array_equal(s.master_values("w"), g["master_m"])


@pytest.mark.parametrize("half", [False, True])
def test_dp2_inprocess_matches_reference(nnl, golden, half):
    import paper_2102_06725_b200.functions as F
    from paper_2102_06725_b200 import networks
    from paper_2102_06725_b200.communicator import DataParallelTrainer
    g = golden("lenet")
    tag = "h" if half else "f"
    _ctx(nnl, half)

    def build(bs):
        xv = nnl.Variable((bs, 1, 28, 28))
        tv = nnl.Variable((bs,))
        return {"x": xv, "label": tv,
                "loss": F.softmax_cross_entropy(networks.lenet(xv, 10), tv)}

    tr = DataParallelTrainer(2, 16, build, lr=0.05, seed=0,
                             loss_scaling=nnl.DynamicLossScaler(8.0, 2.0, 2000) if half else None)
    losses = [tr.step(g["lenet_x"][i], g["lenet_labels"]) for i in range(2)]
    tol = dict(rtol=2e-3, atol=2e-3) if half else dict(rtol=1e-5, atol=1e-6)
    close(losses, g[f"dp2_{tag}_losses"], **tol)
    for k, v in tr.rank0.registry.get_parameters().items():
        close(v.d, g[f"dp2_{tag}_final__{k}"], rtol=1e-2 if half else 1e-5,
              atol=2e-3 if half else 1e-6)


def test_static_equals_dynamic_bitwise(nnl):
    """Reference property (tests/test_graph.py:238-260)."""
    import paper_2102_06725_b200.functions as F
    from paper_2102_06725_b200 import networks
    x = O.uniform(3, 0, (8, 1, 28, 28), 0, 1)
    lab = (np.arange(8) % 10).astype(np.float32)
    outs = []
    for mode in (nnl.Mode.STATIC, nnl.Mode.DYNAMIC):
        nnl.set_default_context(nnl.ExecutionContext(mode=mode, type_config=nnl.TypeConfig.HALF))
        with nnl.registry_scope(nnl.ParameterRegistry(0)) as reg:
            xv = nnl.Variable(x.shape)
            tv = nnl.Variable(lab.shape)
            xv.d = x
            tv.d = lab
            loss = F.softmax_cross_entropy(networks.lenet(xv, 10), tv)
            loss.forward()
            loss.backward(8.0)
            outs.append((loss.d.copy(), reg.get_parameters()["conv1/W"].g.copy()))
    assert np.array_equal(outs[0][0], outs[1][0])
    assert np.array_equal(outs[0][1], outs[1][1])


def _resnet_oracle_step(builder, x, lab, half, lr, n_classes):
    tr = O.Trainer(lambda m, a, t: m.sce(builder(m, a, n_classes), t), 1, x.shape[0], lr,
                   seed=0, half=half, scaler=O.Scaler(8.0, 2.0, 2000) if half else None)
    loss = tr.step(x, lab)
    return loss, tr


def test_step_async_matches_step(nnl, golden):
    """The pipelined `step_async` (copy-stream H2D, async loss read-back) is the
    same step as `step`: identical losses and weights, with and without a
    captured graph."""
    import paper_2102_06725_b200.functions as F
    from paper_2102_06725_b200 import networks
    from paper_2102_06725_b200.communicator import DataParallelTrainer
    g = golden("lenet")
    _ctx(nnl, True)

    def build(bs):
        xv = nnl.Variable((bs, 1, 28, 28))
        tv = nnl.Variable((bs,))
        return {"x": xv, "label": tv,
                "loss": F.softmax_cross_entropy(networks.lenet(xv, 10), tv)}

    def trainer():
        return DataParallelTrainer(1, 16, build, lr=0.05, seed=0,
                                   loss_scaling=nnl.DynamicLossScaler(8.0, 2.0, 2000))

    runs = []
    for graph in (False, True):
        for mode in ("sync", "async"):
            tr = trainer()
            losses = [tr.step(g["lenet_x"][0], g["lenet_labels"])]
            if graph:  # (the capture runs one extra step on resident inputs, in both modes)
                tr.capture_graph()
            if mode == "sync":
                losses += [tr.step(g["lenet_x"][i], g["lenet_labels"]) for i in (1, 2)]
            else:
                pend = [tr.step_async(g["lenet_x"][i], g["lenet_labels"]) for i in (1, 2)]
                losses += [p.result() for p in pend]
            runs.append((graph, losses, {k: v.d.copy() for k, v in
                                         tr.rank0.registry.get_parameters().items()}))
    for i in (1, 3):
        assert runs[i][0] == runs[i - 1][0]
        assert runs[i][1] == runs[i - 1][1]
        for k, v in runs[i][2].items():
            assert np.array_equal(v, runs[i - 1][2][k]), k


@pytest.mark.parametrize("half", [False, True])
def test_resnet18_eval_graph_vs_oracle(nnl, half):
    """Eval graph (BN on running statistics, after one training step updated
    them) and evaluate_classifier against the oracle's eval forward."""
    import paper_2102_06725_b200.functions as F
    from paper_2102_06725_b200 import networks
    from paper_2102_06725_b200.evaluate import evaluate_classifier
    _ctx(nnl, half)
    B = 4
    x = O.uniform(1, 0, (B, 3, 32, 32), 0, 1)
    lab = (np.arange(B) % 10).astype(np.float32)
    xe = O.uniform(2, 0, (6, 3, 32, 32), 0, 1)   # 6 rows: a wrapped tail chunk
    le = (np.arange(6) % 10).astype(np.float32)
    with nnl.registry_scope(nnl.ParameterRegistry(0)) as reg:
        xv, tv = nnl.Variable(x.shape), nnl.Variable(lab.shape)
        loss = F.softmax_cross_entropy(networks.resnet18_cifar(xv, 10), tv)
        solver = nnl.SgdSolver(0.1).setup(reg.get_parameters())
        xv.d, tv.d = x, lab
        loss.forward(clear_buffer=True)
        loss.backward(grad_seed=8.0 if half else 1.0, clear_buffer=True)
        if half:
            assert nnl.dynamic_step(nnl.DynamicLossScaler(8.0, 2.0, 2000), solver).applied
        else:
            solver.update()
        xe_v = nnl.Variable((B, 3, 32, 32))
        logits = networks.resnet18_cifar(xe_v, 10, train=False)
        err, mloss = evaluate_classifier(xe_v, logits, xe, le)
        xe_v.d = xe[:B]
        logits.forward()
        got = logits.d
    _, tr = _resnet_oracle_step(O.resnet18_cifar, x, lab, half, 0.1, 10)
    m = tr.models[0]
    m.batch_stat = False
    oz = O.resnet18_cifar(m, O.Var(xe[:B], half=half), 10)
    tol = 5e-2 if half else 1e-3
    assert np.abs(got - oz.value).max() <= tol * max(1.0, np.abs(oz.value).max())
    # the reference's own expressions on the oracle's logits for all 6 rows
    rows = []
    for start in range(0, 6, B):
        idx = np.arange(start, start + B) % 6
        rows.append(O.resnet18_cifar(m, O.Var(xe[idx], half=half), 10).value[:min(B, 6 - start)])
    lg = np.concatenate(rows)
    want_err = float((np.argmax(lg, axis=1) != le.astype(np.int64)).mean())
    z = lg - lg.max(axis=1, keepdims=True)
    want_loss = float(-(z - np.log(np.exp(z).sum(axis=1, keepdims=True)))[
        np.arange(6), le.astype(np.int64)].sum()) / 6
    assert abs(mloss - want_loss) <= tol * max(1.0, abs(want_loss))
    assert abs(err - want_err) <= 1.0 / 6 + 1e-9  # at most one near-tie row may flip


@pytest.mark.parametrize("net", ["bottleneck", "basic"])
def test_bn_backward_stats_in_dgrad_epilogue(nnl, net):
    """BN-backward statistics fused into the dgrad epilogue of the following
    convolution (fused BN->ReLU->conv, and the residual tail's last gradient
    contributor writing the gated gradient straight into the shortcut's
    gradient) against the same engine with that fusion off: the same step up
    to the f32 summation order of the statistics.  (The kernel itself is
    checked bit for bit in test_dgrad_bn_stats_epilogue.)"""
    import paper_2102_06725_b200.functions as F
    from paper_2102_06725_b200 import graph, networks
    _ctx(nnl, True)
    prev_flag = graph.BNB_FUSION
    B, hw = 8, 16
    x = O.uniform(3, 0, (B, 64, hw, hw), 0, 1)
    lab = (np.arange(B) % 10).astype(np.float32)
    block = networks._bottleneck if net == "bottleneck" else networks._basic
    runs, fused = [], []
    try:
        for bnb in (True, False):
            graph.BNB_FUSION = bnb
            with nnl.registry_scope(nnl.ParameterRegistry(0)) as reg:
                xv = nnl.Variable(x.shape, need_grad=True)
                tv = nnl.Variable(lab.shape)
                h = xv
                blocks = [(64, 1, True), (64, 1, False), (64, 2, True), (64, 1, False)]
                for i, (w, s, proj) in enumerate(blocks):
                    with nnl.parameter_scope(f"b{i}"):
                        h = block(h, w, s, proj)
                h = F.global_average_pooling(h)
                loss = F.softmax_cross_entropy(nnl.parametric.affine(h, 10, name="fc"), tv)
                xv.d = x
                tv.d = lab
                loss.forward(clear_buffer=True)
                loss.backward(grad_seed=8.0, clear_buffer=True)
                grads = {k: v.g for k, v in reg.get_parameters().items()}
                grads["x"] = xv.g
                fused.append(sum(1 for n in _nodes(loss) if n.kind == "BatchNormalization"
                                 and "bwd_parts" in n.state))
                runs.append((float(loss.d), grads))
    finally:
        graph.BNB_FUSION = prev_flag
    # bottleneck: 3 stride-1 conv2 dgrads (BN1), 4 conv3 dgrads (BN2), 3 tails;
    # basic: 4 conv2 dgrads (BN1), 2 tails (stride-1 conv1 of the next block)
    assert fused == [10 if net == "bottleneck" else 6, 0]
    assert runs[0][0] == runs[1][0]
    # conv biases feeding a train-mode BN have a mathematically zero gradient
    # (rounding noise on both sides): floor relative to the largest norm
    norms = [np.linalg.norm(v) for v in runs[1][1].values()]
    for k, a in runs[0][1].items():
        b = runs[1][1][k]
        den = max(np.linalg.norm(b), 1e-2 * max(norms))
        assert np.linalg.norm(a - b) / den < 2e-2, k


def _nodes(loss):
    from paper_2102_06725_b200.graph import _ancestors
    return _ancestors(loss)
