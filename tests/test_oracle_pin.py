"""Pin the oracle (oracle/nnl_oracle.py) before trusting it.

* against the golden vectors produced by the reference (tests/golden/);
* against the live reference where /root/reference exists (marked
  `reference`; skipped on the GPU box).
All CPU-only.
"""

import numpy as np
import pytest

from oracle import nnl_oracle as O


def close(a, b, rtol=1e-5, atol=1e-6):
    np.testing.assert_allclose(np.asarray(a, np.float64), np.asarray(b, np.float64), rtol=rtol,
                               atol=atol, equal_nan=True)


def test_quantize_matches_reference(golden):
    g = golden("numerics")
    q = O.q16(g["q_in"])
    assert np.array_equal(np.isnan(q), np.isnan(g["q_out"]))
    m = ~np.isnan(q)
    assert np.array_equal(q[m].view(np.uint32), g["q_out"][m].view(np.uint32))
    # reference known answers (tests/test_tensor.py:15-41)
    assert np.isinf(O.q16(np.float32(65520.0)))
    assert O.q16(np.float32(65519.9)) == 65504.0
    assert O.q16(np.float32(2.0 ** -25)) == 0.0
    assert O.q16(np.float32(2.0 ** -24)) == np.float32(2.0 ** -24)


def test_splitmix_stream_matches_reference(golden):
    g = golden("numerics")
    for seed, shape, lo, hi in [(0, (64,), 0.0, 1.0), (1, (3, 5, 7), -2.0, 3.0),
                                (2 ** 40 + 7, (33,), -0.5, 0.5)]:
        s = O.Stream(seed)
        got = np.concatenate([s.draw(shape, lo, hi).ravel(), s.draw(shape, lo, hi).ravel()])
        assert np.array_equal(got.view(np.uint32), g[f"rng_{seed}"].view(np.uint32))


def _op_cases(g):
    return sorted({k.split("__")[0] for k in g})


def run_oracle_op(name, g):
    half = name.split("_")[1] == "h"
    xs = []
    i = 0
    while f"{name}__x{i}" in g:
        xs.append(g[f"{name}__x{i}"])
        i += 1
    kind = name.split("_")[0]
    diff = [0, 1, 2] if kind in ("affine", "conv", "bn", "bnchain") else [0]
    f32 = range(1, 5) if kind in ("bn", "bnchain") else ()  # F32 BN parameters
    vs = [O.Var(a, half=(half and j not in f32), need_grad=(j in diff))
          for j, a in enumerate(xs)]
    if kind == "affine":
        y = O.affine(*vs, half)
    elif kind == "conv":
        _, _, cin, cout, k, s, p, hw = name.split("_")
        y = O.conv2d(*vs, (int(s), int(s)), (int(p), int(p)), half)
    elif kind == "pool":
        _, _, k, s, p, ib, hw = name.split("_")
        y = O.max_pooling(vs[0], (int(k), int(k)), (int(s), int(s)), (int(p), int(p)), half,
                          ignore_border=bool(int(ib)))
    elif kind == "relu":
        y = O.relu(vs[0], half)
    elif kind == "sce":
        y = O.softmax_ce(vs[0], vs[1], half)
    elif kind == "bn":
        y = O.batch_norm(*vs, half, batch_stat=bool(int(name.split("_")[2])))
    elif kind == "bnchain":  # BN -> affine -> SCE: a random upstream gradient into BN
        h = O.batch_norm(*vs[:5], half)
        y = O.softmax_ce(O.affine(h, vs[5], vs[6], half), vs[7], half)
    O.backward(y, 1.0)
    return y, vs, diff


def test_ops_match_reference_golden(golden):
    g = golden("ops")
    for name in _op_cases(g):
        y, vs, diff = run_oracle_op(name, g)
        tol = dict(rtol=2e-3, atol=2e-3) if "_h" in name else dict(rtol=1e-5, atol=1e-5)
        close(y.value, g[f"{name}__y"], **tol)
        for j in diff:
            close(vs[j].grad, g[f"{name}__g{j}"], **tol)


def test_pool_argmax_is_first_max(golden):
    g = golden("ops")
    x = np.array([[[[1.0, 1.0], [1.0, 1.0]]]], dtype=np.float32)
    y, arg = O.maxpool_forward(x, (2, 2), (2, 2), (0, 0))
    assert arg.item() == 0
    x = np.array([[[[0.0, np.nan], [np.nan, 5.0]]]], dtype=np.float32)
    y, arg = O.maxpool_forward(x, (2, 2), (2, 2), (0, 0))
    assert arg.item() == 1 and np.isnan(y.item())


def test_dynamic_scaler_sequence(golden):
    g = golden("solver")
    m = O.Model(0, half=True)
    w = O.Var(np.array([1.0, -2.0, 0.5, 3.0], np.float32), half=True, need_grad=True, name="w")
    m.params["w"] = w
    opt = O.Sgd(m, 0.1)
    sc = O.Scaler(8.0, 2.0, 2)
    for i, gr in enumerate(g["seq_grads"]):
        opt._master("w", w)
        w.grad = O.q16(gr * np.float32(sc.loss_scale))
        applied = O.dynamic_step(sc, opt)
        assert applied == bool(g["seq_applied"][i])
        assert sc.loss_scale == g["seq_scales"][i]
        assert np.array_equal(w.value, g["seq_w"][i])
    # interval 2: the overflows at steps 3 and 6 halve the scale and reset the
    # counter before it can exceed the interval, so no doubling happens
    assert list(g["seq_scales"]) == [8, 8, 4, 4, 4, 2, 2, 2]
    assert list(g["seq_applied"]) == [True, True, False, True, True, False, True, True]


@pytest.mark.parametrize("half", [False, True])
def test_clip_grad_by_norm_matches_reference(golden, half):
    """dynamic_step with clip_norm (solver.py:119-155): step 0 clips, step 1 not."""
    g = golden("solver")
    tag = "h" if half else "f"
    m = O.Model(0, half)
    a = O.Var(g[f"clip_{tag}_a_init"], half=half, need_grad=True)
    b = O.Var(g[f"clip_{tag}_b_init"], half=False, need_grad=True)
    m.params.update(a=a, b=b)
    opt = O.Sgd(m, 0.05, clip_norm=1.5)
    sc = O.Scaler(8.0, 2.0, 2000)
    for step in range(2):
        for k, v in (("a", a), ("b", b)):
            opt._master(k, v)
        a.grad = O.store(g[f"clip_{tag}_ga{step}"] * np.float32(sc.loss_scale), half)
        b.grad = O.store(g[f"clip_{tag}_gb{step}"] * np.float32(sc.loss_scale), False)
        assert O.dynamic_step(sc, opt)
        assert np.array_equal(a.grad, g[f"clip_{tag}_a{step}_grad"])
        assert np.array_equal(b.grad, g[f"clip_{tag}_b{step}_grad"])
        assert np.array_equal(opt.master["a"], g[f"clip_{tag}_a{step}_master"])
        assert np.array_equal(a.value, g[f"clip_{tag}_a{step}"])
        assert np.array_equal(b.value, g[f"clip_{tag}_b{step}"])


def _lenet_build(m, x, t):
    return m.sce(O.lenet(m, x, 10), t)


@pytest.mark.parametrize("half", [False, True])
def test_lenet_training_matches_reference(golden, half):
    g = golden("lenet")
    tag = "h" if half else "f"
    tr = O.Trainer(_lenet_build, 1, 16, 0.05, seed=0, half=half,
                   scaler=O.Scaler(8.0, 2.0, 2000) if half else None)
    losses = [tr.step(g["lenet_x"][s], g["lenet_labels"]) for s in range(3)]
    tol = dict(rtol=2e-3, atol=1e-3) if half else dict(rtol=1e-5, atol=1e-6)
    close(losses, g[f"lenet_{tag}_losses"], **tol)
    for k, v in tr.models[0].trainable().items():
        close(v.value, g[f"lenet_{tag}_final__{k}"], **tol)


@pytest.mark.parametrize("half", [False, True])
def test_dp2_matches_reference(golden, half):
    g = golden("lenet")
    tag = "h" if half else "f"
    tr = O.Trainer(_lenet_build, 2, 16, 0.05, seed=0, half=half,
                   scaler=O.Scaler(8.0, 2.0, 2000) if half else None)
    losses = [tr.step(g["lenet_x"][s], g["lenet_labels"]) for s in range(2)]
    tol = dict(rtol=2e-3, atol=1e-3) if half else dict(rtol=1e-5, atol=1e-6)
    close(losses, g[f"dp2_{tag}_losses"], **tol)
    for k, v in tr.models[0].trainable().items():
        close(v.value, g[f"dp2_{tag}_final__{k}"], **tol)


def test_mlp_matches_reference(golden):
    g = golden("mlp")

    def build(m, x, t):
        return m.sce(O.mlp(m, x, 10, hidden=(256,)), t)

    tr = O.Trainer(build, 1, 64, 0.1, seed=0)
    losses = [tr.step(g["mlp_x"][s], g["mlp_labels"]) for s in range(2)]
    close(losses, g["mlp_losses"], rtol=1e-5, atol=1e-6)
    for k, v in tr.models[0].trainable().items():
        close(v.value, g[f"mlp_final__{k}"], rtol=1e-5, atol=1e-6)


@pytest.mark.reference
def test_oracle_conv_grid_matches_live_reference(reference):
    import nanonnl.functions as RF
    rng = np.random.default_rng(0)
    for (cin, cout, k, s, p, hw) in [(5, 3, 3, 1, 1, 6), (2, 4, 3, 2, 0, 9), (3, 3, 1, 1, 0, 4)]:
        x = rng.uniform(-1, 1, (2, cin, hw, hw)).astype(np.float32)
        w = rng.uniform(-1, 1, (cout, cin, k, k)).astype(np.float32)
        b = rng.uniform(-1, 1, (cout,)).astype(np.float32)
        reference.set_default_context(reference.ExecutionContext())
        rv = [reference.Variable(a.shape, need_grad=True) for a in (x, w, b)]
        for v, a in zip(rv, (x, w, b)):
            v.d = a
        ry = RF.convolution(*rv, stride=(s, s), pad=(p, p))
        ry.forward()
        ry.backward(1.0)
        ov = [O.Var(a, need_grad=True) for a in (x, w, b)]
        oy = O.conv2d(*ov, (s, s), (p, p), False)
        O.backward(oy, 1.0)
        close(oy.value, ry.d, rtol=1e-5, atol=1e-5)
        for o, r in zip(ov, rv):
            close(o.grad, r.g, rtol=1e-5, atol=1e-5)


@pytest.mark.reference
def test_oracle_resnet_parameter_order_uses_reference_initializer(reference):
    """The ResNet parameter draws follow the reference initializer + stream."""
    from nanonnl.parameters import default_initializer
    from nanonnl.tensor import RngState
    m = O.Model(0, half=False)
    x = O.Var(np.zeros((2, 3, 32, 32), np.float32))
    O.resnet18_cifar(m, x, 10)
    rng = RngState(0)
    for name, v in m.params.items():
        want = default_initializer(name.rsplit("/", 1)[-1], v.shape, rng)
        if name.endswith("/mean") or name.endswith("/var"):
            want = np.ones(v.shape, np.float32) if name.endswith("/var") else want
        if not (name.endswith("/mean") or name.endswith("/var")):
            assert np.array_equal(v.value, want), name
