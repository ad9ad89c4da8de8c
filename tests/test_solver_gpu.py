"""Solver parity on the device: the Momentum/weight-decay update the benchmark
runs, with dynamic loss scaling and an overflow-skipped step, bitwise against
the oracle (oracle/nnl_oracle.py Sgd, the restatement of solver.py:100-155 +
the NNabla Momentum extension), and clip_grad_by_norm against the reference's
own golden (tests/golden/make_golden.py gen_solver, solver.py:119-129)."""

import numpy as np
import pytest

from oracle import nnl_oracle as O

pytestmark = pytest.mark.gpu


def _params(nnl, half, a0, b0):
    tc = nnl.TypeConfig.HALF if half else nnl.TypeConfig.FLOAT
    nnl.set_default_context(nnl.ExecutionContext(type_config=tc))
    a = nnl.Variable(a0.shape, need_grad=True)
    b = nnl.Variable(b0.shape, need_grad=True, dtype=nnl.Dtype.F32)  # BN-style f32 param
    w = nnl.Variable((3, 4, 3, 3), need_grad=True)  # conv layout: physical KRSC on device
    a.d, b.d = a0, b0
    w.d = O.uniform(9, 0, w.shape, -1, 1)
    return {"a": a, "b": b, "w": w}


@pytest.mark.parametrize("half", [False, True])
@pytest.mark.parametrize("device_scaler", [False, True])
def test_momentum_weight_decay_update_bitwise(nnl, half, device_scaler):
    """4 dynamic steps (lr 0.05, momentum 0.9, wd 1e-4) with an inf gradient at
    step 2: weights, f32 masters and velocities bit-identical to the oracle
    every step; the skipped step leaves all three byte-unchanged."""
    a0 = O.uniform(3, 0, (37, 5), -1, 1)
    b0 = O.uniform(4, 0, (5,), -1, 1)
    params = _params(nnl, half, a0, b0)
    solver = nnl.SgdSolver(0.05, momentum=0.9, weight_decay=1e-4).setup(params)
    host_sc = nnl.DynamicLossScaler(8.0, 2.0, 1)  # interval 1: a doubling happens too
    dev_sc = nnl.DeviceLossScaler(host_sc) if device_scaler else None

    m = O.Model(0, half)
    ov = {k: O.Var(v.d, half=half and k != "b", need_grad=True) for k, v in params.items()}
    m.params.update(ov)
    opt = O.Sgd(m, 0.05, momentum=0.9, weight_decay=1e-4)
    osc = O.Scaler(8.0, 2.0, 1)
    for k, v in ov.items():
        opt._master(k, v)

    prev = None
    for step in range(5):
        scale = osc.loss_scale
        grads = {k: O.uniform(100 + step, 7 * i, v.shape, -2, 2) * np.float32(scale)
                 for i, (k, v) in enumerate(params.items())}
        if step == 2:
            grads["a"][3, 1] = np.inf
        for k, v in params.items():
            v.g = grads[k]
            ov[k].grad = O.store(grads[k], ov[k].half)
        want_applied = O.dynamic_step(osc, opt)
        if device_scaler:
            solver.dynamic_update(dev_sc, check=True)
            got_applied = dev_sc.last_applied()
            assert dev_sc.snapshot().loss_scale == osc.loss_scale
        else:
            got_applied = nnl.dynamic_step(host_sc, solver).applied
            assert host_sc.loss_scale == osc.loss_scale
        assert got_applied == want_applied == (step != 2)
        state = {}
        for k, v in params.items():
            state[k] = (v.d, solver.master_values(k), solver.velocity_values(k))
            assert np.array_equal(state[k][0], ov[k].value), (step, k)
            assert np.array_equal(state[k][1], opt.master[k]), (step, k)
            assert np.array_equal(state[k][2], opt.vel[k]), (step, k)
        if step == 2:  # SkippedInfNan: bytes unchanged
            for k in params:
                for x, y in zip(state[k], prev[k]):
                    assert x.tobytes() == y.tobytes(), k
        prev = state


@pytest.mark.parametrize("half", [False, True])
def test_clip_grad_by_norm_matches_reference(nnl, golden, half):
    """dynamic_step with clip_norm=1.5 against the reference run: step 0 clips
    (global norm ~7.8), step 1 does not.  The global norm is summed in f64 on
    the device, the reference sums per-parameter f32 pairwise sums, so the
    clip factor may differ in its last f32 bit: clipped gradients agree to
    1 ulp of their storage type, everything downstream within that."""
    g = golden("solver")
    tag = "h" if half else "f"
    tc = nnl.TypeConfig.HALF if half else nnl.TypeConfig.FLOAT
    nnl.set_default_context(nnl.ExecutionContext(type_config=tc))
    a = nnl.Variable((37, 5), need_grad=True)
    b = nnl.Variable((5,), need_grad=True, dtype=nnl.Dtype.F32)
    a.d = g[f"clip_{tag}_a_init"]
    b.d = g[f"clip_{tag}_b_init"]
    solver = nnl.SgdSolver(0.05, clip_norm=1.5).setup({"a": a, "b": b})
    sc = nnl.DynamicLossScaler(8.0, 2.0, 2000)
    ulp = 2.0 ** -10 if half else 2.0 ** -23
    for step in range(2):
        a.g = g[f"clip_{tag}_ga{step}"] * np.float32(sc.loss_scale)
        b.g = g[f"clip_{tag}_gb{step}"] * np.float32(sc.loss_scale)
        assert nnl.dynamic_step(sc, solver).applied
        for got, key, u in ((a.g, "a", ulp), (b.g, "b", 2.0 ** -23)):
            want = g[f"clip_{tag}_{key}{step}_grad"]
            np.testing.assert_allclose(got, want, rtol=2 * u, atol=0)
        np.testing.assert_allclose(solver.master_values("a"), g[f"clip_{tag}_a{step}_master"],
                                   rtol=1e-6, atol=1e-7)
        np.testing.assert_allclose(a.d, g[f"clip_{tag}_a{step}"], rtol=2 * ulp, atol=1e-7)
        np.testing.assert_allclose(b.d, g[f"clip_{tag}_b{step}"], rtol=1e-6, atol=1e-7)
        if step == 1:  # below the clip threshold: exactly the unclipped update
            assert np.array_equal(a.g, g[f"clip_{tag}_a{step}_grad"])
