"""Generate golden vectors by running the REFERENCE package (nanonnl).

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

Writes tests/golden/*.npz.  The GPU box has no /root/reference, so these
committed fixtures are what pins both the oracle restatement and the CUDA
path there.  Inputs are seeded through the reference's own RngState.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def _ref():
    sys.path.insert(0, REF)
    import nanonnl as nn
    import nanonnl.functions as F
    import nanonnl.parametric as PF
    from nanonnl import networks
    from nanonnl.communicator import DataParallelTrainer
    return nn, F, PF, networks, DataParallelTrainer


def fresh(nn, half: bool, seed: int = 0):
    tc = nn.TypeConfig.HALF if half else nn.TypeConfig.FLOAT
    nn.set_default_context(nn.ExecutionContext(type_config=tc))
    reg = nn.ParameterRegistry(seed=seed)
    return reg


def gen_numerics(nn):
    from nanonnl.tensor import RngState
    vals = np.array([65520.0, 65519.9, 2.0 ** -25, 2.0 ** -24, 1.0, 1.0 + 2 ** -13, 7e4,
                     -65504.0, 3.14159, -2.0 ** -20, 0.1, 1e-8, 6.1e-5, np.inf, -np.inf],
                    dtype=np.float32)
    rnd = RngState(seed=11).next_uniform((512,), -70000.0, 70000.0)
    tiny = RngState(seed=12).next_uniform((512,), -1e-4, 1e-4)
    q = np.array([nn.quantize_f16(float(v)) for v in np.concatenate([vals, rnd, tiny])],
                 dtype=np.float32)
    draws = {}
    for seed, shape, lo, hi in [(0, (64,), 0.0, 1.0), (1, (3, 5, 7), -2.0, 3.0),
                                (2 ** 40 + 7, (33,), -0.5, 0.5)]:
        r = RngState(seed=seed)
        a = r.next_uniform(shape, lo, hi)
        b = r.next_uniform(shape, lo, hi)
        draws[f"rng_{seed}"] = np.concatenate([a.ravel(), b.ravel()])
    return dict(q_in=np.concatenate([vals, rnd, tiny]), q_out=q, **draws)


def run_op(nn, build, inputs, half, diff, seed=1.0, f32_range=None):
    vs = []
    for i, a in enumerate(inputs):
        dt = nn.Dtype.F32 if (f32_range is not None and f32_range[0] <= i < f32_range[1]) \
            else None
        v = nn.Variable(a.shape, need_grad=(i in diff), dtype=dt)
        v.d = a
        vs.append(v)
    out = build(vs)
    out.forward()
    out.backward(seed)
    res = {"y": out.d.copy()}
    for i in diff:
        res[f"g{i}"] = vs[i].g.copy()
    return res


def gen_ops(nn, F):
    from nanonnl.tensor import RngState
    rng = RngState(seed=5)
    out = {}
    cases = []
    # (name, builder, input shapes/ranges, diff indices)
    for half in (False, True):
        tag = "h" if half else "f"
        fresh(nn, half)
        x = rng.next_uniform((4, 6), -1, 1)
        w = rng.next_uniform((6, 5), -1, 1)
        b = rng.next_uniform((5,), -1, 1)
        cases.append((f"affine_{tag}", half, lambda v: F.affine(*v), [x, w, b], [0, 1, 2]))
        for (cin, cout, k, s, p, hw) in [(3, 4, 3, 1, 1, 7), (2, 3, 3, 2, 1, 8), (4, 2, 1, 2, 0, 6),
                                         (1, 2, 5, 1, 0, 9), (3, 2, 7, 2, 3, 11)]:
            x = rng.next_uniform((2, cin, hw, hw), -1, 1)
            w = rng.next_uniform((cout, cin, k, k), -1, 1)
            b = rng.next_uniform((cout,), -1, 1)
            cases.append((f"conv_{tag}_{cin}_{cout}_{k}_{s}_{p}_{hw}", half,
                          (lambda s_, p_: lambda v: F.convolution(v[0], v[1], v[2], stride=(s_, s_),
                                                                  pad=(p_, p_)))(s, p),
                          [x, w, b], [0, 1, 2]))
        for (k, s, p, ib, hw) in [(2, 2, 0, True, 8), (3, 2, 1, True, 9), (3, 2, 0, False, 8),
                                  (2, 1, 0, True, 5)]:
            x = rng.next_uniform((2, 3, hw, hw), -1, 1)
            x = np.round(x * 4) / 4  # plenty of ties
            cases.append((f"pool_{tag}_{k}_{s}_{p}_{int(ib)}_{hw}", half,
                          (lambda k_, s_, p_, ib_: lambda v: F.max_pooling(
                              v[0], (k_, k_), (s_, s_), ignore_border=ib_, pad=(p_, p_)))(k, s, p, ib),
                          [x], [0]))
        x = np.array([[-1.0, 0.0, 2.0, np.nan, -np.inf, np.inf, 1e-9, -1e-9]], dtype=np.float32)
        cases.append((f"relu_{tag}", half, lambda v: F.relu(v[0]), [x], [0]))
        lg = rng.next_uniform((6, 10), -3, 3)
        lab = (np.arange(6) * 7 % 10).astype(np.float32)
        cases.append((f"sce_{tag}", half, lambda v: F.softmax_cross_entropy(v[0], v[1]), [lg, lab],
                      [0]))
        for bs in (True, False):
            x = rng.next_uniform((3, 4, 5, 5), -2, 2)
            g = rng.next_uniform((4,), 0.5, 1.5)
            be = rng.next_uniform((4,), -0.5, 0.5)
            m = rng.next_uniform((4,), -0.1, 0.1)
            vv = rng.next_uniform((4,), 0.5, 1.5)

            def bnb(v, bs=bs):
                return F.batch_normalization(*v, batch_stat=bs)

            cases.append((f"bn_{tag}_{int(bs)}", half, bnb, [x, g, be, m, vv], [0, 1, 2]))
        # BN backward under a non-trivial upstream gradient: BN -> affine -> SCE
        # (a ones seed straight into BN makes dx and dgamma vanish), with one
        # channel offset far from zero (|mean| >> std: two-pass variance)
        r6 = RngState(seed=6 + int(half))  # own stream: earlier cases keep their draws
        x = r6.next_uniform((4, 3, 6, 6), -1, 1)
        x[:, 1] += 64.0
        g = r6.next_uniform((3,), 0.5, 1.5)
        be = r6.next_uniform((3,), -0.5, 0.5)
        m = np.zeros(3, np.float32)
        vv = np.ones(3, np.float32)
        wa = r6.next_uniform((108, 10), -1, 1)
        ba = r6.next_uniform((10,), -1, 1)
        lab = (np.arange(4) * 3 % 10).astype(np.float32)

        def bn_chain(v):
            y = F.batch_normalization(v[0], v[1], v[2], v[3], v[4])
            return F.softmax_cross_entropy(F.affine(y, v[5], v[6]), v[7])

        cases.append((f"bnchain_{tag}", half, bn_chain, [x, g, be, m, vv, wa, ba, lab], [0, 1, 2]))
    for name, half, build, inputs, diff in cases:
        fresh(nn, half)
        # BN scale/shift/statistics are F32 as PF.batch_normalization makes them
        f32 = {"bn_": (1, 5), "bnchain_": (1, 5)}
        rng32 = next((r for k, r in f32.items() if name.startswith(k)), None)
        res = run_op(nn, build, inputs, half, diff, seed=1.0, f32_range=rng32)
        for i, a in enumerate(inputs):
            out[f"{name}__x{i}"] = a
        for k, v in res.items():
            out[f"{name}__{k}"] = v
    return out


def gen_solver(nn):
    from nanonnl import DynamicLossScaler, SgdSolver, dynamic_step
    out = {}
    # scales [8,8,8,16,16] with interval 2 (reference tests/test_solver.py:175-183)
    fresh(nn, True)
    with nn.registry_scope(nn.ParameterRegistry(0)):
        w = nn.Variable((4,), need_grad=True)
        w.d = np.array([1.0, -2.0, 0.5, 3.0], dtype=np.float32)
        s = SgdSolver(0.1).setup({"w": w})
        sc = DynamicLossScaler(8.0, 2.0, 2)
        scales, applied, ws = [], [], []
        grads = [[1, 2, 3, 4], [0.5, 0.25, 1, 2], [np.inf, 1, 1, 1], [1, 1, 1, 1], [2, 2, 2, 2],
                 [1e5, 1, 1, 1], [0.1, 0.1, 0.1, 0.1], [3, 3, 3, 3]]
        for g in grads:
            w.g = np.array(g, dtype=np.float32) * np.float32(sc.loss_scale)
            o = dynamic_step(sc, s)
            scales.append(sc.loss_scale)
            applied.append(o.applied)
            ws.append(w.d.copy())
        out.update(seq_grads=np.array(grads, dtype=np.float32), seq_scales=np.array(scales),
                   seq_applied=np.array(applied), seq_w=np.array(ws))
        # half master accumulates below the visible resolution (test_solver.py:80-90)
        w2 = nn.Variable((1,), need_grad=True)
        w2.d = np.array([1.0], dtype=np.float32)
        s2 = SgdSolver(2.0 ** -16).setup({"w": w2})
        vis = []
        for _ in range(3):
            w2.g = np.array([1.0], dtype=np.float32)
            s2.update()
            vis.append(float(w2.d[0]))
        out.update(master_w=np.array(vis), master_m=s2.slots["w"].master.copy())
    # clip_grad_by_norm (solver.py:119-129) inside dynamic_step, F16 + F32
    # parameters; step 1 clips (norm > 1.5), step 2 does not
    from nanonnl.tensor import RngState
    for half in (False, True):
        tag = "h" if half else "f"
        fresh(nn, half)
        r = RngState(seed=21)
        with nn.registry_scope(nn.ParameterRegistry(0)):
            a = nn.Variable((37, 5), need_grad=True)
            b = nn.Variable((5,), need_grad=True, dtype=nn.Dtype.F32)
            a.d = r.next_uniform((37, 5), -1, 1)
            b.d = r.next_uniform((5,), -1, 1)
            out[f"clip_{tag}_a_init"] = a.d.copy()
            out[f"clip_{tag}_b_init"] = b.d.copy()
            s3 = SgdSolver(0.05, clip_norm=1.5).setup({"a": a, "b": b})
            sc = DynamicLossScaler(8.0, 2.0, 2000)
            for step, mag in enumerate((1.0, 0.01)):
                ga = r.next_uniform((37, 5), -mag, mag)
                gb = r.next_uniform((5,), -mag, mag)
                out[f"clip_{tag}_ga{step}"] = ga
                out[f"clip_{tag}_gb{step}"] = gb
                a.g = ga * np.float32(sc.loss_scale)
                b.g = gb * np.float32(sc.loss_scale)
                assert dynamic_step(sc, s3).applied
                out[f"clip_{tag}_a{step}"] = a.d.copy()
                out[f"clip_{tag}_b{step}"] = b.d.copy()
                out[f"clip_{tag}_a{step}_grad"] = a.g.copy()
                out[f"clip_{tag}_b{step}_grad"] = b.g.copy()
                out[f"clip_{tag}_a{step}_master"] = s3.slots["a"].master.copy()
    return out


def gen_lenet(nn, networks, DataParallelTrainer):
    import nanonnl.functions as F
    from nanonnl import DynamicLossScaler, SgdSolver, dynamic_step
    from nanonnl.tensor import RngState
    out = {}
    B = 16
    x = RngState(seed=1).next_uniform((3, B, 1, 28, 28), 0, 1)
    lab = (np.arange(B) % 10).astype(np.float32)
    for half in (False, True):
        tag = "h" if half else "f"
        fresh(nn, half)
        with nn.registry_scope(nn.ParameterRegistry(0)) as reg:
            xv = nn.Variable((B, 1, 28, 28))
            tv = nn.Variable((B,))
            logits = networks.lenet(xv, 10)
            loss = F.softmax_cross_entropy(logits, tv)
            params = reg.get_parameters()
            for k, v in params.items():
                out[f"lenet_{tag}_init__{k}"] = v.d.copy()
            solver = SgdSolver(0.05).setup(params)
            sc = DynamicLossScaler(8.0, 2.0, 2000)
            losses = []
            for step in range(3):
                xv.d = x[step]
                tv.d = lab
                loss.forward()
                if half:
                    loss.backward(grad_seed=sc.loss_scale)
                    if step == 0:
                        for k, v in params.items():
                            out[f"lenet_{tag}_grad0__{k}"] = v.g.copy()
                    dynamic_step(sc, solver)
                else:
                    loss.backward()
                    if step == 0:
                        for k, v in params.items():
                            out[f"lenet_{tag}_grad0__{k}"] = v.g.copy()
                    solver.update()
                losses.append(float(loss.d))
            out[f"lenet_{tag}_losses"] = np.array(losses)
            for k, v in params.items():
                out[f"lenet_{tag}_final__{k}"] = v.d.copy()
    out["lenet_x"] = x
    out["lenet_labels"] = lab

    # DataParallelTrainer K=2 on LeNet (F32 and Half, dynamic scaling)
    def build(bs):
        xv = nn.Variable((bs, 1, 28, 28))
        tv = nn.Variable((bs,))
        return {"x": xv, "label": tv, "loss": F.softmax_cross_entropy(networks.lenet(xv, 10), tv)}

    for half in (False, True):
        tag = "h" if half else "f"
        fresh(nn, half)
        tr = DataParallelTrainer(2, B, build, lr=0.05, seed=0,
                                 loss_scaling=DynamicLossScaler(8.0, 2.0, 2000) if half else None)
        losses = [tr.step(x[i], lab) for i in range(2)]
        out[f"dp2_{tag}_losses"] = np.array(losses)
        for k, v in tr.rank0.registry.get_parameters().items():
            out[f"dp2_{tag}_final__{k}"] = v.d.copy()
    return out


def gen_mlp(nn, networks):
    import nanonnl.functions as F
    from nanonnl import SgdSolver
    from nanonnl.tensor import RngState
    out = {}
    fresh(nn, False)
    B = 64
    x = RngState(seed=1).next_uniform((2, B, 784), 0, 1)
    lab = (np.arange(B) % 10).astype(np.float32)
    with nn.registry_scope(nn.ParameterRegistry(0)) as reg:
        xv = nn.Variable((B, 784))
        tv = nn.Variable((B,))
        loss = F.softmax_cross_entropy(networks.mlp(xv, 10, hidden=(256,)), tv)
        params = reg.get_parameters()
        solver = SgdSolver(0.1).setup(params)
        losses = []
        for s in range(2):
            xv.d = x[s]
            tv.d = lab
            loss.forward()
            loss.backward()
            solver.update()
            losses.append(float(loss.d))
        out["mlp_losses"] = np.array(losses)
        for k, v in params.items():
            out[f"mlp_final__{k}"] = v.d.copy()
    out["mlp_x"] = x
    out["mlp_labels"] = lab
    return out


def gen_nnp(nn, networks):
    """The reference's parameter.bin bytes (nnp.py:467-481) for a half LeNet's
    registry (F16 weights, F32 BN-free) plus an F32 record, for the checkpoint
    format test."""
    from nanonnl.nnp import ParameterRecord, emit_parameter_bin
    reg = fresh(nn, True)
    with nn.registry_scope(reg):
        networks.lenet(nn.Variable((2, 1, 28, 28)), 10)
    recs = [ParameterRecord(k, v.shape, v.dtype, v.d.copy(), v.need_grad)
            for k, v in reg.get_parameters(grad_only=False).items()]
    recs.append(ParameterRecord("extra_f32", (3,), nn.Dtype.F32,
                                np.array([1.5, -2.25, 3e-8], np.float32), False))
    out = {"bin": np.frombuffer(emit_parameter_bin(recs), np.uint8).copy(),
           "names": np.array([r.name for r in recs]),
           "f16": np.array([r.dtype is nn.Dtype.F16 for r in recs]),
           "need_grad": np.array([r.need_grad for r in recs])}
    for i, r in enumerate(recs):
        out[f"v{i}"] = r.values
    return out


# operator-protocol cases for the reference-side binding (nanonnl_plugin): the
# reference's own FunctionImpl classes driven exactly as its engine drives them
# (infer_shapes, forward(node, xs), backward(node, gys, want)), float32, with a
# random upstream gradient
PLUGIN_CASES = [
    ("affine", "Affine", {}, [(4, 3, 5), (15, 6), (6,)]),
    ("conv", "Convolution", {"stride": (2, 2), "pad": (1, 1), "kernel": (3, 3)},
     [(2, 3, 9, 9), (4, 3, 3, 3), (4,)]),
    ("pool", "MaxPooling", {"kernel": (3, 3), "stride": (2, 2), "pad": (1, 1)}, [(2, 3, 7, 7)]),
    ("relu", "ReLU", {}, [(3, 10)]),
    ("sce", "SoftmaxCrossEntropy", {}, [(5, 7), (5,)]),
    ("bn", "BatchNormalization", {"eps": 1e-5, "momentum": 0.9, "batch_stat": True},
     [(4, 3, 5, 5), (3,), (3,), (3,), (3,)]),
]


def gen_plugin(nn):
    from types import SimpleNamespace

    import nanonnl.functions as RF
    from nanonnl.tensor import RngState
    rng = RngState(seed=21)
    fresh(nn, False)
    out = {}
    for name, kind, args, shapes in PLUGIN_CASES:
        xs = [rng.next_uniform(s, -1.0, 1.0) for s in shapes]
        if kind == "SoftmaxCrossEntropy":
            xs[1] = (np.arange(shapes[1][0]) * 3 % shapes[0][1]).astype(np.float32)
        if kind == "BatchNormalization":
            xs[1] = rng.next_uniform(shapes[1], 0.5, 1.5)
            xs[4] = rng.next_uniform(shapes[4], 0.5, 1.5)
        if kind == "MaxPooling":
            xs[0] = np.round(xs[0] * 4) / 4  # ties: first max wins
        vs = []
        for i, a in enumerate(xs):
            v = nn.Variable(a.shape, need_grad=not (kind == "SoftmaxCrossEntropy" and i == 1))
            v.d = a
            vs.append(v)
        impl = RF.REGISTRY[kind](**args)
        ys_shapes = impl.infer_shapes([v.shape for v in vs])
        node = SimpleNamespace(inputs=vs, state={})
        ys = impl.forward(node, [v.data.values for v in vs])
        gys = [rng.next_uniform(s, -1.0, 1.0) for s in ys_shapes]
        want = [v.need_grad for v in vs]
        gxs = impl.backward(node, gys, want)
        for i, a in enumerate(xs):
            out[f"{name}__x{i}"] = a
        for j, (y, gy) in enumerate(zip(ys, gys)):
            out[f"{name}__y{j}"] = np.asarray(y, np.float32)
            out[f"{name}__gy{j}"] = gy
        for i, g in enumerate(gxs):
            if g is not None:
                out[f"{name}__g{i}"] = np.asarray(g, np.float32)
        if kind == "BatchNormalization":
            out[f"{name}__mean"] = vs[3].d.copy()
            out[f"{name}__var"] = vs[4].d.copy()
    return out


def main():
    nn, F, PF, networks, DPT = _ref()
    np.savez_compressed(os.path.join(HERE, "nnp.npz"), **gen_nnp(nn, networks))
    np.savez_compressed(os.path.join(HERE, "numerics.npz"), **gen_numerics(nn))
    np.savez_compressed(os.path.join(HERE, "ops.npz"), **gen_ops(nn, F))
    np.savez_compressed(os.path.join(HERE, "solver.npz"), **gen_solver(nn))
    np.savez_compressed(os.path.join(HERE, "lenet.npz"), **gen_lenet(nn, networks, DPT))
    np.savez_compressed(os.path.join(HERE, "mlp.npz"), **gen_mlp(nn, networks))
    np.savez_compressed(os.path.join(HERE, "plugin.npz"), **gen_plugin(nn))
    for f in sorted(os.listdir(HERE)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(HERE, f)))


if __name__ == "__main__":
    main()
