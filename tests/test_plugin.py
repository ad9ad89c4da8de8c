"""The reference-side binding (paper_2102_06725_b200/nanonnl_plugin.py): libnnl
kernels registered into nanonnl's own operator REGISTRY.

* `reference` tests (build container): install into the live nanonnl, check the
  device classes are the reference's classes (KIND/ARGS/infer_shapes and its
  errors) and that the golden fixture is what the reference computes.
* `gpu` tests: the device classes driven exactly as nanonnl's engine drives an
  operator (infer_shapes, forward(node, xs), backward(node, gys, want);
  src/graph.py:226-237, 353-363) against tests/golden/plugin.npz, which the
  reference produced through the same protocol (make_golden.gen_plugin).
"""

import numpy as np
import pytest

ARGS = {  # tests/golden/make_golden.py PLUGIN_CASES
    "affine": ("Affine", {}),
    "conv": ("Convolution", {"stride": (2, 2), "pad": (1, 1), "kernel": (3, 3)}),
    "pool": ("MaxPooling", {"kernel": (3, 3), "stride": (2, 2), "pad": (1, 1)}),
    "relu": ("ReLU", {}),
    "sce": ("SoftmaxCrossEntropy", {}),
    "bn": ("BatchNormalization", {"eps": 1e-5, "momentum": 0.9, "batch_stat": True}),
}


@pytest.mark.reference
def test_install_into_reference_registry(reference):
    import nanonnl.functions as RF
    import nanonnl.parametric as PF
    from nanonnl.errors import ShapeMismatch

    from paper_2102_06725_b200 import nanonnl_plugin as P
    before = dict(RF.REGISTRY)
    saved = P.install(RF)
    try:
        for kind in P.KINDS:
            cls = RF.REGISTRY[kind]
            assert issubclass(cls, before[kind]) and cls is not before[kind]
            assert cls.KIND == before[kind].KIND and cls.ARGS == before[kind].ARGS
        reference.set_default_context(reference.ExecutionContext())
        with reference.registry_scope(reference.ParameterRegistry(0)):
            x = reference.Variable((2, 3, 8, 8), need_grad=True)
            y = PF.convolution(x, 4, (3, 3), pad=(1, 1))
            assert type(y.parent.impl).__name__ == "DeviceConvolution"
            assert y.shape == (2, 4, 8, 8)
            # the reference's own shape errors, raised eagerly at apply()
            w = reference.Variable((5, 7))
            b = reference.Variable((7,))
            with pytest.raises(ShapeMismatch):
                RF.affine(x, w, b)
    finally:
        P.uninstall(RF, saved)
    assert RF.REGISTRY == before


@pytest.mark.reference
def test_plugin_golden_is_the_reference(reference, golden):
    import os
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(__file__), "golden"))
    import make_golden
    fresh = make_golden.gen_plugin(reference)
    g = golden("plugin")
    assert sorted(fresh) == sorted(g)
    for k, v in fresh.items():
        a, b = np.atleast_1d(np.asarray(v)), np.atleast_1d(np.asarray(g[k]))
        assert a.dtype == b.dtype and np.array_equal(a.view(np.uint8), b.view(np.uint8)), k


class _Data:
    def __init__(self, values):
        self.values = np.asarray(values, np.float32)

    def write(self, values):
        self.values = np.asarray(values, np.float32)


class _Var:
    """What nanonnl's engine hands an operator: .data.values / .data.write, .need_grad."""

    def __init__(self, values, need_grad):
        self.data = _Data(values)
        self.need_grad = need_grad


class _Node:
    def __init__(self, inputs):
        self.inputs = inputs
        self.state = {}


def _close(got, want, rtol=2e-5):
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    scale = np.abs(want).max() + 1e-6
    assert got.shape == want.shape
    assert np.abs(got - want).max() <= rtol * scale + 1e-7, (np.abs(got - want).max(), scale)


@pytest.mark.gpu
@pytest.mark.parametrize("case", sorted(ARGS))
def test_device_operator_protocol_matches_reference(nnl, golden, case):
    from paper_2102_06725_b200 import _lib, nanonnl_plugin as P
    g = golden("plugin")
    kind, args = ARGS[case]
    impl = P.make_impls()[kind](**args)
    xs = []
    i = 0
    while f"{case}__x{i}" in g:
        xs.append(g[f"{case}__x{i}"])
        i += 1
    vs = [_Var(a, not (kind == "SoftmaxCrossEntropy" and j == 1)) for j, a in enumerate(xs)]
    shapes = impl.infer_shapes([v.data.values.shape for v in vs])
    node = _Node(vs)
    before = _lib.lib().nnl_launch_count(0)
    ys = impl.forward(node, [v.data.values for v in vs])
    assert _lib.lib().nnl_launch_count(0) > before  # computed by libnnl
    assert [tuple(np.shape(y)) for y in ys] == [tuple(s) for s in shapes]
    for j, y in enumerate(ys):
        _close(y, g[f"{case}__y{j}"])
    if kind == "BatchNormalization":  # running statistics written back into the inputs
        _close(vs[3].data.values, g[f"{case}__mean"])
        _close(vs[4].data.values, g[f"{case}__var"])
    gys = [g[f"{case}__gy{j}"] for j in range(len(ys))]
    gxs = impl.backward(node, gys, [v.need_grad for v in vs])
    for j, gx in enumerate(gxs):
        key = f"{case}__g{j}"
        if key in g:
            _close(gx, g[key], rtol=5e-5)
        else:
            assert gx is None
