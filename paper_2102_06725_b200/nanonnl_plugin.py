"""Reference-side binding: libnnl kernels behind nanonnl's OWN operator protocol.

The reference engine (``nanonnl``, ``src/graph.py:226-237`` and ``:353-363``)
calls ``impl.forward(node, xs) -> [np.ndarray]`` and
``impl.backward(node, gys, want) -> [np.ndarray | None]`` on the classes in
``nanonnl.functions.REGISTRY`` (``src/functions.py:444-447``).  ``install()``
replaces those entries with device-backed subclasses of the reference's own
classes, so ``KIND``/``ARGS``/``infer_shapes``/``output_dtype``/
``backward_reads_input``/``args_dict`` (and every error they raise) stay the
reference's, while the arithmetic runs in libnnl on the GPU:

    import nanonnl, nanonnl.functions
    from paper_2102_06725_b200 import nanonnl_plugin
    nanonnl_plugin.install(nanonnl.functions)      # returns the replaced classes
    ...  # nanonnl graphs, solvers, DataParallelTrainer unchanged
    nanonnl_plugin.uninstall(nanonnl.functions, saved)

Each reference node gets a one-node shadow graph of this package in float32
(``TypeConfig.FLOAT``): inputs are uploaded, the kernel runs, outputs are
returned as float32 host arrays and the reference engine quantizes them on
write (R1) exactly as it does its own numpy results.  Per-node device state
(max-pool indices, batch-norm statistics, softmax probabilities) lives in the
shadow node, which is cached in ``node.state`` and reused while the shapes
hold.  BatchNormalization's running-statistics update is written back into
the reference's mean/var inputs (``src/functions.py:404-409``).

No import of nanonnl happens here: the base classes come from the module passed
to ``install``/``make_impls``; without one, this package's own operator
classes (same KIND/ARGS and shape rules) stand in, which is what the GPU tests
use on hosts without the reference.
"""

from __future__ import annotations

import numpy as np

KINDS = ("Affine", "Convolution", "MaxPooling", "ReLU", "SoftmaxCrossEntropy",
         "BatchNormalization")


class _Shadow:
    """A one-node graph of this package mirroring one reference node."""

    def __init__(self, kind: str, args: dict, in_shapes, need_grads):
        from . import graph
        self._graph = graph
        # float32 storage, static mode: apply() builds the node, forward() runs it
        ctx = graph.ExecutionContext(mode=graph.Mode.STATIC, type_config=graph.TypeConfig.FLOAT)
        with graph.context_scope(ctx):
            self.inputs = [graph.Variable(tuple(s), need_grad=bool(g))
                           for s, g in zip(in_shapes, need_grads)]
            self.outputs = graph.apply(kind, self.inputs, args)
        self.node = self.outputs[0].parent
        self.shapes = [tuple(s) for s in in_shapes]

    def forward(self, xs):
        for v, a in zip(self.inputs, xs):
            v.d = np.asarray(a, dtype=np.float32)
        self._graph._execute(self.node)
        return [np.asarray(o.d, dtype=np.float32) for o in self.outputs]

    def backward(self, gys, want):
        node = self.node
        for o, g in zip(self.outputs, gys):
            o.g = np.asarray(g, dtype=np.float32)
        gxs = []
        for v, w in zip(self.inputs, want):
            if w and v.need_grad:
                v.grad.fill(0.0)
                gxs.append(v.grad)
            else:
                gxs.append(None)
        node.impl.backward(node, [o.grad for o in self.outputs], gxs, [False] * len(gxs))
        return [np.asarray(v.g, dtype=np.float32) if g is not None else None
                for v, g in zip(self.inputs, gxs)]


def _shadow(impl, node, xs) -> _Shadow:
    shapes = [tuple(np.shape(a)) for a in xs]
    sh = node.state.get("nnl_shadow")
    if sh is None or sh.shapes != shapes:
        need = [getattr(v, "need_grad", True) for v in node.inputs]
        sh = _Shadow(impl.KIND, impl.args_dict(), shapes, need)
        node.state["nnl_shadow"] = sh
    return sh


def _device_class(base: type) -> type:
    """A subclass of the reference operator `base` whose arithmetic is libnnl's."""

    def forward(self, node, xs):
        sh = _shadow(self, node, xs)
        outs = sh.forward(xs)
        if self.KIND == "BatchNormalization" and getattr(self, "batch_stat", True):
            # running statistics, updated in place like src/functions.py:406-409
            for i in (3, 4):
                node.inputs[i].data.write(np.asarray(sh.inputs[i].d, dtype=np.float32))
        return outs

    def backward(self, node, gys, want):
        sh = node.state["nnl_shadow"]
        want = list(want)
        if self.KIND == "BatchNormalization":  # backward reads gamma now (src/functions.py:423)
            sh.inputs[1].d = np.asarray(node.inputs[1].data.values, dtype=np.float32)
            want[3:] = [False] * (len(want) - 3)  # running statistics carry no gradient
        return sh.backward(gys, want)

    return type(f"Device{base.__name__}", (base,), {
        "forward": forward, "backward": backward,
        "__doc__": f"{base.__name__} computed by libnnl (paper_2102_06725_b200.nanonnl_plugin)."})


def make_impls(functions_module=None) -> dict:
    """Device-backed operator classes keyed by KIND, subclassing the classes of
    `functions_module` (nanonnl.functions) or of this package when None."""
    if functions_module is None:
        from . import functions as functions_module
    return {k: _device_class(functions_module.REGISTRY[k]) for k in KINDS
            if k in functions_module.REGISTRY}


def install(functions_module) -> dict:
    """Register the device classes into `functions_module.REGISTRY` (nanonnl's
    lookup table, consulted by apply() at node creation); returns the entries
    they replaced, for uninstall()."""
    impls = make_impls(functions_module)
    saved = {k: functions_module.REGISTRY[k] for k in impls}
    functions_module.REGISTRY.update(impls)
    return saved


def uninstall(functions_module, saved: dict) -> None:
    functions_module.REGISTRY.update(saved)
