"""The engine's concurrency is invisible in the numbers: weight gradients on the
side stream (NNL_WG_STREAM) and projection shortcuts on the branch stream
(NNL_BRANCH) must give bit-identical training to the single-stream engine --
every kernel is deterministic and each accumulation keeps its program order,
so only a missing dependency (a race) could make them differ.  Checked on
ResNet-50 (every fusion and both kinds of branch) over two eager steps and a
CUDA-graph replay."""

import numpy as np
import pytest

from oracle import nnl_oracle as O

pytestmark = pytest.mark.gpu


def _run(nnl, monkeypatch, streams: bool):
    import paper_2102_06725_b200.functions as F
    from paper_2102_06725_b200 import networks
    from paper_2102_06725_b200.communicator import DataParallelTrainer
    v = "1" if streams else "0"
    monkeypatch.setenv("NNL_WG_STREAM", v)
    monkeypatch.setenv("NNL_BRANCH", v)
    nnl.set_default_context(nnl.ExecutionContext(type_config=nnl.TypeConfig.HALF))
    B, hw = 4, 96
    shape = (B, 3, hw, hw)

    def build(bs):
        xv = nnl.Variable((bs, 3, hw, hw))
        tv = nnl.Variable((bs,))
        return {"x": xv, "label": tv,
                "loss": F.softmax_cross_entropy(networks.resnet50(xv, 100), tv)}

    with nnl.registry_scope(nnl.ParameterRegistry(seed=0)):
        tr = DataParallelTrainer(1, B, build, lr=0.1, seed=0, momentum=0.9, weight_decay=1e-4,
                                 loss_scaling=nnl.DynamicLossScaler(8.0, 2.0, 2000))
        losses = []
        for k in range(2):
            x = O.uniform(1, k * int(np.prod(shape)), shape, 0.0, 1.0)
            losses.append(tr.step(x, (np.arange(B) * (k + 3) % 100).astype(np.float32)))
        tr.capture_graph()  # its warm-up is a third (eager, captured-stream) step
        tr.step_resident()
        rep = tr.rank0
        w = {k: p.d.copy() for k, p in rep.registry.get_parameters(grad_only=False).items()}
        g = {k: p.g.copy() for k, p in rep.registry.get_parameters().items()}
    return losses, w, g


def test_streams_are_bit_identical_to_one_stream(nnl, monkeypatch):
    l1, w1, g1 = _run(nnl, monkeypatch, True)
    l0, w0, g0 = _run(nnl, monkeypatch, False)
    assert l1 == l0
    assert sorted(w1) == sorted(w0)
    for k in w0:
        assert np.array_equal(w1[k].view(np.uint32), w0[k].view(np.uint32)), k
    for k in g0:
        assert np.array_equal(g1[k].view(np.uint32), g0[k].view(np.uint32)), k
