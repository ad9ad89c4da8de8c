"""Checkpoint format (the reference's NNP parameter.bin records) and resume."""

import numpy as np
import pytest

from paper_2102_06725_b200 import checkpoint as ck


def _golden_records(golden):
    g = golden("nnp")
    recs = []
    for i, name in enumerate(g["names"]):
        v = g[f"v{i}"]
        recs.append(ck.Record(str(name), tuple(v.shape), bool(g["f16"][i]), v,
                              bool(g["need_grad"][i])))
    return g, recs


def test_encode_matches_reference_parameter_bin(golden):
    """Byte-identical to nanonnl.nnp.emit_parameter_bin on the same records."""
    g, recs = _golden_records(golden)
    assert ck.encode(recs) == g["bin"].tobytes()


def test_decode_reference_parameter_bin(golden):
    g, recs = _golden_records(golden)
    back = ck.decode(g["bin"].tobytes())
    assert [r.name for r in back] == [r.name for r in recs]
    for a, b in zip(back, recs):
        assert a.shape == b.shape and a.f16 == b.f16 and a.need_grad == b.need_grad
        assert np.array_equal(a.values, np.asarray(b.values, np.float32))


def test_decode_rejects_damage(golden):
    g, _ = _golden_records(golden)
    raw = g["bin"].tobytes()
    with pytest.raises(ValueError):
        ck.decode(raw[:-3])
    with pytest.raises(ValueError):
        ck.decode(raw + b"\0")
    with pytest.raises(ValueError):
        ck.decode(b"XXXX" + raw[4:])


@pytest.mark.gpu
def test_resume_continues_bit_identically(nnl, golden, tmp_path):
    """save after 2 steps, 2 more steps; a fresh trainer loading the file and
    taking the same 2 steps ends bit-identical (weights, masters, momentum,
    device loss scaler)."""
    import paper_2102_06725_b200.functions as F
    from paper_2102_06725_b200 import networks
    from paper_2102_06725_b200.communicator import DataParallelTrainer
    g = golden("lenet")
    nnl.set_default_context(nnl.ExecutionContext(type_config=nnl.TypeConfig.HALF))

    def build(bs):
        xv = nnl.Variable((bs, 1, 28, 28))
        tv = nnl.Variable((bs,))
        return {"x": xv, "label": tv,
                "loss": F.softmax_cross_entropy(networks.lenet(xv, 10), tv)}

    def trainer(seed):
        return DataParallelTrainer(1, 16, build, lr=0.05, seed=seed, momentum=0.9,
                                   weight_decay=1e-4,
                                   loss_scaling=nnl.DynamicLossScaler(8.0, 2.0, 1))

    a = trainer(0)
    for i in range(2):
        a.step(g["lenet_x"][i], g["lenet_labels"])
    path = str(tmp_path / "ck.bin")
    a.save_checkpoint(path)
    la = [a.step(g["lenet_x"][i], g["lenet_labels"]) for i in (2, 0)]
    b = trainer(7)  # different init: everything must come from the file
    b.load_checkpoint(path)
    lb = [b.step(g["lenet_x"][i], g["lenet_labels"]) for i in (2, 0)]
    assert la == lb
    pa, pb = a.rank0.registry.get_parameters(), b.rank0.registry.get_parameters()
    for k in pa:
        assert np.array_equal(pa[k].d, pb[k].d), k
        assert np.array_equal(a.rank0.solver.master_values(k), b.rank0.solver.master_values(k))
