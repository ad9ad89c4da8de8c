import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")
REFERENCE_SRC = "/root/reference/pkg/src"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libnnl.so")
    config.addinivalue_line("markers", "reference: needs /root/reference (build container only)")


def _cuda_ok() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:  # noqa: BLE001
        return False


def pytest_collection_modifyitems(config, items):
    cuda = _cuda_ok()
    ref = os.path.isdir(REFERENCE_SRC)
    for item in items:
        if "gpu" in item.keywords and not cuda:
            item.add_marker(pytest.mark.skip(reason="no CUDA device"))
        if "reference" in item.keywords and not ref:
            item.add_marker(pytest.mark.skip(reason="/root/reference not present"))


@pytest.fixture
def golden():
    import numpy as np

    cache = {}

    def load(name):
        if name not in cache:
            cache[name] = dict(np.load(os.path.join(GOLDEN, f"{name}.npz")))
        return cache[name]

    return load


@pytest.fixture
def nnl():
    """The B200 package with a fresh default context and registry (gpu tests)."""
    import paper_2102_06725_b200 as nn

    nn.set_default_context(nn.ExecutionContext())
    with nn.registry_scope(nn.ParameterRegistry(seed=0)):
        yield nn
    nn.set_default_context(nn.ExecutionContext())


@pytest.fixture
def reference():
    """The real reference package (build container only)."""
    if REFERENCE_SRC not in sys.path:
        sys.path.insert(0, REFERENCE_SRC)
    import nanonnl
    return nanonnl
