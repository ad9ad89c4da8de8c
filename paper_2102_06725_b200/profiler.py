"""CUDA-event timing of individual graph nodes (the build's tracing hook).

When enabled, the engine brackets every node's forward / backward launch
sequence with CUDA events on the current stream; ``summary()`` then gives
per-kind device time, and ``gemm_flops`` the algorithmic FLOPs of each
Convolution / Affine call (2*M*N*K per GEMM pass) for roofline fractions.
"""

from __future__ import annotations

import contextlib
from collections import defaultdict

from . import _lib


class _Profiler:
    def __init__(self):
        self.enabled = False
        self.gpu_lead_cycles = 0  # > 0: spin the GPU this long before each region
        self.records = []  # (kind, phase, flops, start_event, end_event, description)
        self.nodes = []    # (node, phase) of each record

    def reset(self):
        self.records = []
        self.nodes = []

    def gemm_bound_ms(self, tflops: float, hbm_gbs: float) -> float:
        """Sum of the per-pass roofline bounds of the recorded GEMM nodes."""
        return 1e3 * sum(gemm_bound_s(nd, ph, tflops, hbm_gbs) for nd, ph in self.nodes)

    @contextlib.contextmanager
    def region(self, node, phase: str):
        if not self.enabled:
            yield
            return
        t = _lib.torch()
        s = t.cuda.Event(enable_timing=True)
        e = t.cuda.Event(enable_timing=True)
        if self.gpu_lead_cycles:
            # keep the GPU busy while the host enqueues this node, so the events
            # time the node's kernels, not the host's launch latency
            t.cuda._sleep(self.gpu_lead_cycles)
        s.record()
        yield
        e.record()
        self.records.append((node.kind, phase, gemm_flops(node, phase), s, e, _describe(node)))
        self.nodes.append((node, phase))

    def per_node(self) -> list[dict]:
        """One entry per recorded node call, in launch order."""
        _lib.torch().cuda.synchronize()
        return [{"kind": k, "phase": ph, "shape": desc, "ms": s.elapsed_time(e), "flops": fl}
                for k, ph, fl, s, e, desc in self.records]

    def summary(self) -> dict:
        _lib.torch().cuda.synchronize()
        out = defaultdict(lambda: {"ms": 0.0, "flops": 0.0, "calls": 0})
        for kind, phase, flops, s, e, _ in self.records:
            d = out[f"{kind}.{phase}"]
            d["ms"] += s.elapsed_time(e)
            d["flops"] += flops
            d["calls"] += 1
        return dict(out)


PROFILER = _Profiler()


def _describe(node) -> str:
    ins = "x".join(str(d) for d in node.inputs[0].shape)
    if node.kind == "Convolution":
        o, c, kh, kw = node.inputs[1].shape
        s = node.impl.stride[0]
        return f"{ins} -> {o} k{kh} s{s}"
    return ins


def gemm_bound_s(node, phase: str, tflops: float, hbm_gbs: float) -> float:
    """Per-pass roofline bound of a node's implicit GEMMs: for each GEMM the
    node runs in `phase`, max(FLOPs / tensor peak, bytes / HBM) with every
    operand and the output moved once in the storage dtype (the per-layer
    bound of tools/conv_bench.py)."""
    if node.kind not in ("Convolution", "Affine"):
        return 0.0
    es = 2 if node.outputs[0].dtype.value == "f16" else 4

    def n(shape):
        k = 1
        for d in shape:
            k *= d
        return k
    x, w, y = n(node.inputs[0].shape), n(node.inputs[1].shape), n(node.outputs[0].shape)
    one = gemm_flops(node, "fwd")

    def bound(bytes_):
        return max(one / (tflops * 1e12), es * bytes_ / (hbm_gbs * 1e9))
    if phase == "fwd":
        return bound(x + w + y)
    t = 0.0
    if node.inputs[0].need_grad:
        t += bound(y + w + x)   # dgrad: dy, W -> dx
    if node.inputs[1].need_grad:
        t += bound(x + y + w)   # wgrad: x, dy -> dW
    return t


def gemm_flops(node, phase: str) -> float:
    """Algorithmic FLOPs of the implicit GEMMs a node runs in `phase`."""
    if node.kind == "Convolution":
        x = node.inputs[0].shape
        y = node.outputs[0].shape
        o, c, kh, kw = node.inputs[1].shape
        one = 2.0 * y[0] * y[2] * y[3] * o * c * kh * kw
        if phase == "fwd":
            return one
        n = 0
        if node.inputs[0].need_grad:
            n += 1
        if node.inputs[1].need_grad:
            n += 1
        return one * n
    if node.kind == "Affine":
        b = node.inputs[0].shape[0]
        i, o = node.inputs[1].shape
        one = 2.0 * b * i * o
        if phase == "fwd":
            return one
        return one * (int(node.inputs[0].need_grad) + int(node.inputs[1].need_grad))
    return 0.0
