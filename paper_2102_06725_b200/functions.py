"""Function library: the operator boundary of the reference (src/functions.py).

Each kind keeps the reference's wire vocabulary (``KIND``/``ARGS``), its
eager shape inference and error behaviour, and its numeric contract; the
compute is a libnnl call on device buffers:

    forward(node, xs, ys)            writes the outputs ys (NdArrays)
    backward(node, gys, gxs, acc)    writes input grads; acc[i] -> accumulate

instead of the reference's "return numpy arrays and let the engine copy".
``Add2`` and ``GlobalAveragePooling`` are extensions needed by ResNet; their
CPU restatement lives in oracle/nnl_oracle.py.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import _lib
from .errors import (DegenerateBatch, DtypeMismatch, KernelTooLarge, LabelOutOfRange,
                     ShapeMismatch)
from .graph import ExecutionContext, Variable, apply
from .tensor import Dtype, NdArray

__all__ = [
    "REGISTRY", "supported_kinds", "affine", "convolution", "max_pooling", "relu",
    "softmax_cross_entropy", "batch_normalization", "add2", "global_average_pooling",
]


def _pair(value, name: str) -> tuple[int, int]:
    if isinstance(value, int):
        value = (value, value)
    value = tuple(int(v) for v in value)
    if len(value) != 2:
        raise ShapeMismatch(f"{name} must be an int or a pair, got {value!r}")
    return value


def _require(cond: bool, message: str) -> None:
    if not cond:
        raise ShapeMismatch(message)


def _flag(acc) -> int:
    return 1 if acc else 0


def _st() -> int:
    return _lib.stream()


def _state_buf(node, key: str, numel: int, dtype=None):
    """A per-node device scratch buffer, allocated once and reused."""
    t = _lib.torch()
    dtype = dtype or t.float32
    buf = node.state.get(key)
    if buf is None or buf.numel() < numel or buf.dtype != dtype:
        buf = t.empty(max(numel, 1), dtype=dtype, device=_lib.device())
        node.state[key] = buf
    return buf


class FunctionImpl:
    """Operator protocol (reference src/functions.py:54-79) on device buffers."""

    KIND: str = ""
    ARGS: dict[str, str] = {}

    def infer_shapes(self, in_shapes: list[tuple]) -> list[tuple]:
        raise NotImplementedError

    def output_dtype(self, ctx: ExecutionContext) -> Dtype:
        return ctx.storage_dtype

    # inputs that must be stored in float32 whatever the storage dtype
    F32_INPUTS: tuple = ()

    def check_dtypes(self, in_dtypes: list, out_dtype: Dtype) -> None:
        """Every kernel computes in one storage type taken from its first input:
        the other data operands and the output must share it (the reference
        computes on f32 values, so it never meets this; the device path refuses
        rather than misreading a buffer)."""
        for i, d in enumerate(in_dtypes):
            want = Dtype.F32 if i in self.F32_INPUTS else out_dtype
            if d is not want:
                raise DtypeMismatch(
                    f"{self.KIND} input {i} is {d.value}, expected {want.value} "
                    f"(output dtype {out_dtype.value}: build the graph and its inputs under "
                    f"one TypeConfig)")

    def forward(self, node, xs: list[NdArray], ys: list[NdArray]) -> None:
        raise NotImplementedError

    def backward(self, node, gys: list[NdArray], gxs: list, acc: list) -> None:
        raise NotImplementedError

    def backward_reads_input(self, index: int) -> bool:
        return True

    def can_fuse_relu(self, node) -> bool:
        return False

    def args_dict(self) -> dict:
        return {name: getattr(self, name) for name in self.ARGS}


def _same_dtype(xs) -> int:
    return xs[0].code


class Affine(FunctionImpl):
    """y = x.W + b, x flattened after the batch axis (reference :82-119)."""

    KIND = "Affine"
    ARGS = {"out_features": "int"}

    def __init__(self, out_features: int = 0):
        self.out_features = int(out_features)

    def infer_shapes(self, in_shapes):
        _require(len(in_shapes) == 3, f"Affine takes x, W, b; got {len(in_shapes)} inputs")
        xs, ws, bs = in_shapes
        _require(len(xs) >= 2, f"Affine input must have a batch axis, got {xs}")
        fan_in = int(np.prod(xs[1:], dtype=np.int64))
        _require(len(ws) == 2, f"Affine weight must be rank 2, got {ws}")
        _require(ws[0] == fan_in, f"Affine weight rows {ws[0]} != flattened input {fan_in}")
        if self.out_features == 0:
            self.out_features = ws[1]
        _require(ws[1] == self.out_features,
                 f"Affine weight cols {ws[1]} != out_features {self.out_features}")
        _require(bs == (self.out_features,), f"Affine bias shape {bs} != ({self.out_features},)")
        return [(xs[0], self.out_features)]

    @staticmethod
    def _dims(x: NdArray):
        b = x.shape[0]
        fan_in = int(np.prod(x.shape[1:], dtype=np.int64))
        in_c = x.shape[1] if len(x.shape) == 4 else fan_in
        return b, fan_in, in_c

    def forward(self, node, xs, ys):
        x, w, b = xs
        bsz, fi, in_c = self._dims(x)
        ws = _lib.workspace(_lib.lib().nnl_affine_workspace_size(x.code, bsz, fi, self.out_features, 0))
        _lib.call("nnl_affine_fwd", x.code, bsz, fi, in_c, self.out_features, x.ptr, w.ptr, b.ptr,
                  ys[0].ptr, ws[0], ws[1], _st())

    def backward(self, node, gys, gxs, acc):
        x, w, _ = (v.data for v in node.inputs)
        gy = gys[0]
        bsz, fi, in_c = self._dims(x)
        o = self.out_features
        if gxs[0] is not None:
            ws = _lib.workspace(_lib.lib().nnl_affine_workspace_size(x.code, bsz, fi, o, 1))
            _lib.call("nnl_affine_bwd_data", x.code, bsz, fi, in_c, o, gy.ptr, w.ptr,
                      gxs[0].ptr, _flag(acc[0]), ws[0], ws[1], _st())
        if gxs[1] is not None or gxs[2] is not None:
            ws = _lib.workspace(_lib.lib().nnl_affine_workspace_size(x.code, bsz, fi, o, 2))
            _lib.call("nnl_affine_bwd_weight", x.code, bsz, fi, in_c, o, x.ptr, gy.ptr,
                      gxs[1].ptr if gxs[1] is not None else None, _flag(acc[1]),
                      gxs[2].ptr if gxs[2] is not None else None, _flag(acc[2]),
                      node.state.get("nonfinite_ptr"), ws[0], ws[1], _st())

    def backward_reads_input(self, index):
        return index in (0, 1)


def _conv_out_extent(extent: int, k: int, s: int, p: int) -> int:
    if extent + 2 * p < k:
        raise KernelTooLarge(f"window {k} exceeds padded extent {extent + 2 * p}")
    return (extent + 2 * p - k) // s + 1


class Convolution(FunctionImpl):
    """2-D cross-correlation with per-map bias (reference :152-214)."""

    KIND = "Convolution"
    ARGS = {"out_maps": "int", "kernel": "pair", "stride": "pair", "pad": "pair"}

    def __init__(self, out_maps: int = 0, kernel=(1, 1), stride=(1, 1), pad=(0, 0)):
        self.out_maps = int(out_maps)
        self.kernel = _pair(kernel, "kernel")
        self.stride = _pair(stride, "stride")
        self.pad = _pair(pad, "pad")
        _require(min(self.kernel) >= 1, f"kernel extents must be >= 1, got {self.kernel}")
        _require(min(self.stride) >= 1, f"stride extents must be >= 1, got {self.stride}")
        _require(min(self.pad) >= 0, f"pads must be >= 0, got {self.pad}")

    def infer_shapes(self, in_shapes):
        _require(len(in_shapes) == 3, f"Convolution takes x, W, b; got {len(in_shapes)} inputs")
        xs, ws, bs = in_shapes
        _require(len(xs) == 4, f"Convolution input must be (B,C,H,W), got {xs}")
        kh, kw = self.kernel
        if self.out_maps == 0:
            self.out_maps = ws[0] if len(ws) == 4 else 0
        _require(ws == (self.out_maps, xs[1], kh, kw),
                 f"Convolution weight shape {ws} != ({self.out_maps},{xs[1]},{kh},{kw})")
        _require(bs == (self.out_maps,), f"Convolution bias shape {bs} != ({self.out_maps},)")
        oh = _conv_out_extent(xs[2], kh, self.stride[0], self.pad[0])
        ow = _conv_out_extent(xs[3], kw, self.stride[1], self.pad[1])
        return [(xs[0], self.out_maps, oh, ow)]

    def shape_struct(self, x_shape) -> _lib.ConvShape:
        b, c, h, w = x_shape
        kh, kw = self.kernel
        oh = _conv_out_extent(h, kh, self.stride[0], self.pad[0])
        ow = _conv_out_extent(w, kw, self.stride[1], self.pad[1])
        return _lib.ConvShape(b, h, w, c, self.out_maps, kh, kw, self.stride[0], self.stride[1],
                              self.pad[0], self.pad[1], oh, ow)

    def stat_rows(self, node) -> int:
        x = node.inputs[0].data
        cs = self.shape_struct(x.shape)
        return int(_lib.lib().nnl_conv2d_stat_rows(C.byref(cs), x.code))

    def epilogue_stats(self, node) -> bool:
        """Whether the following BatchNormalization's statistics come from this
        convolution's epilogue (default) or from BN's own streaming pass.
        Measured on the ResNet-50 step: epilogue statistics everywhere 20.34
        ms; a separate 2 B/elem pass for the expanding layers (cin*kh*kw <
        4*cout, whose epilogue sums cost the most in isolation) 20.78 ms.
        NNL_EPI_STATS=0 selects the streaming pass (probes)."""
        if os.environ.get("NNL_EPI_STATS", "") == "0":
            return False
        return self.stat_rows(node) > 0

    def _workspace(self, node, cs, code, pass_):
        """The shared workspace, or for narrow-channel inputs (the stem) the node's
        own, so that the weight gradient can reuse the space-to-depth copy of x
        its forward built there (nnl_conv2d_prep_reuse)."""
        if node.inputs[0].shape[1] > 4:
            return _lib.workspace(_lib.lib().nnl_conv2d_workspace_size(C.byref(cs), code, pass_))
        n = max(int(_lib.lib().nnl_conv2d_workspace_size(C.byref(cs), code, p)) for p in (0, 2))
        buf = _state_buf(node, "ws_own", (n + 3) // 4)
        return buf.data_ptr(), buf.numel() * 4

    def forward(self, node, xs, ys):
        x, w, b = xs
        cs = self.shape_struct(x.shape)
        stats = shift = None
        bn = node.state.get("stat_bn")
        if node.state.get("emit_stats"):
            rows = self.stat_rows(node)
            # the epilogue sums are centred on the BN's shift (its previous batch
            # mean); the BN's first forward takes its own centred pass instead
            if rows > 0 and bn is not None and bn.state.get("shift_ready"):
                stats = _state_buf(node, "stats", rows * 2 * self.out_maps)
                shift = bn.state["shift"]
                node.state["stat_rows"] = rows
            else:
                node.state.pop("emit_stats", None)
        ws = self._workspace(node, cs, x.code, 0)
        _lib.call("nnl_conv2d_fwd", C.byref(cs), x.code, x.ptr, w.ptr, b.ptr, ys[0].ptr,
                  stats.data_ptr() if stats is not None else None,
                  shift.data_ptr() if shift is not None else None, ws[0], ws[1], _st())

    def bnb_rows(self, node) -> int:
        """Partial rows of the dgrad with the preceding BN's backward statistics
        fused into its epilogue (0: not available for this shape)."""
        x = node.inputs[0].data
        if x.dtype is not Dtype.F16:
            return 0
        cs = self.shape_struct(x.shape)
        return int(_lib.lib().nnl_conv2d_bwd_data_bn_rows(C.byref(cs), x.code))

    def _dgrad_bn(self, node, cs, x, w, gy, gx, acc0, plan, ws):
        """dgrad + the statistics pass of the BN before this convolution
        (engine fusion, graph.py backward): writes the gated gradient to
        plan["out"] (or gx) and (gy, gy*xhat) column partials to the BN."""
        bn = plan["bn"]
        bx = bn.inputs[0].data
        c = bx.shape[1]
        rows = plan["rows"]
        parts = _state_buf(bn, "bwd_parts", rows * 2 * c)
        gate = plan.get("gate")
        out = plan.get("out")
        relu = plan["kind"] == "relu"
        bf = _lib.BnBwdFuse(bx.ptr, gate.ptr if gate is not None else None,
                            bn.inputs[1].data.ptr if relu else None,
                            bn.inputs[2].data.ptr if relu else None,
                            bn.state["mean"].data_ptr(), bn.state["istd"].data_ptr(),
                            1 if relu else 0, 0 if relu else 1,
                            out.ptr if out is not None else None, parts.data_ptr())
        _lib.call("nnl_conv2d_bwd_data_bn", C.byref(cs), x.code, gy.ptr, w.ptr, gx.ptr,
                  _flag(acc0), C.byref(bf), ws[0], ws[1], _st())
        bn.state["bwd_fused"] = {"parts": parts, "rows": rows,
                                 "gy": out if out is not None else gx}

    def backward(self, node, gys, gxs, acc):
        x, w = node.inputs[0].data, node.inputs[1].data
        gy = gys[0]
        cs = self.shape_struct(x.shape)
        if gxs[0] is not None:
            ws = _lib.workspace(_lib.lib().nnl_conv2d_workspace_size(C.byref(cs), x.code, 1))
            plan = node.state.pop("bnb", None)
            if plan is not None:
                self._dgrad_bn(node, cs, x, w, gy, gxs[0], acc[0], plan, ws)
            else:
                _lib.call("nnl_conv2d_bwd_data", C.byref(cs), x.code, gy.ptr, w.ptr, gxs[0].ptr,
                          _flag(acc[0]), ws[0], ws[1], _st())
        # the bias gradient was already reduced by the following BN's backward
        gb = None if node.state.get("bias_by_bn") else gxs[2]
        if gxs[1] is not None or gb is not None:
            own = x.shape[1] <= 4
            # inside the engine's backward loop the weight gradient runs on the
            # side stream: nothing later in backward reads dW, and its inputs
            # (x, dy) are final, so it overlaps the rest of the backward chain
            # (graph.backward joins before the optimizer)
            st = _lib.side_fork()
            if st is not None and not own:
                ws = _lib.side_workspace(
                    _lib.lib().nnl_conv2d_workspace_size(C.byref(cs), x.code, 2))
            else:
                ws = self._workspace(node, cs, x.code, 2)
            if st is None:
                st = _st()
            if own:
                _lib.lib().nnl_conv2d_prep_reuse(1)
            try:
                _lib.call("nnl_conv2d_bwd_weight", C.byref(cs), x.code, x.ptr, gy.ptr,
                          gxs[1].ptr if gxs[1] is not None else None, _flag(acc[1]),
                          gb.ptr if gb is not None else None, _flag(acc[2]),
                          node.state.get("nonfinite_ptr"), ws[0], ws[1], st)
            finally:
                if own:
                    _lib.lib().nnl_conv2d_prep_reuse(0)

    def backward_reads_input(self, index):
        return index in (0, 1)


class MaxPooling(FunctionImpl):
    """Window maximum; ties to the first element in row-major order (:217-291)."""

    KIND = "MaxPooling"
    ARGS = {"kernel": "pair", "stride": "pair", "ignore_border": "bool", "pad": "pair"}

    def __init__(self, kernel=(1, 1), stride=None, ignore_border: bool = True, pad=(0, 0)):
        self.kernel = _pair(kernel, "kernel")
        self.stride = self.kernel if stride is None else _pair(stride, "stride")
        self.ignore_border = bool(ignore_border)
        self.pad = _pair(pad, "pad")
        _require(min(self.kernel) >= 1, f"kernel extents must be >= 1, got {self.kernel}")
        _require(min(self.stride) >= 1, f"stride extents must be >= 1, got {self.stride}")
        _require(min(self.pad) >= 0, f"pads must be >= 0, got {self.pad}")

    def _out_extent(self, extent: int, k: int, s: int, p: int) -> int:
        if extent + 2 * p < k:
            raise KernelTooLarge(f"window {k} exceeds padded extent {extent + 2 * p}")
        if self.ignore_border:
            return (extent + 2 * p - k) // s + 1
        return -((extent + 2 * p - k) // -s) + 1

    def infer_shapes(self, in_shapes):
        _require(len(in_shapes) == 1, "MaxPooling takes one input")
        xs = in_shapes[0]
        _require(len(xs) == 4, f"MaxPooling input must be (B,C,H,W), got {xs}")
        oh = self._out_extent(xs[2], self.kernel[0], self.stride[0], self.pad[0])
        ow = self._out_extent(xs[3], self.kernel[1], self.stride[1], self.pad[1])
        return [(xs[0], xs[1], oh, ow)]

    def _ps(self, x_shape):
        b, c, h, w = x_shape
        oh, ow = self.infer_shapes([x_shape])[0][2:]
        return _lib.PoolShape(b, h, w, c, self.kernel[0], self.kernel[1], self.stride[0],
                              self.stride[1], self.pad[0], self.pad[1], oh, ow)

    def forward(self, node, xs, ys):
        x = xs[0]
        ps = self._ps(x.shape)
        t = _lib.torch()
        arg = _state_buf(node, "argmax", ys[0].size, t.uint8)
        _lib.call("nnl_maxpool_fwd", x.code, C.byref(ps), x.ptr, ys[0].ptr, arg.data_ptr(), _st())

    def backward(self, node, gys, gxs, acc):
        if gxs[0] is None:
            return
        x = node.inputs[0].data
        ps = self._ps(x.shape)
        _lib.call("nnl_maxpool_bwd", x.code, C.byref(ps), gys[0].ptr,
                  node.state["argmax"].data_ptr(), gxs[0].ptr, _flag(acc[0]), _st())

    def backward_reads_input(self, index):
        return False


class ReLU(FunctionImpl):
    """max(x, 0); the gradient gate is closed at 0 (:294-317)."""

    KIND = "ReLU"
    ARGS = {"inplace": "bool"}

    def __init__(self, inplace: bool = False):
        self.inplace = bool(inplace)

    def infer_shapes(self, in_shapes):
        _require(len(in_shapes) == 1, "ReLU takes one input")
        return [in_shapes[0]]

    def forward(self, node, xs, ys):
        _lib.call("nnl_relu_fwd", xs[0].code, xs[0].size, xs[0].ptr, ys[0].ptr, _st())

    def backward(self, node, gys, gxs, acc):
        if gxs[0] is None:
            return
        x = node.inputs[0].data
        _lib.call("nnl_relu_bwd", x.code, x.size, x.ptr, gys[0].ptr, gxs[0].ptr, _flag(acc[0]),
                  _st())


class SoftmaxCrossEntropy(FunctionImpl):
    """Batch-mean of -log softmax(logits)[label] (:320-360); rank-0 output."""

    KIND = "SoftmaxCrossEntropy"
    ARGS = {}

    def infer_shapes(self, in_shapes):
        _require(len(in_shapes) == 2, "SoftmaxCrossEntropy takes logits and labels")
        ls, ts = in_shapes
        _require(len(ls) == 2, f"logits must be (B,K), got {ls}")
        _require(ts == (ls[0],), f"labels must be ({ls[0]},), got {ts}")
        return [()]

    def on_input_written(self, node, v, values):
        """Validate host-written labels (the reference checks in forward, :337-339)."""
        if node.inputs[1] is not v:
            return
        k = node.inputs[0].shape[1]
        lab = np.broadcast_to(np.asarray(values, dtype=np.float32), v.shape)
        ids = lab.astype(np.int64)
        ok = bool(np.array_equal(ids, lab) and ids.min(initial=0) >= 0
                  and ids.max(initial=0) < k)
        node.state["labels_ok"] = ok

    def forward(self, node, xs, ys):
        logits, labels = xs
        b, k = logits.shape
        ok = node.state.get("labels_ok")
        if ok is False:
            raise LabelOutOfRange(f"labels must be integers in [0, {k})")
        t = _lib.torch()
        stats = _state_buf(node, "rows", 3 * b)
        err = None
        if ok is None:  # labels produced on the device: check there, then sync
            err = _state_buf(node, "label_err", 1, t.int32)
            err.zero_()
        _lib.call("nnl_sce_fwd", logits.code, b, k, logits.ptr, labels.ptr, ys[0].ptr,
                  stats.data_ptr(), err.data_ptr() if err is not None else None, _st())
        if err is not None and int(err.item()):
            raise LabelOutOfRange(f"labels must be integers in [0, {k})")

    def backward(self, node, gys, gxs, acc):
        if gxs[0] is None:
            return
        logits, labels = node.inputs[0].data, node.inputs[1].data
        b, k = logits.shape
        _lib.call("nnl_sce_bwd", logits.code, b, k, logits.ptr, labels.ptr,
                  node.state["rows"].data_ptr(), gys[0].ptr, gxs[0].ptr, _flag(acc[0]), _st())

    def backward_reads_input(self, index):
        return index == 0


class BatchNormalization(FunctionImpl):
    """Per-channel normalisation, f32 statistics and math (:363-441)."""

    KIND = "BatchNormalization"
    ARGS = {"eps": "float", "momentum": "float", "batch_stat": "bool"}
    F32_INPUTS = (1, 2, 3, 4)  # gamma, beta, mean, var (reference parametric.py:67-70)

    def __init__(self, eps: float = 1e-5, momentum: float = 0.9, batch_stat: bool = True):
        self.eps = float(eps)
        self.momentum = float(momentum)
        self.batch_stat = bool(batch_stat)

    def infer_shapes(self, in_shapes):
        _require(len(in_shapes) == 5, "BatchNormalization takes x, gamma, beta, mean, var")
        xs = in_shapes[0]
        _require(len(xs) >= 2, f"input must have batch and channel axes, got {xs}")
        _require(len(xs) in (2, 4), f"device BatchNormalization supports rank 2 or 4, got {xs}")
        c = xs[1]
        for name, s in zip(("gamma", "beta", "mean", "var"), in_shapes[1:]):
            _require(s == (c,), f"{name} shape {s} != ({c},)")
        if self.batch_stat:
            n = int(np.prod(xs, dtype=np.int64)) // c
            if n <= 1:
                raise DegenerateBatch(f"cannot take batch statistics over {n} element(s)")
        return [xs]

    @staticmethod
    def _rows(x: NdArray) -> int:
        return x.size // x.shape[1]

    def can_fuse_relu(self, node) -> bool:
        return True

    def _forward(self, node, y: NdArray, relu: bool, residual: NdArray | None = None):
        x, gamma, beta, mean, var = (v.data for v in node.inputs)
        c = x.shape[1]
        rows = self._rows(x)
        sm = _state_buf(node, "mean", c)
        si = _state_buf(node, "istd", c)
        if self.batch_stat:
            parts, nparts = None, 0
            prod = node.inputs[0].parent
            if prod is not None and prod.state.get("emit_stats") and "stats" in prod.state:
                parts, nparts = prod.state["stats"].data_ptr(), prod.state["stat_rows"]
            ws = _lib.workspace(_lib.lib().nnl_bn_workspace_size(rows, c))
            # per-channel centre of the statistics: in/out, the batch mean of
            # this call becomes the centre of the next (and of the producing
            # convolution's epilogue sums)
            shift = _state_buf(node, "shift", c)
            _lib.call("nnl_bn_fwd_train", x.code, rows, c, x.ptr, gamma.ptr, beta.ptr, mean.ptr,
                      var.ptr, float(np.float32(self.eps)), float(np.float32(self.momentum)),
                      parts, nparts, shift.data_ptr(), sm.data_ptr(), si.data_ptr(),
                      y.ptr if y is not None else None,
                      residual.ptr if residual is not None else None, 1 if relu else 0,
                      ws[0], ws[1], _st())
            node.state["shift_ready"] = True
        else:
            _lib.call("nnl_bn_fwd_eval", x.code, rows, c, x.ptr, gamma.ptr, beta.ptr, mean.ptr,
                      var.ptr, float(np.float32(self.eps)), sm.data_ptr(), si.data_ptr(), y.ptr,
                      residual.ptr if residual is not None else None, 1 if relu else 0, _st())

    def forward(self, node, xs, ys):
        self._forward(node, ys[0], relu=False)

    def forward_fused(self, node, relu_node, stats):
        # backward recomputes the ReLU gate from x, so the output may be released
        self._forward(node, relu_node.outputs[0].data, relu=True)

    def can_fuse_relu_pool(self, node, pool_node) -> bool:
        """BN -> ReLU -> MaxPooling as one pass (nnl_bn_relu_maxpool_fwd): batch
        statistics, fp16, and a 3x3 / stride-2 pool the fused kernel covers."""
        try:
            x = node.inputs[0].data
            ps = pool_node.impl._ps(x.shape)
            return bool(self.batch_stat and node.inputs[0].data.code == _lib.F16
                        and node.inputs[2].data.code == _lib.F32
                        and _lib.lib().nnl_bn_relu_maxpool_ok(x.code, C.byref(ps)))
        except Exception:
            return False

    def forward_fused_pool(self, node, relu_node, pool_node):
        # statistics (finalize) only, then BN-apply + ReLU + pool in one pass:
        # relu(BN(x)) is never written; the pool's backward uses its argmax and
        # BN's backward recomputes the ReLU gate from x
        self._forward(node, None, relu=True)
        x, gamma, beta = (v.data for v in node.inputs[:3])
        ps = pool_node.impl._ps(x.shape)
        y = pool_node.outputs[0].data
        arg = _state_buf(pool_node, "argmax", y.size, _lib.torch().uint8)
        _lib.call("nnl_bn_relu_maxpool_fwd", x.code, C.byref(ps), x.ptr, gamma.ptr, beta.ptr,
                  node.state["mean"].data_ptr(), node.state["istd"].data_ptr(), y.ptr,
                  arg.data_ptr(), _st())

    def _backward(self, node, gy: NdArray, fused_relu: bool, gxs, acc, gate=None, dres=None,
                  acc_res=False):
        x = node.inputs[0].data
        gamma = node.inputs[1].data
        beta = node.inputs[2].data
        c = x.shape[1]
        rows = self._rows(x)
        ws = _lib.workspace(_lib.lib().nnl_bn_workspace_size(rows, c))
        conv = node.inputs[0].parent
        cbias = None
        if gxs[0] is not None and conv is not None and conv.state.get("bias_by_bn"):
            cbias = conv.inputs[2].grad.ptr  # sole consumer: first contribution overwrites
        _lib.call("nnl_bn_bwd", x.code, rows, c, x.ptr, gy.ptr, 1 if fused_relu else 0,
                  gate.ptr if gate is not None else None,
                  dres.ptr if dres is not None else None, _flag(acc_res),
                  gamma.ptr, beta.ptr,
                  node.state["mean"].data_ptr(), node.state["istd"].data_ptr(),
                  1 if self.batch_stat else 0,
                  gxs[0].ptr if gxs[0] is not None else None, _flag(acc[0]),
                  gxs[1].ptr if gxs[1] is not None else None, _flag(acc[1]),
                  gxs[2].ptr if gxs[2] is not None else None, _flag(acc[2]),
                  cbias, 0, node.state.get("nonfinite_ptr"), ws[0], ws[1], _st())

    def _backward_apply(self, node, fz, gxs, acc):
        """Backward whose statistics pass ran in the next convolution's dgrad
        epilogue (Convolution._dgrad_bn): finalize + apply only."""
        x = node.inputs[0].data
        gamma = node.inputs[1].data
        c = x.shape[1]
        rows = self._rows(x)
        ws = _lib.workspace(_lib.lib().nnl_bn_workspace_size(rows, c))
        conv = node.inputs[0].parent
        cbias = None
        if gxs[0] is not None and conv is not None and conv.state.get("bias_by_bn"):
            cbias = conv.inputs[2].grad.ptr
        _lib.call("nnl_bn_bwd_apply", x.code, rows, c, x.ptr, fz["gy"].ptr,
                  fz["parts"].data_ptr(), fz["rows"], gamma.ptr,
                  node.state["mean"].data_ptr(), node.state["istd"].data_ptr(),
                  1 if self.batch_stat else 0,
                  gxs[0].ptr if gxs[0] is not None else None, _flag(acc[0]),
                  gxs[1].ptr if gxs[1] is not None else None, _flag(acc[1]),
                  gxs[2].ptr if gxs[2] is not None else None, _flag(acc[2]),
                  cbias, 0, node.state.get("nonfinite_ptr"), ws[0], ws[1], _st())

    def backward(self, node, gys, gxs, acc):
        self._backward(node, gys[0], False, gxs, acc)

    def backward_fused(self, node, relu_node, gxs, acc):
        fz = node.state.pop("bwd_fused", None)
        if fz is not None:
            self._backward_apply(node, fz, gxs, acc)
            return
        self._backward(node, relu_node.outputs[0].grad, True, gxs, acc)

    # residual tail BN -> Add2 -> ReLU (engine fusion, graph.py::_plan): the
    # BN output and the Add2 output are never materialised
    def forward_residual(self, node, residual: NdArray, relu_node):
        relu_node.state["keep_output"] = True  # the backward gate
        self._forward(node, relu_node.outputs[0].data, relu=True, residual=residual)

    def backward_residual(self, node, relu_node, gxs, acc, dres, acc_res):
        fz = node.state.pop("bwd_fused", None)
        if fz is not None:  # the gated gradient (= dres) and statistics are done
            self._backward_apply(node, fz, gxs, acc)
            return
        z = relu_node.outputs[0]
        self._backward(node, z.grad, False, gxs, acc, gate=z.data, dres=dres, acc_res=acc_res)

    def backward_reads_input(self, index):
        return index in (0, 1)


class Add2(FunctionImpl):
    """Extension: y = x0 + x1 (residual connection); restated in oracle/."""

    KIND = "Add2"
    ARGS = {}

    def infer_shapes(self, in_shapes):
        _require(len(in_shapes) == 2, "Add2 takes two inputs")
        _require(in_shapes[0] == in_shapes[1], f"Add2 shapes differ: {in_shapes}")
        return [in_shapes[0]]

    def can_fuse_relu(self, node) -> bool:
        return True

    def forward(self, node, xs, ys):
        a, b = xs
        _lib.call("nnl_add2_fwd", a.code, a.size, a.ptr, b.ptr, ys[0].ptr, 0, _st())

    def forward_fused(self, node, relu_node, stats):
        relu_node.state["keep_output"] = True
        a, b = (v.data for v in node.inputs)
        y = relu_node.outputs[0].data
        _lib.call("nnl_add2_fwd", a.code, a.size, a.ptr, b.ptr, y.ptr, 1, _st())

    def backward(self, node, gys, gxs, acc):
        gy = gys[0]
        for i in range(2):
            if gxs[i] is not None:
                _lib.call("nnl_accumulate", gy.code, gy.size, gy.ptr, gxs[i].ptr, _flag(acc[i]),
                          _st())

    def backward_fused(self, node, relu_node, gxs, acc):
        z = relu_node.outputs[0]
        for i in range(2):
            if gxs[i] is not None:
                _lib.call("nnl_relu_bwd", z.data.code, z.data.size, z.data.ptr, z.grad.ptr,
                          gxs[i].ptr, _flag(acc[i]), _st())

    def backward_reads_input(self, index):
        return False


class GlobalAveragePooling(FunctionImpl):
    """Extension: (B,C,H,W) -> (B,C,1,1) spatial mean; restated in oracle/."""

    KIND = "GlobalAveragePooling"
    ARGS = {}

    def infer_shapes(self, in_shapes):
        _require(len(in_shapes) == 1, "GlobalAveragePooling takes one input")
        xs = in_shapes[0]
        _require(len(xs) == 4, f"GlobalAveragePooling input must be (B,C,H,W), got {xs}")
        return [(xs[0], xs[1], 1, 1)]

    def forward(self, node, xs, ys):
        x = xs[0]
        b, c, h, w = x.shape
        _lib.call("nnl_gap_fwd", x.code, b, h * w, c, x.ptr, ys[0].ptr, _st())

    def backward(self, node, gys, gxs, acc):
        if gxs[0] is None:
            return
        b, c, h, w = node.inputs[0].shape
        _lib.call("nnl_gap_bwd", gys[0].code, b, h * w, c, gys[0].ptr, gxs[0].ptr,
                  _flag(acc[0]), _st())

    def backward_reads_input(self, index):
        return False


REGISTRY: dict[str, type[FunctionImpl]] = {
    cls.KIND: cls
    for cls in (Affine, Convolution, MaxPooling, ReLU, SoftmaxCrossEntropy, BatchNormalization,
                Add2, GlobalAveragePooling)
}

REFERENCE_KINDS = ("Affine", "Convolution", "MaxPooling", "ReLU", "SoftmaxCrossEntropy",
                   "BatchNormalization")


def supported_kinds() -> set[str]:
    return set(REGISTRY)


# --- graph-building wrappers (reference :457-486) ---------------------------

def affine(x: Variable, weight: Variable, bias: Variable) -> Variable:
    return apply("Affine", [x, weight, bias], {"out_features": weight.shape[1]})[0]


def convolution(x: Variable, weight: Variable, bias: Variable, stride=(1, 1),
                pad=(0, 0)) -> Variable:
    args = {"out_maps": weight.shape[0], "kernel": weight.shape[2:4], "stride": stride,
            "pad": pad}
    return apply("Convolution", [x, weight, bias], args)[0]


def max_pooling(x: Variable, kernel, stride=None, ignore_border: bool = True,
                pad=(0, 0)) -> Variable:
    args = {"kernel": kernel, "stride": stride, "ignore_border": ignore_border, "pad": pad}
    return apply("MaxPooling", [x], args)[0]


def relu(x: Variable, inplace: bool = False) -> Variable:
    return apply("ReLU", [x], {"inplace": inplace})[0]


def softmax_cross_entropy(logits: Variable, labels: Variable) -> Variable:
    return apply("SoftmaxCrossEntropy", [logits, labels])[0]


def batch_normalization(x: Variable, gamma: Variable, beta: Variable, mean: Variable,
                        var: Variable, batch_stat: bool = True, eps: float = 1e-5,
                        momentum: float = 0.9) -> Variable:
    args = {"eps": eps, "momentum": momentum, "batch_stat": batch_stat}
    return apply("BatchNormalization", [x, gamma, beta, mean, var], args)[0]


def add2(x0: Variable, x1: Variable) -> Variable:
    return apply("Add2", [x0, x1])[0]


def global_average_pooling(x: Variable) -> Variable:
    return apply("GlobalAveragePooling", [x])[0]
