"""CPU restatement of the reference hot path — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
arm may import this module, and only as the checker / the CPU baseline.  The
product package (paper_2102_06725_b200) never imports it.

It re-derives, in plain numpy, the algorithms of the reference package
``nanonnl`` (/root/reference/pkg/src/nanonnl) that the B200 path replaces,
citing the reference line each piece follows.  It is pinned against the
reference itself (tests/test_oracle_pin.py, run in the build container where
/root/reference exists) and against golden vectors generated from the
reference (tests/golden/, script tests/golden/make_golden.py).

Extensions with no reference implementation (parity unpinned by reference
tests; defined here and matched by the CUDA kernels):
  * Add2: y = q(x0 + x1) (f32 add);  bwd: both inputs receive gy.
  * GlobalAveragePooling: y[b,c] = q(sum_hw x / f32(H*W)), sum in f32 in
    raster order;  bwd: gx = q(gy / f32(H*W)) broadcast.
  * Momentum SGD with weight decay (NNabla Momentum solver):
        d = g + wd*master ; v = m*v + lr*d ; master = master - v
    which for m = wd = 0 is the reference update master -= lr*g.

Layout: every array here is the reference's logical layout (NCHW, affine W
as (I,O), conv W as (O,C,kh,kw)).
"""

from __future__ import annotations

import itertools
import math
from dataclasses import dataclass, field

import numpy as np

F32 = np.float32

# ---------------------------------------------------------------------------
# numerics: binary16 storage rounding (tensor.py:46-50) and SplitMix64 (:211-252)


def q16(a) -> np.ndarray:
    """Round float32 values to binary16 (RNE, overflow -> inf), kept in float32."""
    with np.errstate(over="ignore", invalid="ignore"):
        return np.asarray(a, dtype=F32).astype(np.float16).astype(F32)


def store(a, half: bool) -> np.ndarray:
    a = np.asarray(a, dtype=F32)
    return q16(a) if half else a.copy()


_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def splitmix64(x: np.ndarray) -> np.ndarray:
    """tensor.py:217-222 (uint64 wrap-around arithmetic)."""
    with np.errstate(over="ignore"):
        z = x + np.uint64(0x9E3779B97F4B7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def uniform(seed: int, counter: int, shape, low: float, high: float) -> np.ndarray:
    """Draws counter..counter+n-1 of stream `seed` in [low, high) (tensor.py:241-252)."""
    n = int(np.prod(shape, dtype=np.int64))
    idx = np.arange(counter, counter + n, dtype=np.uint64)
    with np.errstate(over="ignore"):
        bits = splitmix64(np.uint64(seed) * np.uint64(0xBF58476D1CE4E5B9) + idx)
    u = (bits >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)
    return (low + (high - low) * u).astype(F32).reshape(shape)


class Stream:
    """Counter-based stream (seed, counter) (tensor.py:225-239)."""

    def __init__(self, seed: int):
        self.seed = int(seed)
        self.counter = 0

    def draw(self, shape, low=0.0, high=1.0) -> np.ndarray:
        out = uniform(self.seed, self.counter, shape, low, high)
        self.counter += out.size
        return out


# ---------------------------------------------------------------------------
# tape-based autodiff with the reference engine's rules (graph.py:192-367)

_order = itertools.count()


class Var:
    def __init__(self, value=None, shape=None, half=False, need_grad=False, name=None):
        self.half = half
        self.shape = tuple(shape if shape is not None else np.shape(value))
        self.value = None if value is None else store(value, half)
        self.grad = np.zeros(self.shape, dtype=F32)
        self.need_grad = need_grad
        self.parent: Node | None = None
        self.name = name
        self.consumers: list[Node] = []

    def set(self, value):
        self.value = store(np.broadcast_to(np.asarray(value, dtype=F32), self.shape), self.half)


@dataclass
class Node:
    kind: str
    inputs: list
    outputs: list
    bwd: object  # callable(gys, want) -> list of grads or None
    seq: int = field(default_factory=lambda: next(_order))


class Ctx:
    half: bool = False


def _emit(kind, inputs, results, bwd, half) -> list[Var]:
    need = any(v.need_grad for v in inputs)
    outs = [Var(r, half=half, need_grad=need) for r in results]
    node = Node(kind, list(inputs), outs, bwd)
    for o in outs:
        o.parent = node
    for v in inputs:
        v.consumers.append(node)
    return outs


def ancestors(root: Var) -> list[Node]:
    seen, out, todo = set(), [], [root.parent] if root.parent else []
    while todo:
        n = todo.pop()
        if id(n) in seen:
            continue
        seen.add(id(n))
        out.append(n)
        todo.extend(v.parent for v in n.inputs if v.parent is not None)
    return sorted(out, key=lambda n: n.seq)


def backward(root: Var, seed: float = 1.0) -> None:
    """graph.py:311-367: reset to zero, seed q(seed), reverse creation order,
    each contribution accumulated as q(prev + g)."""
    nodes = ancestors(root)
    active: dict[int, Var] = {}
    for n in nodes:
        hit = False
        for v in n.inputs:
            if v.parent is None and v.need_grad:
                active[id(v)] = v
            hit = hit or id(v) in active
        if hit:
            for o in n.outputs:
                active[id(o)] = o
    for v in active.values():
        v.grad = np.zeros(v.shape, dtype=F32)
    root.grad = store(np.full(root.shape, F32(seed), dtype=F32), root.half)
    active[id(root)] = root
    for n in reversed(nodes):
        if not any(id(o) in active for o in n.outputs):
            continue
        want = [id(v) in active for v in n.inputs]
        if not any(want):
            continue
        gxs = n.bwd([o.grad for o in n.outputs], want)
        for v, g, w in zip(n.inputs, gxs, want):
            if w and g is not None:
                v.grad = store(v.grad + np.asarray(g, dtype=F32), v.half)


# ---------------------------------------------------------------------------
# functions (functions.py) — each forward rounds its output once (R1)

def affine(x: Var, w: Var, b: Var, half: bool) -> Var:
    """functions.py:104-116."""
    bsz = x.shape[0]
    x2 = x.value.reshape(bsz, -1)
    y = x2 @ w.value + b.value

    def bwd(gys, want):
        gy = gys[0]
        x2b = x.value.reshape(bsz, -1)
        return [(gy @ w.value.T).reshape(x.shape) if want[0] else None,
                x2b.T @ gy if want[1] else None,
                gy.sum(axis=0) if want[2] else None]

    return _emit("Affine", [x, w, b], [y], bwd, half)[0]


def conv_out(n, k, s, p):
    return (n + 2 * p - k) // s + 1


def _patches(xv, kh, kw, sh, sw, ph, pw):
    """(B,C,H,W) -> (B,C,kh,kw,OH,OW) view of the zero-padded input."""
    xp = np.pad(xv, ((0, 0), (0, 0), (ph, ph), (pw, pw)))
    win = np.lib.stride_tricks.sliding_window_view(xp, (kh, kw), axis=(2, 3))
    win = win[:, :, ::sh, ::sw]          # (B,C,OH,OW,kh,kw)
    return win.transpose(0, 1, 4, 5, 2, 3)


def conv2d(x: Var, w: Var, b: Var, stride, pad, half: bool) -> Var:
    """functions.py:187-212: cross-correlation, f32 sums, bias per map."""
    sh, sw = stride
    ph, pw = pad
    o, c, kh, kw = w.shape
    bsz, _, hh, ww = x.shape
    oh, ow = conv_out(hh, kh, sh, ph), conv_out(ww, kw, sw, pw)
    cols = _patches(x.value, kh, kw, sh, sw, ph, pw).reshape(bsz, c * kh * kw, oh * ow)
    y = np.matmul(w.value.reshape(o, -1), cols) + b.value[None, :, None]
    y = y.reshape(bsz, o, oh, ow)

    def bwd(gys, want):
        gy = gys[0].reshape(bsz, o, oh * ow)
        gx = gw = gb = None
        if want[1]:
            colsb = _patches(x.value, kh, kw, sh, sw, ph, pw).reshape(bsz, c * kh * kw, oh * ow)
            gw = np.einsum("bol,bkl->ok", gy, colsb, optimize=True).reshape(w.shape)
        if want[0]:
            gcols = np.matmul(w.value.reshape(o, -1).T, gy).reshape(bsz, c, kh, kw, oh, ow)
            gxp = np.zeros((bsz, c, hh + 2 * ph, ww + 2 * pw), dtype=F32)
            for i in range(kh):
                for j in range(kw):
                    gxp[:, :, i:i + sh * oh:sh, j:j + sw * ow:sw] += gcols[:, :, i, j]
            gx = gxp[:, :, ph:ph + hh, pw:pw + ww]
        if want[2]:
            gb = gy.sum(axis=(0, 2))
        return [gx, gw, gb]

    return _emit("Convolution", [x, w, b], [y], bwd, half)[0]


def pool_out(n, k, s, p, ignore_border):
    if ignore_border:
        return (n + 2 * p - k) // s + 1
    return -((n + 2 * p - k) // -s) + 1


def maxpool_forward(xv, kernel, stride, pad, ignore_border=True):
    """functions.py:248-274.  Returns (y, window-local argmax uint8).

    Windows read -inf outside the input; np.argmax picks the first maximum
    (and the first NaN) in row-major window order."""
    kh, kw = kernel
    sh, sw = stride
    ph, pw = pad
    bsz, c, hh, ww = xv.shape
    oh = pool_out(hh, kh, sh, ph, ignore_border)
    ow = pool_out(ww, kw, sw, pw, ignore_border)
    th = max((oh - 1) * sh + kh, hh + 2 * ph)
    tw = max((ow - 1) * sw + kw, ww + 2 * pw)
    xp = np.full((bsz, c, th, tw), -np.inf, dtype=F32)
    xp[:, :, ph:ph + hh, pw:pw + ww] = xv
    win = np.stack([xp[:, :, i:i + sh * oh:sh, j:j + sw * ow:sw]
                    for i in range(kh) for j in range(kw)], axis=-1)
    arg = win.argmax(axis=-1)
    return win.max(axis=-1), arg.astype(np.uint8)


def maxpool_backward(gy, arg, x_shape, kernel, stride, pad):
    """functions.py:276-288: scatter-add in output raster order, f32."""
    kh, kw = kernel
    sh, sw = stride
    ph, pw = pad
    bsz, c, hh, ww = x_shape
    oh, ow = gy.shape[2:]
    th = max((oh - 1) * sh + kh, hh + 2 * ph)
    tw = max((ow - 1) * sw + kw, ww + 2 * pw)
    rows = np.arange(oh)[:, None] * sh + arg // kw
    cols = np.arange(ow)[None, :] * sw + arg % kw
    flat = (rows * tw + cols).reshape(bsz, c, -1)
    g = np.zeros((bsz, c, th * tw), dtype=F32)
    np.add.at(g, (np.arange(bsz)[:, None, None], np.arange(c)[None, :, None], flat),
              gy.reshape(bsz, c, -1))
    return g.reshape(bsz, c, th, tw)[:, :, ph:ph + hh, pw:pw + ww]


def max_pooling(x: Var, kernel, stride=None, pad=(0, 0), half=False, ignore_border=True) -> Var:
    stride = kernel if stride is None else stride
    y, arg = maxpool_forward(x.value, kernel, stride, pad, ignore_border)

    def bwd(gys, want):
        return [maxpool_backward(gys[0], arg, x.shape, kernel, stride, pad) if want[0] else None]

    out = _emit("MaxPooling", [x], [y], bwd, half)[0]
    out.argmax = arg
    return out


def relu(x: Var, half: bool) -> Var:
    """functions.py:307-314: NaN passes forward; backward is a multiply."""
    y = np.maximum(x.value, F32(0))

    def bwd(gys, want):
        return [gys[0] * (x.value > 0) if want[0] else None]

    return _emit("ReLU", [x], [y], bwd, half)[0]


class LabelError(ValueError):
    pass


def softmax_ce(logits: Var, labels: Var, half: bool) -> Var:
    """functions.py:334-357: max-shifted log-softmax in f32, mean NLL."""
    lv = logits.value
    k = lv.shape[1]
    ids = labels.value.astype(np.int64)
    if not np.array_equal(ids, labels.value) or ids.min(initial=0) < 0 or ids.max(initial=0) >= k:
        raise LabelError(f"labels must be integers in [0, {k})")
    z = lv - lv.max(axis=1, keepdims=True)
    logp = z - np.log(np.exp(z).sum(axis=1, keepdims=True))
    probs = np.exp(logp)
    loss = F32(-logp[np.arange(lv.shape[0]), ids].mean())

    def bwd(gys, want):
        if not want[0]:
            return [None, None]
        g = probs.copy()
        g[np.arange(g.shape[0]), ids] -= F32(1.0)
        g *= F32(gys[0]) / g.shape[0]
        return [g, None]

    return _emit("SoftmaxCrossEntropy", [logits, labels], [np.asarray(loss, dtype=F32)], bwd,
                 half)[0]


def batch_norm(x: Var, gamma: Var, beta: Var, mean: Var, var: Var, half: bool,
               batch_stat=True, eps=1e-5, momentum=0.9) -> Var:
    """functions.py:401-438 (all statistics f32, biased variance)."""
    xv = x.value
    axes = (0,) + tuple(range(2, xv.ndim))
    shp = (1, -1) + (1,) * (xv.ndim - 2)
    if batch_stat:
        mu = xv.mean(axis=axes)
        vb = xv.var(axis=axes)
        m = F32(momentum)
        mean.value = (m * mean.value + (1 - m) * mu).astype(F32)
        var.value = (m * var.value + (1 - m) * vb).astype(F32)
    else:
        mu, vb = mean.value, var.value
    istd = F32(1.0) / np.sqrt(vb + F32(eps))
    xhat = (xv - mu.reshape(shp)) * istd.reshape(shp)
    y = gamma.value.reshape(shp) * xhat + beta.value.reshape(shp)

    def bwd(gys, want):
        gy = gys[0]
        gbeta = gy.sum(axis=axes)
        ggamma = (gy * xhat).sum(axis=axes)
        gx = None
        if want[0]:
            g = (gamma.value * istd).reshape(shp)
            if batch_stat:
                n = gy.size // gy.shape[1]
                gx = (g / n) * (n * gy - gbeta.reshape(shp) - xhat * ggamma.reshape(shp))
            else:
                gx = g * gy
        return [gx, ggamma if want[1] else None, gbeta if want[2] else None, None, None]

    out = _emit("BatchNormalization", [x, gamma, beta, mean, var], [y], bwd, half)[0]
    out.bn_state = (mu, istd)
    return out


def add2(a: Var, b: Var, half: bool) -> Var:
    """Extension (see module docstring)."""
    y = a.value + b.value

    def bwd(gys, want):
        return [gys[0] if want[0] else None, gys[0] if want[1] else None]

    return _emit("Add2", [a, b], [y], bwd, half)[0]


def gap(x: Var, half: bool) -> Var:
    """Extension (see module docstring): raster-order f32 sum / f32(H*W)."""
    bsz, c, hh, ww = x.shape
    flat = x.value.reshape(bsz, c, hh * ww)
    s = np.zeros((bsz, c), dtype=F32)
    for j in range(hh * ww):
        s = s + flat[:, :, j]
    y = (s / F32(hh * ww)).reshape(bsz, c, 1, 1)

    def bwd(gys, want):
        if not want[0]:
            return [None]
        g = gys[0].reshape(bsz, c, 1, 1) / F32(hh * ww)
        return [np.broadcast_to(g, x.shape).astype(F32)]

    return _emit("GlobalAveragePooling", [x], [y], bwd, half)[0]


# ---------------------------------------------------------------------------
# parameters (parameters.py:40-129) and layers (parametric.py:36-72)

def initial_values(leaf: str, shape, stream: Stream) -> np.ndarray:
    if leaf == "W":
        if len(shape) == 2:
            fi, fo = shape
        elif len(shape) == 4:
            rf = shape[2] * shape[3]
            fi, fo = shape[1] * rf, shape[0] * rf
        else:
            fi = fo = int(np.prod(shape))
        lim = math.sqrt(6.0 / (fi + fo))
        return stream.draw(shape, -lim, lim)
    return np.full(shape, 1.0 if leaf in ("gamma", "var") else 0.0, dtype=F32)


class Model:
    """Parameter store + layer helpers (creation order drives the RNG, R12)."""

    def __init__(self, seed: int = 0, half: bool = False):
        self.params: dict[str, Var] = {}
        self.stream = Stream(seed)
        self.half = half
        self.scope: list[str] = []
        self.batch_stat = True  # False: BN uses the running statistics (eval graph)

    def param(self, path: str, shape, need_grad=True, f32=False) -> Var:
        full = "/".join(self.scope + [path])
        if full in self.params:
            return self.params[full]
        leaf = full.rsplit("/", 1)[-1]
        half = self.half and not f32
        v = Var(initial_values(leaf, tuple(shape), self.stream), half=half,
                need_grad=need_grad, name=full)
        self.params[full] = v
        return v

    def trainable(self) -> dict[str, Var]:
        return {k: v for k, v in self.params.items() if v.need_grad}

    # layers
    def affine(self, x: Var, n_out: int, name: str) -> Var:
        fi = int(np.prod(x.shape[1:]))
        w = self.param(f"{name}/W", (fi, n_out))
        b = self.param(f"{name}/b", (n_out,))
        return affine(x, w, b, self.half)

    def conv(self, x: Var, maps: int, k, name: str, stride=(1, 1), pad=(0, 0)) -> Var:
        kh, kw = (k, k) if isinstance(k, int) else k
        w = self.param(f"{name}/W", (maps, x.shape[1], kh, kw))
        b = self.param(f"{name}/b", (maps,))
        return conv2d(x, w, b, stride, pad, self.half)

    def bn(self, x: Var, name: str, batch_stat=True) -> Var:
        c = x.shape[1]
        g = self.param(f"{name}/gamma", (c,), f32=True)
        be = self.param(f"{name}/beta", (c,), f32=True)
        m = self.param(f"{name}/mean", (c,), need_grad=False, f32=True)
        v = self.param(f"{name}/var", (c,), need_grad=False, f32=True)
        return batch_norm(x, g, be, m, v, self.half, batch_stat=batch_stat)

    def relu(self, x):
        return relu(x, self.half)

    def pool(self, x, k, stride=None, pad=(0, 0)):
        return max_pooling(x, k, stride, pad, self.half)

    def add2(self, a, b):
        return add2(a, b, self.half)

    def gap(self, x):
        return gap(x, self.half)

    def sce(self, logits, labels):
        return softmax_ce(logits, labels, self.half)


# networks (networks.py:13-55 and the ResNet builders of the package)

def lenet(m: Model, x: Var, n_classes=10) -> Var:
    h = m.pool(m.conv(x, 16, 5, "conv1"), (2, 2))
    h = m.relu(h)
    h = m.pool(m.conv(h, 16, 5, "conv2"), (2, 2))
    h = m.relu(h)
    h = m.relu(m.affine(h, 50, "affine3"))
    return m.affine(h, n_classes, "affine4")


def mlp(m: Model, x: Var, n_classes=10, hidden=(32,)) -> Var:
    h = x
    for i, wdt in enumerate(hidden):
        h = m.relu(m.affine(h, wdt, f"fc{i + 1}"))
    return m.affine(h, n_classes, "out")


def _conv_bn(m, x, maps, k, stride, pad, name, act):
    h = m.conv(x, maps, k, name, (stride, stride), (pad, pad))
    h = m.bn(h, f"{name}_bn", batch_stat=m.batch_stat)
    return m.relu(h) if act else h


def _bottleneck(m, x, width, stride, project):
    h = _conv_bn(m, x, width, 1, 1, 0, "conv1", True)
    h = _conv_bn(m, h, width, 3, stride, 1, "conv2", True)
    h = _conv_bn(m, h, width * 4, 1, 1, 0, "conv3", False)
    s = _conv_bn(m, x, width * 4, 1, stride, 0, "shortcut", False) if project else x
    return m.relu(m.add2(h, s))


def _basic(m, x, width, stride, project):
    h = _conv_bn(m, x, width, 3, stride, 1, "conv1", True)
    h = _conv_bn(m, h, width, 3, 1, 1, "conv2", False)
    s = _conv_bn(m, x, width, 1, stride, 0, "shortcut", False) if project else x
    return m.relu(m.add2(h, s))


def _stages(m, h, stages, block, expansion):
    in_c = h.shape[1]
    for si, (width, blocks, stride) in enumerate(stages):
        for bi in range(blocks):
            m.scope.append(f"stage{si + 1}_block{bi + 1}")
            s = stride if bi == 0 else 1
            h = block(m, h, width, s, bi == 0 and (s != 1 or in_c != width * expansion))
            m.scope.pop()
            in_c = width * expansion
    return h


RESNET50_STAGES = ((64, 3, 1), (128, 4, 2), (256, 6, 2), (512, 3, 2))
RESNET18_STAGES = ((64, 2, 1), (128, 2, 2), (256, 2, 2), (512, 2, 2))


def resnet50(m: Model, x: Var, n_classes=1000) -> Var:
    h = _conv_bn(m, x, 64, 7, 2, 3, "stem", True)
    h = m.pool(h, (3, 3), (2, 2), (1, 1))
    h = _stages(m, h, RESNET50_STAGES, _bottleneck, 4)
    return m.affine(m.gap(h), n_classes, "fc")


def resnet18_cifar(m: Model, x: Var, n_classes=10) -> Var:
    h = _conv_bn(m, x, 64, 3, 1, 1, "stem", True)
    h = _stages(m, h, RESNET18_STAGES, _basic, 1)
    return m.affine(m.gap(h), n_classes, "fc")


# ---------------------------------------------------------------------------
# solver (solver.py:67-164) and the data-parallel fold (communicator.py:99-105)

def has_nonfinite(arrays) -> bool:
    return any(a.size and not np.isfinite(a).all() for a in arrays)


@dataclass
class Scaler:
    loss_scale: float = 8.0
    factor: float = 2.0
    interval: int = 2000
    counter: int = 0


class Sgd:
    """SgdSolver (solver.py:67-129) over a Model's trainable parameters.

    Masters are taken lazily on first use; parameters do not change before
    the first update, so this equals setup()-time copies (R11)."""

    def __init__(self, model: "Model", lr: float, momentum=0.0, weight_decay=0.0,
                 clip_norm=None):
        self.model = model
        self.lr = lr
        self.momentum = momentum
        self.wd = weight_decay
        self.clip_norm = clip_norm
        self.master: dict[str, np.ndarray] = {}
        self.vel: dict[str, np.ndarray] = {}

    @property
    def params(self) -> dict[str, Var]:
        return self.model.trainable()

    def _master(self, k, v):
        if k not in self.master:
            self.master[k] = v.value.astype(F32).copy()
            self.vel[k] = np.zeros_like(self.master[k])
        return self.master[k]

    def scale_grad(self, factor: float):
        for v in self.params.values():
            v.grad = store(v.grad * F32(factor), v.half)                          # R10

    def clip_grad_by_norm(self):
        """solver.py:119-129: per-parameter f32 sums of squares, summed as Python
        floats, f32 sqrt; scale by clip/total only when total exceeds clip."""
        if self.clip_norm is None:
            return
        total = np.sqrt(F32(sum(float(np.sum(np.square(v.grad, dtype=F32)))
                                for v in self.params.values())))
        if total > self.clip_norm:
            self.scale_grad(self.clip_norm / float(total))

    def update(self):
        lr = F32(self.lr)
        for k, v in self.params.items():
            g = v.grad
            m = self._master(k, v)
            if self.wd:
                g = g + F32(self.wd) * m
            step = lr * g
            if self.momentum:
                step = F32(self.momentum) * self.vel[k] + step
                self.vel[k] = step
            self.master[k] = (m - step).astype(F32)
            v.value = store(self.master[k], v.half)

    def nonfinite(self) -> bool:
        return has_nonfinite([v.grad for v in self.params.values()])


def dynamic_step(sc: Scaler, opt: Sgd) -> bool:
    """solver.py:132-155; returns True when the update was applied."""
    if opt.nonfinite():
        sc.loss_scale /= sc.factor
        sc.counter = 0
        return False
    opt.scale_grad(1.0 / sc.loss_scale)
    opt.clip_grad_by_norm()
    opt.update()
    if sc.counter > sc.interval:
        sc.loss_scale *= sc.factor
        sc.counter = 0
    sc.counter += 1
    return True


def fold_mean(per_rank: list[list[np.ndarray]], halves: list[bool], division=True):
    """communicator.py:99-105: f32 fold in ascending rank order, /f32(n), round."""
    n = len(per_rank)
    out = []
    for i in range(len(per_rank[0])):
        acc = per_rank[0][i].astype(F32, copy=True)
        for r in range(1, n):
            acc += per_rank[r][i]
        if division:
            acc /= F32(n)
        out.append(store(acc, halves[i]))
    return out


# ---------------------------------------------------------------------------
# a whole training step, single replica or K replicas (communicator.py:206-244)

@dataclass
class Trainer:
    """K replicas built from one seed; the oracle of DataParallelTrainer.

    ``build(model, x, label) -> loss`` constructs the (eager) graph; it is
    called every step and creates parameters on first use like PF.* does."""

    build: object
    workers: int
    batch: int
    lr: float
    seed: int = 0
    half: bool = False
    scaler: Scaler | None = None
    static_scale: float | None = None
    momentum: float = 0.0
    weight_decay: float = 0.0

    def __post_init__(self):
        self.shard = self.batch // self.workers
        self.models = [Model(self.seed, self.half) for _ in range(self.workers)]
        self.opts = [Sgd(m, self.lr, self.momentum, self.weight_decay) for m in self.models]
        self.scalers = [Scaler(**vars(self.scaler)) if self.scaler else None
                        for _ in range(self.workers)]
        self.last_losses: list[Var] = []

    def step(self, x_batch, label_batch) -> float:
        losses = []
        self.last_losses = []
        for r, m in enumerate(self.models):
            lo = r * self.shard
            x = Var(x_batch[lo:lo + self.shard], half=self.half)
            t = Var(label_batch[lo:lo + self.shard], half=self.half)
            loss = self.build(m, x, t)
            for k, v in m.trainable().items():
                self.opts[r]._master(k, v)
            seed = 1.0
            if self.scalers[r] is not None:
                seed = self.scalers[r].loss_scale
            elif self.static_scale is not None:
                seed = self.static_scale
            backward(loss, seed)
            losses.append(float(loss.value))
            self.last_losses.append(loss)
        if self.workers > 1:
            names = list(self.opts[0].params)
            halves = [self.opts[0].params[k].half for k in names]
            red = fold_mean([[o.params[k].grad for k in names] for o in self.opts], halves)
            for o in self.opts:
                for k, g in zip(names, red):
                    o.params[k].grad = g.copy()
        for r, o in enumerate(self.opts):
            if self.scalers[r] is not None:
                dynamic_step(self.scalers[r], o)
            else:
                if self.static_scale is not None:
                    o.scale_grad(1.0 / self.static_scale)
                o.update()
        return float(np.mean(losses))
