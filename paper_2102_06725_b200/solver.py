"""SGD with float32 masters and loss scaling (reference src/solver.py).

The host-facing API is the reference's (``SgdSolver``, ``DynamicLossScaler``,
``dynamic_step``, ``static_scaling_step``) with identical semantics.  Every
multi-parameter pass is one libnnl launch over a chunk table covering all
parameters:

* ``check_inf_or_nan_grad``  -> nnl_multi_nonfinite (one read of all grads)
* ``scale_grad``             -> nnl_multi_scale_grad
* ``update``                 -> nnl_multi_sgd_update

``DeviceLossScaler`` + ``SgdSolver.dynamic_update`` keep the scaler state in
HBM so a training step never synchronises with the host: the overflow flag is
OR-ed by the gradient-producing kernels, the update kernel skips itself when
the flag is set, and ``nnl_scaler_finish`` applies the reference's
halve/double bookkeeping (solver.py:142-153).

Extension (unpinned by the reference, which has plain SGD only):
``momentum`` and ``weight_decay`` follow NNabla's Momentum solver,
v = m*v + lr*(g + wd*w); w -= v, which reduces to the reference update for
m = wd = 0.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import EmptyParameterSet, NotSetup
from .graph import Variable
from .tensor import DeviceScalar, Dtype

__all__ = ["SgdSolver", "MomentumSgdSolver", "DynamicLossScaler", "DeviceLossScaler",
           "StepOutcome", "dynamic_step", "static_scaling_step"]

CHUNK = 4096


@dataclass
class StepOutcome:
    applied: bool
    loss_scale_after: float
    reason: str  # "Applied" or "SkippedInfNan"


@dataclass
class DynamicLossScaler:
    """Host-side scaler state (reference solver.py:49-64)."""

    loss_scale: float = 8.0
    scaling_factor: float = 2.0
    interval: int = 2000
    counter: int = 0

    def __post_init__(self):
        if self.loss_scale <= 0:
            raise ValueError("loss_scale must stay positive")
        if self.scaling_factor <= 1:
            raise ValueError("scaling_factor must exceed 1")
        if self.interval < 1:
            raise ValueError("interval must be >= 1")


class DeviceLossScaler:
    """The same state machine resident in device memory (nnl_scaler_state)."""

    def __init__(self, template: DynamicLossScaler | None = None):
        t = _lib.torch()
        tpl = template or DynamicLossScaler()
        st = _lib.ScalerState(float(tpl.loss_scale), float(tpl.scaling_factor),
                              int(tpl.interval), int(tpl.counter), 0, 1)
        raw = bytes(st)
        self._buf = t.frombuffer(bytearray(raw), dtype=t.uint8).to(_lib.device())
        self.ptr = self._buf.data_ptr()
        self.loss_scale_ptr = DeviceScalar(self._buf[:8].view(t.float64))

    @property
    def nonfinite_ptr(self) -> int:
        return self.ptr + _lib.ScalerState.nonfinite.offset

    def snapshot(self) -> DynamicLossScaler:
        raw = bytes(self._buf.cpu().numpy().tobytes())
        st = _lib.ScalerState.from_buffer_copy(raw)
        return DynamicLossScaler(st.loss_scale, st.scaling_factor, st.interval, st.counter)

    def last_applied(self) -> bool:
        raw = bytes(self._buf.cpu().numpy().tobytes())
        return bool(_lib.ScalerState.from_buffer_copy(raw).applied)

    def restore(self, loss_scale: float, scaling_factor: float, interval: int,
                counter: int) -> None:
        """Overwrite the device state in place (checkpoint resume)."""
        t = _lib.torch()
        st = _lib.ScalerState(float(loss_scale), float(scaling_factor), int(interval),
                              int(counter), 0, 1)
        self._buf.copy_(t.frombuffer(bytearray(bytes(st)), dtype=t.uint8))


@dataclass
class _Slot:
    param: Variable
    master: object  # torch f32 tensor, physical layout of the parameter storage
    velocity: object | None


def _device_table(structs: list) -> object:
    t = _lib.torch()
    if not structs:
        return t.empty(1, dtype=t.uint8, device=_lib.device())
    arr = (type(structs[0]) * len(structs))(*structs)
    return t.frombuffer(bytearray(bytes(arr)), dtype=t.uint8).to(_lib.device())


def build_chunks(sizes: list[int], chunk: int = CHUNK) -> list:
    out = []
    for s, n in enumerate(sizes):
        for start in range(0, n, chunk):
            out.append(_lib.Chunk(s, min(chunk, n - start), start))
    return out


class SgdSolver:
    """w <- w - lr*g on float32 masters (reference solver.py:67-129)."""

    def __init__(self, lr: float, clip_norm: float | None = None, momentum: float = 0.0,
                 weight_decay: float = 0.0):
        if lr <= 0:
            raise ValueError(f"lr must be positive, got {lr}")
        self.lr = float(lr)
        self.clip_norm = clip_norm
        self.momentum = float(momentum)
        self.weight_decay = float(weight_decay)
        self.slots: dict[str, _Slot] | None = None
        self._tables = None

    def setup(self, params: dict[str, Variable]) -> "SgdSolver":
        items = list(params.items())
        if not items:
            raise EmptyParameterSet("solver needs at least one parameter")
        for name, v in items:
            if not v.need_grad:
                raise ValueError(f"parameter {name!r} is frozen (need_grad=False)")
        t = _lib.torch()
        slots = {}
        for name, v in items:
            master = t.empty(v.data.size, dtype=t.float32, device=_lib.device())
            # R11: master = f32 copy of the (already rounded) visible weight
            _lib.call("nnl_export_f32", v.data.code, 1, 1, v.data.size, v.data.ptr,
                      master.data_ptr(), _lib.stream())
            vel = t.zeros_like(master) if self.momentum != 0.0 else None
            v.grad  # allocate the grad buffer now so its address is stable
            slots[name] = _Slot(v, master, vel)
        self.slots = slots
        self._build_tables()
        return self

    set_parameters = setup

    def _build_tables(self):
        descs = []
        sizes = []
        for s in self.slots.values():
            p = s.param
            descs.append(_lib.ParamSlot(p.data.ptr, p.grad.ptr, s.master.data_ptr(),
                                        s.velocity.data_ptr() if s.velocity is not None else None,
                                        p.data.size, p.data.code, 0))
            sizes.append(p.data.size)
        chunks = build_chunks(sizes)
        self._tables = (_device_table(descs), _device_table(chunks), len(chunks))

    def _require_setup(self) -> dict[str, _Slot]:
        if self.slots is None:
            raise NotSetup("call setup() before using the solver")
        return self.slots

    def _args(self):
        self._require_setup()
        slots, chunks, n = self._tables
        return slots.data_ptr(), chunks.data_ptr(), n

    # -- reference API -----------------------------------------------------
    def update(self) -> None:
        """master <- master - lr*grad; visible weight <- q(master)."""
        s, c, n = self._args()
        _lib.call("nnl_multi_sgd_update", s, c, n, float(np.float32(self.lr)),
                  float(np.float32(self.momentum)), float(np.float32(self.weight_decay)), None,
                  _lib.stream())
        self._mark_written()

    def scale_grad(self, factor: float) -> None:
        s, c, n = self._args()
        _lib.call("nnl_multi_scale_grad", s, c, n, float(np.float32(factor)), _lib.stream())

    def zero_grad(self) -> None:
        for slot in self._require_setup().values():
            slot.param.grad.fill(0.0)

    def check_inf_or_nan_grad(self) -> bool:
        s, c, n = self._args()
        t = _lib.torch()
        flag = t.zeros(1, dtype=t.int32, device=_lib.device())
        _lib.call("nnl_multi_nonfinite", s, c, n, flag.data_ptr(), _lib.stream())
        return bool(flag.item())

    def clip_grad_by_norm(self) -> None:
        if self.clip_norm is None:
            return
        s, c, n = self._args()
        t = _lib.torch()
        acc = t.zeros(1, dtype=t.float64, device=_lib.device())
        _lib.call("nnl_multi_sumsq", s, c, n, acc.data_ptr(), _lib.stream())
        total = np.sqrt(np.float32(acc.item()))
        if total > self.clip_norm:
            self.scale_grad(self.clip_norm / float(total))

    # -- device-resident fast path ------------------------------------------
    def dynamic_update(self, scaler: DeviceLossScaler, check: bool = True) -> None:
        """dynamic_step without a host sync.

        check=False when every gradient-producing kernel already OR-ed the
        overflow flag into ``scaler`` (the trainer arranges that)."""
        if self.clip_norm is not None:
            raise NotImplementedError("clip_norm needs the host-synchronous dynamic_step")
        s, c, n = self._args()
        st = _lib.stream()
        if check:
            _lib.call("nnl_multi_nonfinite", s, c, n, scaler.nonfinite_ptr, st)
        _lib.call("nnl_multi_sgd_update", s, c, n, float(np.float32(self.lr)),
                  float(np.float32(self.momentum)), float(np.float32(self.weight_decay)),
                  scaler.ptr, st)
        _lib.call("nnl_scaler_finish", scaler.ptr, st)
        self._mark_written()

    def _mark_written(self):
        for slot in self.slots.values():
            slot.param.data.mark_set()

    def master_values(self, name: str) -> np.ndarray:
        """Host copy of a master in the parameter's logical order."""
        slot = self._require_setup()[name]
        return self._logical(slot, slot.master)

    def velocity_values(self, name: str) -> np.ndarray | None:
        """Host copy of a momentum buffer (None without momentum)."""
        slot = self._require_setup()[name]
        return None if slot.velocity is None else self._logical(slot, slot.velocity)

    @staticmethod
    def _logical(slot, m) -> np.ndarray:
        shape = slot.param.shape
        if len(shape) == 4:
            o, c, kh, kw = shape
            return m.view(o, kh, kw, c).permute(0, 3, 1, 2).cpu().numpy()
        return m.view(shape).cpu().numpy()


class MomentumSgdSolver(SgdSolver):
    """Extension: NNabla-style Momentum SGD with weight decay."""

    def __init__(self, lr: float, momentum: float = 0.9, weight_decay: float = 0.0,
                 clip_norm: float | None = None):
        super().__init__(lr, clip_norm=clip_norm, momentum=momentum, weight_decay=weight_decay)


def dynamic_step(scaler: DynamicLossScaler, solver: SgdSolver) -> StepOutcome:
    """One adaptive-scale step (reference solver.py:132-155), host-synchronous."""
    if solver.check_inf_or_nan_grad():
        scaler.loss_scale /= scaler.scaling_factor
        scaler.counter = 0
        return StepOutcome(False, scaler.loss_scale, "SkippedInfNan")
    solver.scale_grad(1.0 / scaler.loss_scale)
    solver.clip_grad_by_norm()
    solver.update()
    if scaler.counter > scaler.interval:
        scaler.loss_scale *= scaler.scaling_factor
        scaler.counter = 0
    scaler.counter += 1
    assert scaler.loss_scale > 0
    return StepOutcome(True, scaler.loss_scale, "Applied")


def static_scaling_step(loss: Variable, solver: SgdSolver, loss_scale: float = 8.0) -> None:
    """backward(loss_scale), unscale, update (reference solver.py:158-164)."""
    solver._require_setup()
    loss.backward(grad_seed=loss_scale)
    solver.scale_grad(1.0 / loss_scale)
    solver.clip_grad_by_norm()
    solver.update()
