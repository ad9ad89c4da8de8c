"""Checkpoint / resume of the training state.

The file is the reference's NNP ``parameter.bin`` record stream
(nnp.py:467-535: magic ``NNPB``, u32 record count, then per record the UTF-8
name, dtype byte (1 = F16, 0 = F32), need_grad byte, u32 rank, u32 dims and the
little-endian payload) — parameters are written as their genuine storage words
(F16 for half parameters), so a reference NNP reader loads them unchanged.  The
resume state the reference has no format for is appended as extra F32 records
with reserved names:

    ``__master__/<name>``    f32 master copy (solver.py:89-92), logical order
    ``__momentum__/<name>``  f32 velocity of the momentum extension
    ``__scaler__``           [loss_scale, scaling_factor, interval, counter]

Everything is read back from device buffers once per save; a load writes the
device buffers in place (addresses unchanged, so a captured CUDA graph stays
valid).
"""

from __future__ import annotations

import struct
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import ShapeMismatch

MAGIC = 0x4E4E5042
MASTER = "__master__/"
MOMENTUM = "__momentum__/"
SCALER = "__scaler__"


@dataclass
class Record:
    name: str
    shape: tuple
    f16: bool
    values: np.ndarray  # float32 host values in logical order
    need_grad: bool = False


def encode(records: list[Record]) -> bytes:
    """Serialise records exactly as the reference's emit_parameter_bin."""
    out = bytearray(struct.pack("<II", MAGIC, len(records)))
    for r in records:
        name = r.name.encode("utf-8")
        out += struct.pack("<I", len(name)) + name
        out += struct.pack("<BB", 1 if r.f16 else 0, 1 if r.need_grad else 0)
        out += struct.pack("<I", len(r.shape))
        for d in r.shape:
            out += struct.pack("<I", int(d))
        out += np.asarray(r.values, np.float32).astype("<f2" if r.f16 else "<f4").tobytes()
    return bytes(out)


def decode(data: bytes) -> list[Record]:
    """Parse a record stream (inverse of `encode`); raises ValueError on damage."""
    pos = 0

    def take(n: int) -> bytes:
        nonlocal pos
        if pos + n > len(data):
            raise ValueError("checkpoint truncated")
        chunk = data[pos:pos + n]
        pos += n
        return chunk

    magic, count = struct.unpack("<II", take(8))
    if magic != MAGIC:
        raise ValueError(f"bad checkpoint magic {magic:#x}")
    out = []
    for _ in range(count):
        (ln,) = struct.unpack("<I", take(4))
        name = take(ln).decode("utf-8")
        f16, ng = struct.unpack("<BB", take(2))
        if f16 not in (0, 1) or ng not in (0, 1):
            raise ValueError(f"record {name!r}: bad dtype/need_grad byte")
        (nd,) = struct.unpack("<I", take(4))
        shape = tuple(struct.unpack("<I", take(4))[0] for _ in range(nd))
        n = int(np.prod(shape, dtype=np.int64)) if shape else 1
        vals = np.frombuffer(take(n * (2 if f16 else 4)), "<f2" if f16 else "<f4")
        out.append(Record(name, shape, bool(f16), vals.astype(np.float32).reshape(shape),
                          bool(ng)))
    if pos != len(data):
        raise ValueError("trailing bytes after the last record")
    return out


def _physical_to_logical(flat, shape):
    if len(shape) == 4:  # conv weights live as [O][kh][kw][C]
        o, c, kh, kw = shape
        return flat.reshape(o, kh, kw, c).transpose(0, 3, 1, 2)
    return flat.reshape(shape)


def _logical_to_physical(values, shape):
    if len(shape) == 4:
        return np.ascontiguousarray(np.asarray(values, np.float32).transpose(0, 2, 3, 1))
    return np.ascontiguousarray(np.asarray(values, np.float32))


def save(path: str, params: dict, solver=None, scaler=None) -> None:
    """Write parameters (+ solver masters/momentum, + loss-scaler state)."""
    from .tensor import Dtype
    recs = []
    for name, v in params.items():
        recs.append(Record(name, tuple(v.shape), v.dtype is Dtype.F16, v.d, bool(v.need_grad)))
    if solver is not None and solver.slots is not None:
        for name, slot in solver.slots.items():
            shape = tuple(slot.param.shape)
            recs.append(Record(MASTER + name, shape, False,
                               _physical_to_logical(slot.master.cpu().numpy(), shape)))
            if slot.velocity is not None:
                recs.append(Record(MOMENTUM + name, shape, False,
                                   _physical_to_logical(slot.velocity.cpu().numpy(), shape)))
    if scaler is not None:
        st = scaler.snapshot() if hasattr(scaler, "snapshot") else scaler
        recs.append(Record(SCALER, (4,), False,
                           np.array([st.loss_scale, st.scaling_factor, st.interval, st.counter],
                                    np.float32)))
    with open(path, "wb") as f:
        f.write(encode(recs))


def load(path: str, params: dict, solver=None, scaler=None) -> None:
    """Restore what `save` wrote into existing (same-shape) objects in place."""
    with open(path, "rb") as f:
        recs = {r.name: r for r in decode(f.read())}
    t = _lib.torch()
    for name, v in params.items():
        if name not in recs:
            raise KeyError(f"parameter {name!r} missing from {path}")
        r = recs[name]
        if tuple(r.shape) != tuple(v.shape):
            raise ShapeMismatch(f"{name}: checkpoint shape {r.shape} != {v.shape}")
        v.d = r.values
    if solver is not None and solver.slots is not None:
        for name, slot in solver.slots.items():
            shape = tuple(slot.param.shape)
            for key, dst in ((MASTER + name, slot.master), (MOMENTUM + name, slot.velocity)):
                if dst is None:
                    continue
                if key not in recs:
                    # a params-only file (e.g. the reference's parameter.bin): the
                    # master restarts from the loaded weight (R11, solver.py:89-92)
                    # and the velocity from zero, as a fresh setup() would
                    if key.startswith(MASTER):
                        p = slot.param.data
                        _lib.call("nnl_export_f32", p.code, 1, 1, p.size, p.ptr,
                                  dst.data_ptr(), _lib.stream())
                    else:
                        dst.zero_()
                    continue
                if tuple(recs[key].shape) != shape:
                    raise ShapeMismatch(f"{key}: checkpoint shape {recs[key].shape} != {shape}")
                src = t.from_numpy(_logical_to_physical(recs[key].values, shape).reshape(-1))
                dst.copy_(src.to(dst.device))
    if scaler is not None and SCALER in recs:
        ls, sf, iv, ct = (float(x) for x in recs[SCALER].values)
        if hasattr(scaler, "restore"):
            scaler.restore(ls, sf, int(iv), int(ct))
        else:
            scaler.loss_scale, scaler.scaling_factor = ls, sf
            scaler.interval, scaler.counter = int(iv), int(ct)
