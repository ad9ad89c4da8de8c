"""Device-resident arrays with the reference's storage rules.

``NdArray`` mirrors the reference ``NdArray`` (src/tensor.py:62-150) but its
buffer lives in HBM: F16 arrays are genuine binary16 words, F32 arrays are
float32.  Every mutating entry point rounds exactly like the reference's
quantize-on-write (round to nearest even, overflow to inf, subnormals kept),
because the rounding happens in the libnnl kernels (``cvt.rn.f16.f32``).

Physical layout: rank-4 arrays are stored channels-last (NHWC; for conv
weights (O,C,kh,kw) that is KRSC), every other rank row-major.  ``.values``
and ``write`` speak the reference's logical row-major order, converting at
the boundary with ``nnl_export_f32`` / ``nnl_import_f32``.
"""

from __future__ import annotations

import warnings
from dataclasses import dataclass
from enum import Enum

import numpy as np

from . import _lib
from .errors import InvalidRange, ShapeMismatch

__all__ = ["Dtype", "NdArray", "quantize_f16", "has_inf_or_nan", "RngState", "DeviceScalar"]


class Dtype(Enum):
    """Declared storage precision (reference src/tensor.py:39-43)."""

    F32 = "f32"
    F16 = "f16"


def dtype_code(d: Dtype) -> int:
    return _lib.F16 if d is Dtype.F16 else _lib.F32


def torch_dtype(d: Dtype):
    t = _lib.torch()
    return t.float16 if d is Dtype.F16 else t.float32


def _geom(shape: tuple) -> tuple[int, int, int]:
    """(n, c, hw) for the import/export kernels."""
    if len(shape) == 4:
        return shape[0], shape[1], shape[2] * shape[3]
    n = 1
    for d in shape:
        n *= d
    return 1, 1, n


class NdArray:
    """Contiguous device buffer with a declared precision.

    Differences from the host reference are only where the data lives:
    ``values`` returns a host copy (read-only semantics are the same as the
    reference's documented contract), and ``t`` exposes the device tensor to
    the kernels.
    """

    __slots__ = ("dtype", "shape", "_t", "_set", "__weakref__")

    def __init__(self, shape, dtype: Dtype = Dtype.F32, zero: bool = True):
        self.shape = tuple(int(d) for d in shape)
        if any(d < 0 for d in self.shape):
            raise ShapeMismatch(f"negative extent in shape {self.shape}")
        self.dtype = dtype
        self._t = None
        self._set = False
        self._alloc()
        if zero:
            self.fill(0.0)

    def _alloc(self):
        t = _lib.torch()
        kw = dict(dtype=torch_dtype(self.dtype), device=_lib.device())
        if len(self.shape) == 4:
            self._t = t.empty(self.shape, memory_format=t.channels_last, **kw)
        else:
            self._t = t.empty(self.shape, **kw)

    # -- reference API ---------------------------------------------------------
    @classmethod
    def from_values(cls, values, dtype: Dtype = Dtype.F32) -> "NdArray":
        arr = cls(np.shape(values), dtype, zero=False)
        arr.write(values)
        return arr

    @property
    def size(self) -> int:
        n = 1
        for d in self.shape:
            n *= d
        return n

    @property
    def is_set(self) -> bool:
        return self._set

    @property
    def t(self):
        """The device tensor (physical layout); kernels read/write it in place."""
        return self._t

    @property
    def ptr(self) -> int:
        return self._t.data_ptr()

    @property
    def code(self) -> int:
        return dtype_code(self.dtype)

    @property
    def values(self) -> np.ndarray:
        """Host float32 copy in logical (reference) order."""
        if not self._set:
            raise ValueError("buffer has been released")
        t = _lib.torch()
        out = t.empty(self.shape, dtype=t.float32, device=self._t.device)
        n, c, hw = _geom(self.shape)
        _lib.call("nnl_export_f32", self.code, n, c, hw, self.ptr, out.data_ptr(), _lib.stream())
        return out.cpu().numpy()

    def write(self, values) -> None:
        """Replace the contents (host values), quantizing if F16."""
        src = np.asarray(values, dtype=np.float32)
        if src.shape != self.shape:
            raise ShapeMismatch(f"cannot write shape {src.shape} into {self.shape}")
        t = _lib.torch()
        if not src.flags.c_contiguous:
            src = np.array(src, dtype=np.float32, order="C")
        with warnings.catch_warnings():  # read-only views are only read here
            warnings.simplefilter("ignore", UserWarning)
            host = t.from_numpy(src)
        dev = host.to(self._t.device, non_blocking=host.is_pinned())
        self.write_f32_device(dev)

    def write_f32_device(self, dev) -> None:
        """Replace the contents from a logical-order f32 device tensor."""
        n, c, hw = _geom(self.shape)
        _lib.call("nnl_import_f32", self.code, n, c, hw, dev.data_ptr(), self.ptr, _lib.stream())
        self._set = True

    def copy_from(self, other: "NdArray") -> None:
        """Device-to-device write of another array of identical shape/dtype."""
        if other.shape != self.shape or other.dtype is not self.dtype:
            raise ShapeMismatch("copy_from needs identical shape and dtype")
        _lib.call("nnl_accumulate", self.code, self.size, other.ptr, self.ptr, 0, _lib.stream())
        self._set = True

    def accumulate(self, values) -> None:
        """In-place add (float32 math), re-quantizing if F16."""
        if isinstance(values, NdArray):
            if values.shape != self.shape or values.dtype is not self.dtype:
                raise ShapeMismatch("accumulate needs identical shape and dtype")
            _lib.call("nnl_accumulate", self.code, self.size, values.ptr, self.ptr, 1,
                      _lib.stream())
            return
        src = np.asarray(values, dtype=np.float32)
        if src.shape != self.shape:
            raise ShapeMismatch(f"cannot accumulate shape {src.shape} into {self.shape}")
        tmp = NdArray(self.shape, Dtype.F32, zero=False)
        tmp.write(src)
        if self.dtype is Dtype.F32:
            _lib.call("nnl_accumulate", self.code, self.size, tmp.ptr, self.ptr, 1, _lib.stream())
        else:
            # f32 add then one rounding: stage the current values in f32
            cur = NdArray(self.shape, Dtype.F32, zero=False)
            _lib.call("nnl_export_f32", self.code, 1, 1, self.size, self.ptr, cur.ptr,
                      _lib.stream())
            _lib.call("nnl_accumulate", _lib.F32, self.size, tmp.ptr, cur.ptr, 1, _lib.stream())
            _lib.call("nnl_import_f32", self.code, 1, 1, self.size, cur.ptr, self.ptr,
                      _lib.stream())
        self._set = True

    def fill(self, value) -> None:
        """Uniform fill; a DeviceScalar value is read on the device (no sync)."""
        if isinstance(value, DeviceScalar):
            _lib.call("nnl_fill_from_device", self.code, self.size, self.ptr, value.ptr,
                      _lib.stream())
        else:
            _lib.call("nnl_fill", self.code, self.size, self.ptr, float(np.float32(value)),
                      _lib.stream())
        self._set = True

    def release(self) -> None:
        """Mark the buffer unreadable (memory is kept for the next write)."""
        self._set = False

    def mark_set(self) -> None:
        self._set = True

    def copy(self) -> "NdArray":
        out = NdArray(self.shape, self.dtype, zero=False)
        if self._set:
            out.copy_from(self)
        return out

    def tobytes(self) -> bytes:
        """Bytes of the float32 logical values (as the reference's tobytes)."""
        return np.ascontiguousarray(self.values).tobytes()

    def raw_bytes(self) -> bytes:
        """Bytes of the physical storage (genuine binary16 words for F16)."""
        return self._t.contiguous().view(-1).view(_lib.torch().uint8).cpu().numpy().tobytes()

    def __repr__(self):
        state = "released" if not self._set else f"{self.size} elements on {self._t.device}"
        return f"NdArray(shape={self.shape}, dtype={self.dtype.value}, {state})"


class DeviceScalar:
    """A float64 scalar in device memory (e.g. the dynamic loss scale)."""

    __slots__ = ("_t",)

    def __init__(self, tensor):
        self._t = tensor

    @property
    def ptr(self) -> int:
        return self._t.data_ptr()

    def item(self) -> float:
        return float(self._t.item())


def quantize_f16(x: float) -> float:
    """Round a float32 value to binary16 (reference src/tensor.py:52-59), on device."""
    t = _lib.torch()
    src = t.tensor([np.float32(x)], dtype=t.float32, device=_lib.device())
    out = t.empty_like(src)
    _lib.call("nnl_quantize_f16", 1, src.data_ptr(), out.data_ptr(), _lib.stream())
    return float(out.item())


def quantize_f16_array(x) -> np.ndarray:
    t = _lib.torch()
    src = t.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).to(_lib.device())
    out = t.empty_like(src)
    _lib.call("nnl_quantize_f16", src.numel(), src.data_ptr(), out.data_ptr(), _lib.stream())
    return out.cpu().numpy()


def has_inf_or_nan(a: NdArray) -> bool:
    """True iff any element is inf or NaN (reference src/tensor.py:153-157)."""
    if a.size == 0:
        return False
    t = _lib.torch()
    flag = t.zeros(1, dtype=t.int32, device=_lib.device())
    _lib.call("nnl_nonfinite", a.code, a.size, a.ptr, flag.data_ptr(), _lib.stream())
    return bool(flag.item())


_MIX1 = 0xBF58476D1CE4E5B9
_GOLDEN = 0x9E3779B97F4B7C15
_M64 = (1 << 64) - 1


def _splitmix64_int(x: int) -> int:
    z = (x + _GOLDEN) & _M64
    z = ((z ^ (z >> 30)) * _MIX1) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return z ^ (z >> 31)


@dataclass
class RngState:
    """Counter-based SplitMix64 stream (reference src/tensor.py:225-257).

    Draws are generated on the device by ``nnl_rng_uniform``; draw i is a
    pure function of (seed, counter + i), bit-identical to the reference.
    """

    seed: int
    counter: int = 0

    def derived(self, tag: int) -> "RngState":
        mixed = _splitmix64_int(tag & _M64)
        return RngState(seed=_splitmix64_int((self.seed ^ mixed) & _M64))

    def next_uniform_device(self, shape, low: float = 0.0, high: float = 1.0,
                            dtype: Dtype = Dtype.F32):
        """Draw into a new logical-order device tensor of `dtype`."""
        if low >= high:
            raise InvalidRange(f"empty range [{low}, {high})")
        t = _lib.torch()
        n = int(np.prod(shape, dtype=np.int64))
        out = t.empty(tuple(int(d) for d in shape), dtype=torch_dtype(dtype),
                      device=_lib.device())
        _lib.call("nnl_rng_uniform", self.seed & _M64, self.counter & _M64, n, float(low),
                  float(high), dtype_code(dtype), out.data_ptr(), _lib.stream())
        self.counter += n
        return out

    def next_uniform(self, shape, low: float = 0.0, high: float = 1.0) -> np.ndarray:
        """Host copy of a device draw (reference API returns numpy)."""
        return self.next_uniform_device(shape, low, high).cpu().numpy()

    def permutation(self, n: int) -> np.ndarray:
        keys = self.next_uniform((n,))
        return np.argsort(keys, kind="stable")
