"""ctypes binding of libnnl.so (include/nnl.h) and device plumbing.

This is the only module that talks to the native library.  Every call goes
through :func:`call`, which turns a nonzero status into the matching
exception class of :mod:`errors`.  There is no fallback: if the shared
library is missing, or no CUDA device is visible, using the package raises.
"""

from __future__ import annotations

import contextlib
import ctypes as C
import os
import threading

from . import errors as E

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("NNL_LIB_PATH") or os.path.join(_HERE, "libnnl.so")

F32, F16 = 0, 1

_STATUS = {
    1: E.ShapeMismatch,
    2: E.KernelTooLarge,
    3: E.LabelOutOfRange,
    4: E.DegenerateBatch,
    5: E.NotSetup,
    6: E.CollectiveTimeout,
    7: E.ShapeMismatchAcrossRanks,
    8: E.InvalidRange,
}

p = C.c_void_p
i32 = C.c_int32
i64 = C.c_int64
u64 = C.c_uint64
f32 = C.c_float
f64 = C.c_double
sz = C.c_size_t


class ConvShape(C.Structure):
    _fields_ = [(n, i32) for n in ("n", "h", "w", "c", "k", "r", "s", "stride_h", "stride_w",
                                   "pad_h", "pad_w", "p", "q")]


class PoolShape(C.Structure):
    _fields_ = [(n, i32) for n in ("n", "h", "w", "c", "kh", "kw", "sh", "sw", "ph", "pw",
                                   "p", "q")]


class BnBwdFuse(C.Structure):
    """nnl_bn_bwd_fuse (include/nnl.h)."""
    _fields_ = [("x", p), ("gate", p), ("gamma", p), ("beta", p), ("save_mean", p),
                ("save_istd", p), ("relu", i32), ("canonical", i32), ("out", p),
                ("partials", p)]


class ParamSlot(C.Structure):
    _fields_ = [("data", p), ("grad", p), ("master", p), ("momentum", p), ("n", i64),
                ("dtype", i32), ("pad_", i32)]


class Chunk(C.Structure):
    _fields_ = [("slot", i32), ("len", i32), ("start", i64)]


class ScalerState(C.Structure):
    _fields_ = [("loss_scale", f64), ("scaling_factor", f64), ("interval", i64),
                ("counter", i64), ("nonfinite", i32), ("applied", i32)]


_SIGS = {
    "nnl_last_error": (C.c_char_p, []),
    "nnl_version": (C.c_int, []),
    "nnl_launch_count": (i64, [C.c_int]),
    "nnl_set_tc_enabled": (C.c_int, [C.c_int]),
    "nnl_set_tc_pairs": (C.c_int, [C.c_int]),
    "nnl_set_pdl": (C.c_int, [C.c_int]),
    "nnl_set_tc_resident_b": (C.c_int, [C.c_int]),
    "nnl_set_tc_s2d4": (C.c_int, [C.c_int]),
    "nnl_set_tc_tile4": (C.c_int, [C.c_int]),
    "nnl_set_tc_halo": (C.c_int, [C.c_int]),
    "nnl_set_tc_epi_il": (C.c_int, [C.c_int]),
    "nnl_conv2d_prep_reuse": (C.c_int, [C.c_int]),
    "nnl_quantize_f16": (C.c_int, [i64, p, p, p]),
    "nnl_fill": (C.c_int, [C.c_int, i64, p, f32, p]),
    "nnl_fill_from_device": (C.c_int, [C.c_int, i64, p, p, p]),
    "nnl_accumulate": (C.c_int, [C.c_int, i64, p, p, C.c_int, p]),
    "nnl_nonfinite": (C.c_int, [C.c_int, i64, p, p, p]),
    "nnl_rng_uniform": (C.c_int, [u64, u64, i64, f64, f64, C.c_int, p, p]),
    "nnl_affine_workspace_size": (sz, [C.c_int, i64, i64, i64, C.c_int]),
    "nnl_affine_fwd": (C.c_int, [C.c_int, i64, i64, i64, i64, p, p, p, p, p, sz, p]),
    "nnl_affine_bwd_data": (C.c_int, [C.c_int, i64, i64, i64, i64, p, p, p, C.c_int, p, sz, p]),
    "nnl_affine_bwd_weight": (C.c_int, [C.c_int, i64, i64, i64, i64, p, p, p, C.c_int, p,
                                        C.c_int, p, p, sz, p]),
    "nnl_conv2d_workspace_size": (sz, [p, C.c_int, C.c_int]),
    "nnl_conv2d_stat_rows": (i32, [p, C.c_int]),
    "nnl_conv2d_fwd": (C.c_int, [p, C.c_int, p, p, p, p, p, p, p, sz, p]),
    "nnl_conv2d_bwd_data": (C.c_int, [p, C.c_int, p, p, p, C.c_int, p, sz, p]),
    "nnl_conv2d_bwd_weight": (C.c_int, [p, C.c_int, p, p, p, C.c_int, p, C.c_int, p, p, sz, p]),
    "nnl_conv2d_bwd_data_bn_rows": (i32, [p, C.c_int]),
    "nnl_conv2d_bwd_data_bn": (C.c_int, [p, C.c_int, p, p, p, C.c_int, p, p, sz, p]),
    "nnl_maxpool_fwd": (C.c_int, [C.c_int, p, p, p, p, p]),
    "nnl_maxpool_bwd": (C.c_int, [C.c_int, p, p, p, p, C.c_int, p]),
    "nnl_bn_relu_maxpool_ok": (C.c_int, [C.c_int, p]),
    "nnl_bn_relu_maxpool_fwd": (C.c_int, [C.c_int, p, p, p, p, p, p, p, p, p]),
    "nnl_relu_fwd": (C.c_int, [C.c_int, i64, p, p, p]),
    "nnl_relu_bwd": (C.c_int, [C.c_int, i64, p, p, p, C.c_int, p]),
    "nnl_add2_fwd": (C.c_int, [C.c_int, i64, p, p, p, C.c_int, p]),
    "nnl_gap_fwd": (C.c_int, [C.c_int, i64, i64, i64, p, p, p]),
    "nnl_gap_bwd": (C.c_int, [C.c_int, i64, i64, i64, p, p, C.c_int, p]),
    "nnl_sce_fwd": (C.c_int, [C.c_int, i64, i64, p, p, p, p, p, p]),
    "nnl_sce_bwd": (C.c_int, [C.c_int, i64, i64, p, p, p, p, p, C.c_int, p]),
    "nnl_bn_workspace_size": (sz, [i64, i32]),
    "nnl_bn_fwd_train": (C.c_int, [C.c_int, i64, i32, p, p, p, p, p, f32, f32, p, i32, p, p, p,
                                   p, p, C.c_int, p, sz, p]),
    "nnl_bn_fwd_eval": (C.c_int, [C.c_int, i64, i32, p, p, p, p, p, f32, p, p, p, p, C.c_int,
                                  p]),
    "nnl_bn_bwd": (C.c_int, [C.c_int, i64, i32, p, p, C.c_int, p, p, C.c_int, p, p, p, p,
                             C.c_int, p, C.c_int, p, C.c_int, p, C.c_int, p, C.c_int, p, p, sz,
                             p]),
    "nnl_bn_bwd_apply": (C.c_int, [C.c_int, i64, i32, p, p, p, i32, p, p, p, C.c_int, p,
                                   C.c_int, p, C.c_int, p, C.c_int, p, C.c_int, p, p, sz, p]),
    "nnl_multi_nonfinite": (C.c_int, [p, p, i32, p, p]),
    "nnl_multi_scale_grad": (C.c_int, [p, p, i32, f32, p]),
    "nnl_multi_sumsq": (C.c_int, [p, p, i32, p, p]),
    "nnl_multi_sgd_update": (C.c_int, [p, p, i32, f32, f32, f32, p, p]),
    "nnl_scaler_finish": (C.c_int, [p, p]),
    "nnl_bucket_pack": (C.c_int, [p, p, p, i32, p, p]),
    "nnl_bucket_unpack_mean": (C.c_int, [p, p, p, i32, p, i32, p, p]),
    "nnl_fold_f32": (C.c_int, [i32, p, i64, p, p]),
    "nnl_comm_unique_id": (C.c_int, [p]),
    "nnl_comm_init": (C.c_int, [C.POINTER(p), i32, i32, p, i32]),
    "nnl_comm_destroy": (C.c_int, [p]),
    "nnl_comm_bucket_elems": (i64, [p, i64]),
    "nnl_comm_workspace_size": (sz, [p, i64]),
    "nnl_comm_allreduce_mean": (C.c_int, [p, p, p, p, i32, p, i64, i32, p, p, sz, p]),
    "nnl_comm_allreduce_sum_f32": (C.c_int, [p, p, i64, p]),
    "nnl_import_f32": (C.c_int, [C.c_int, i32, i32, i32, p, p, p]),
    "nnl_export_f32": (C.c_int, [C.c_int, i32, i32, i32, p, p, p]),
}

_lib = None
_lock = threading.Lock()


def lib():
    """Load libnnl.so once; raise DeviceError if it is absent (no fallback)."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not os.path.exists(LIB_PATH):
                    raise E.DeviceError(
                        f"{LIB_PATH} is missing: build it with __graft_entry__.build() "
                        "(make -C paper_2102_06725_b200/csrc)")
                handle = C.CDLL(LIB_PATH)
                for name, (res, args) in _SIGS.items():
                    fn = getattr(handle, name)
                    fn.restype = res
                    fn.argtypes = args
                _lib = handle
    return _lib


def exported_symbols() -> list[str]:
    return sorted(_SIGS)


def last_error() -> str:
    return lib().nnl_last_error().decode(errors="replace")


def call(name: str, *args) -> int:
    """Invoke a status-returning entry point; raise the mapped error class."""
    rc = getattr(lib(), name)(*args)
    if rc != 0:
        msg = last_error()
        raise _STATUS.get(rc, E.DeviceError)(f"{name}: {msg} (status {rc})")
    return rc


# --- device plumbing ----------------------------------------------------------

_torch = None


def torch():
    """PyTorch is used for device memory, streams and torch.distributed only."""
    global _torch
    if _torch is None:
        import torch as t
        _torch = t
    return _torch


def device():
    t = torch()
    if not t.cuda.is_available():
        raise E.DeviceError("no CUDA device visible: this package has no CPU path")
    return t.device("cuda", t.cuda.current_device())


def stream() -> int:
    """Raw cudaStream_t of torch's current stream on the current device."""
    return torch().cuda.current_stream().cuda_stream


class _Workspace(threading.local):
    def __init__(self):
        self.buf = None


_ws = _Workspace()


def workspace(nbytes: int):
    """A per-thread scratch buffer shared by consecutive kernels on one stream.

    Grows monotonically; returns (pointer, size).  Callers never hold it
    across an API call, so reuse by the next kernel on the same stream is safe.
    Inside `branch_scope()` the branch stream's own buffer is returned.
    """
    if _branch.active:
        return _branch_workspace(nbytes)
    t = torch()
    nbytes = int(max(nbytes, 1 << 20))
    if _ws.buf is None or _ws.buf.numel() < nbytes:
        _ws.buf = t.empty(nbytes + (nbytes >> 2), dtype=t.uint8, device=device())
    return _ws.buf.data_ptr(), _ws.buf.numel()


class _Branch(threading.local):
    """A forward branch issued on a second stream (graph.forward)."""

    def __init__(self):
        self.stream = None
        self.buf = None
        self.active = False
        self.pending = False


_branch = _Branch()


def _branch_workspace(nbytes: int):
    t = torch()
    nbytes = int(max(nbytes, 1 << 20))
    if _branch.buf is None or _branch.buf.numel() < nbytes:
        if _branch.buf is not None:
            _branch.stream.synchronize()  # the old buffer is idle before it is freed
        _branch.buf = t.empty(nbytes + (nbytes >> 2), dtype=t.uint8, device=device())
    return _branch.buf.data_ptr(), _branch.buf.numel()


@contextlib.contextmanager
def branch_scope():
    """Issue the enclosed work on the branch stream, ordered after everything
    issued so far on the current stream; `branch_join()` later makes the
    current stream wait for it."""
    t = torch()
    cur = t.cuda.current_stream()
    if _branch.stream is None:
        _branch.stream = t.cuda.Stream()
    _branch.stream.wait_stream(cur)
    _branch.active = True
    try:
        with t.cuda.stream(_branch.stream):
            yield
    finally:
        _branch.active = False
        _branch.pending = True


def branch_join() -> None:
    if _branch.pending:
        torch().cuda.current_stream().wait_stream(_branch.stream)
        _branch.pending = False


class _Side(threading.local):
    """The weight-gradient stream of the engine's backward loop (per thread)."""

    def __init__(self):
        self.stream = None
        self.buf = None
        self.allowed = False
        self.pending = False


_side = _Side()


def side_begin(allowed: bool) -> None:
    """Open a backward pass whose weight gradients may run on the side stream
    (graph.backward; NNL_WG_STREAM=0 keeps everything on the current stream)."""
    _side.allowed = bool(allowed) and os.environ.get("NNL_WG_STREAM", "1") != "0"
    _side.pending = False


def side_fork():
    """Raw handle of the side stream, ordered after everything issued so far on
    the current stream; None outside an engine backward pass."""
    if not _side.allowed:
        return None
    t = torch()
    if _side.stream is None:
        _side.stream = t.cuda.Stream()
    _side.stream.wait_stream(t.cuda.current_stream())
    _side.pending = True
    return _side.stream.cuda_stream


def wait_aux(stream) -> None:
    """Make `stream` wait for the side (weight-gradient) and branch streams
    where they have pending work: a gradient bucket issued on the
    communication stream may hold gradients either produced."""
    if _side.pending and _side.stream is not None:
        stream.wait_stream(_side.stream)
    if _branch.pending and _branch.stream is not None:
        stream.wait_stream(_branch.stream)


def side_end() -> None:
    """Join the side stream into the current stream (before the optimizer
    reads the weight gradients) and close the pass."""
    if _side.pending:
        torch().cuda.current_stream().wait_stream(_side.stream)
    _side.pending = False
    _side.allowed = False


def side_workspace(nbytes: int):
    """The side stream's own scratch buffer (kernels on it run concurrently
    with the shared workspace's users).  Growth waits for the side stream so
    the old buffer is idle when it is freed; sizes settle in the first step,
    before any CUDA-graph capture."""
    t = torch()
    nbytes = int(max(nbytes, 1 << 20))
    if _side.buf is None or _side.buf.numel() < nbytes:
        if _side.buf is not None and _side.stream is not None:
            _side.stream.synchronize()
        _side.buf = t.empty(nbytes + (nbytes >> 2), dtype=t.uint8, device=device())
    return _side.buf.data_ptr(), _side.buf.numel()


def reserve_workspace(nbytes: int) -> None:
    workspace(nbytes)
