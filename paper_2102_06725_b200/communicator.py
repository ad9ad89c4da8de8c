"""Data-parallel gradient exchange (reference src/communicator.py).

Two transports behind the reference API (``Communicator.all_reduce(buffers,
division)``, ``barrier``, ``rank``, ``n_workers``):

* ``DataParallelCommunicator`` — one process per GPU (the paper's
  ``MultiProcessDataParalellCommunicator``).  Gradients are
  packed by ``nnl_bucket_pack`` into float32 buckets (the reference folds in
  f32, communicator.py:99-103, so fp16 partial sums that overflow where the
  reference does not are avoided), summed with NCCL over NVLink via
  ``torch.distributed``, and unpacked by ``nnl_bucket_unpack_mean`` which
  divides by f32(n), rounds once into the gradient storage and ORs the
  overflow flag.  Buckets are issued as soon as their last gradient is
  final (``BucketedAllReduce``), on a communication stream.
* ``CommunicatorGroup`` — K ranks as threads of one process sharing one
  GPU, exact to the reference's rank-ordered fold (``nnl_fold_f32``).  It is
  the drop-in for the reference's simulated trainer and the K-replica parity
  tests.
"""

from __future__ import annotations

import ctypes as C
import hashlib
import threading
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .errors import (CollectiveTimeout, DivergedReplicas, InvalidWorkerCount, ShapeMismatch,
                     ShapeMismatchAcrossRanks)
from .graph import Variable, _note_host_values
from .parameters import ParameterRegistry, registry_scope
from .solver import (DeviceLossScaler, DynamicLossScaler, SgdSolver, _device_table,
                     build_chunks, dynamic_step)
from .tensor import NdArray

__all__ = ["Communicator", "CommunicatorGroup", "DataParallelCommunicator",
           "MultiProcessDataParalellCommunicator", "MultiProcessDataParallelCommunicator",
           "DataParallelTrainer", "data_parallel_step", "BucketPlan"]


def plan_buckets(sizes: list[int], bucket_bytes: int) -> list[list[int]]:
    """Group consecutive buffers (in list order) into f32 buckets of at least
    `bucket_bytes` (the last may be smaller).  Pure host logic, shared by the
    NCCL path and the gloo tests."""
    groups, cur, size = [], [], 0
    for i, n in enumerate(sizes):
        cur.append(i)
        size += int(n) * 4
        if size >= bucket_bytes:
            groups.append(cur)
            cur, size = [], 0
    if cur:
        groups.append(cur)
    return groups


def bucket_layout(sizes: list[int]) -> list[int]:
    """Element offset of each buffer inside its f32 bucket (concatenation)."""
    offs, o = [], 0
    for n in sizes:
        offs.append(o)
        o += int(n)
    return offs


class BucketPlan:
    """Packing of a list of gradient NdArrays into one f32 device bucket
    (``pad_to``: bucket elements, >= the packed total; the exact all-reduce
    needs a multiple of the world size)."""

    def __init__(self, arrays: list[NdArray], slot_base=None, pad_to: int = 0):
        t = _lib.torch()
        self.arrays = list(arrays)
        self.total = sum(a.size for a in arrays)
        descs = [_lib.ParamSlot(None, a.ptr, None, None, a.size, a.code, 0) for a in arrays]
        chunks = build_chunks([a.size for a in arrays])
        pos = np.zeros(len(chunks), dtype=np.int64)
        offs = np.cumsum([0] + [a.size for a in arrays])
        for i, ch in enumerate(chunks):
            pos[i] = offs[ch.slot] + ch.start
        self._slots = _device_table(descs)
        self._chunks = _device_table(chunks)
        self._pos = t.from_numpy(pos).to(_lib.device()) if len(pos) else \
            t.zeros(1, dtype=t.int64, device=_lib.device())
        self.n_chunks = len(chunks)
        self.bucket = t.empty(max(self.total, pad_to, 1), dtype=t.float32, device=_lib.device())
        self.signature = tuple((a.shape, a.dtype.value) for a in arrays)

    def pack(self, stream: int) -> None:
        _lib.call("nnl_bucket_pack", self._slots.data_ptr(), self._chunks.data_ptr(),
                  self._pos.data_ptr(), self.n_chunks, self.bucket.data_ptr(), stream)

    def tables(self):
        return (self._slots.data_ptr(), self._chunks.data_ptr(), self._pos.data_ptr(),
                self.n_chunks)

    def unpack_mean(self, src_ptr: int, world: int, nonfinite_ptr, stream: int) -> None:
        _lib.call("nnl_bucket_unpack_mean", self._slots.data_ptr(), self._chunks.data_ptr(),
                  self._pos.data_ptr(), self.n_chunks, src_ptr, world, nonfinite_ptr, stream)
        for a in self.arrays:
            a.mark_set()


# ---------------------------------------------------------------------------
# in-process thread group (reference-exact fold)

class _SharedState:
    def __init__(self, n: int, timeout: float):
        self.n = n
        self.timeout = timeout
        self.barrier = threading.Barrier(n)
        self.slots: list = [None] * n
        self.error: Exception | None = None
        self.plans: dict = {}


class Communicator:
    """One rank's view of an in-process worker group."""

    def __init__(self, rank: int, state: _SharedState):
        self.rank = rank
        self.n_workers = state.n
        self._state = state

    def _wait(self) -> None:
        try:
            self._state.barrier.wait(timeout=self._state.timeout)
        except threading.BrokenBarrierError:
            raise CollectiveTimeout(
                f"rank {self.rank}: a peer failed to join within {self._state.timeout}s"
            ) from None

    def barrier(self) -> None:
        self._wait()

    def all_reduce(self, buffers: list[NdArray], division: bool = False) -> None:
        st = self._state
        st.slots[self.rank] = list(buffers)
        self._wait()
        if self.rank == 0:
            try:
                self._reduce(division)
            except Exception as exc:
                st.error = exc
        self._wait()
        err = st.error
        self._wait()
        if self.rank == 0:
            st.error = None
            st.slots = [None] * st.n
        if err is not None:
            raise type(err)(str(err))

    def _reduce(self, division: bool) -> None:
        st = self._state
        counts = {len(s) for s in st.slots}
        if len(counts) != 1:
            raise ShapeMismatchAcrossRanks(f"buffer counts differ across ranks: {sorted(counts)}")
        for i in range(counts.pop()):
            shapes = {s[i].shape for s in st.slots}
            if len(shapes) != 1:
                raise ShapeMismatchAcrossRanks(f"buffer {i} shapes differ: {sorted(shapes)}")
        key = tuple(tuple(a.ptr for a in s) for s in st.slots)
        plans = st.plans.get(key)
        t = _lib.torch()
        if plans is None:
            plans = [BucketPlan(s) for s in st.slots]
            ptrs = t.tensor([p.bucket.data_ptr() for p in plans], dtype=t.int64,
                            device=_lib.device())
            acc = t.empty_like(plans[0].bucket)
            plans = (plans, ptrs, acc)
            st.plans[key] = plans
        plist, ptrs, acc = plans
        stream = _lib.stream()
        for p in plist:
            p.pack(stream)
        # acc = r0 + r1 + ... in ascending rank order (communicator.py:99-102)
        _lib.call("nnl_fold_f32", st.n, ptrs.data_ptr(), plist[0].total, acc.data_ptr(), stream)
        world = st.n if division else 1
        for p in plist:
            p.unpack_mean(acc.data_ptr(), world, None, stream)


class CommunicatorGroup:
    def __init__(self, n_workers: int, timeout: float = 60.0):
        if n_workers < 1:
            raise InvalidWorkerCount(f"need at least one worker, got {n_workers}")
        self.n_workers = n_workers
        self._shared = _SharedState(n_workers, timeout)
        self.communicators = [Communicator(r, self._shared) for r in range(n_workers)]

    def run(self, fn) -> list:
        results: list = [None] * self.n_workers
        failures: list = [None] * self.n_workers
        dev = _lib.torch().cuda.current_device() if _lib.torch().cuda.is_available() else None

        def target(rank: int):
            try:
                if dev is not None:
                    _lib.torch().cuda.set_device(dev)
                results[rank] = fn(self.communicators[rank])
            except Exception as exc:  # noqa: BLE001 - re-raised below
                failures[rank] = exc
                self._shared.barrier.abort()

        threads = [threading.Thread(target=target, args=(r,), name=f"worker-{r}")
                   for r in range(self.n_workers)]
        for th in threads:
            th.start()
        for th in threads:
            th.join()
        self._shared.barrier.reset()
        root = [e for e in failures if e is not None and not isinstance(e, CollectiveTimeout)]
        if root:
            raise root[0]
        for exc in failures:
            if exc is not None:
                raise exc
        return results


# ---------------------------------------------------------------------------
# multi-process transport: libnnl's NCCL communicator (nnl_comm_*)

COMM_MODES = {"nccl": 0, "exact": 1}


class NcclComm:
    """Owner of one ``nnl_comm`` handle (include/nnl.h): NCCL over NVLink,
    driven entirely from libnnl on the caller's stream.  torch.distributed is
    only the rendezvous: it broadcasts rank 0's ncclUniqueId."""

    def __init__(self, dist, group, rank: int, world: int, mode: str):
        t = _lib.torch()
        self.mode = mode
        idbuf = t.zeros(128, dtype=t.uint8, device=_lib.device())
        if rank == 0:
            raw = (C.c_uint8 * 128)()
            _lib.call("nnl_comm_unique_id", raw)
            idbuf.copy_(t.frombuffer(bytearray(bytes(raw)), dtype=t.uint8))
        src = dist.get_global_rank(group, 0) if group is not None else 0
        dist.broadcast(idbuf, src=src, group=group)
        uid = (C.c_uint8 * 128).from_buffer_copy(bytes(idbuf.cpu().numpy()))
        handle = C.c_void_p()
        _lib.call("nnl_comm_init", C.byref(handle), world, rank, uid, COMM_MODES[mode])
        self.handle = handle

    def bucket_elems(self, n: int) -> int:
        return int(_lib.lib().nnl_comm_bucket_elems(self.handle, n))

    def allreduce_mean(self, plan: "BucketPlan", divide: bool, nonfinite_ptr, stream: int,
                       ws=None) -> None:
        nbytes = int(_lib.lib().nnl_comm_workspace_size(self.handle, plan.total))
        wp = ws.data_ptr() if ws is not None else None
        if nbytes and (ws is None or ws.numel() < nbytes):
            raise ValueError("exact all-reduce workspace too small")
        _lib.call("nnl_comm_allreduce_mean", self.handle, *plan.tables(), plan.bucket.data_ptr(),
                  plan.total, 1 if divide else 0, nonfinite_ptr, wp, nbytes, stream)
        for a in plan.arrays:
            a.mark_set()

    def allreduce_sum_f32(self, tensor, stream: int) -> None:
        _lib.call("nnl_comm_allreduce_sum_f32", self.handle, tensor.data_ptr(), tensor.numel(),
                  stream)

    def workspace(self, n: int):
        nbytes = int(_lib.lib().nnl_comm_workspace_size(self.handle, n))
        if not nbytes:
            return None
        t = _lib.torch()
        return t.empty(nbytes, dtype=t.uint8, device=_lib.device())

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            try:
                _lib.lib().nnl_comm_destroy(h)
            except Exception:  # noqa: BLE001 - interpreter shutdown
                pass
            self.handle = None


class DataParallelCommunicator:
    """One rank per process (paper Listing 3, MultiProcessDataParalellCommunicator).

    Over an NCCL process group the exchange is libnnl's communicator
    (``NcclComm``: pack + ncclAllReduce / rank-ordered exact fold + unpack in
    one C call, CUDA-graph capturable); over gloo (CPU hosts, or several
    ranks sharing one GPU in tests) the f32 bucket goes through
    torch.distributed.  ``mode="exact"`` reproduces the reference's ascending
    rank-order fold bit for bit (communicator.py:99-103) on either backend."""

    def __init__(self, group=None, bucket_bytes: int = 32 << 20, mode: str | None = None):
        import os

        import torch.distributed as dist
        if not dist.is_initialized():
            raise InvalidWorkerCount("torch.distributed is not initialised")
        self._dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.n_workers = dist.get_world_size(group)
        self.bucket_bytes = bucket_bytes
        self.mode = mode or os.environ.get("NNL_COMM_MODE", "nccl")
        if self.mode not in COMM_MODES:
            raise ValueError(f"unknown communicator mode {self.mode!r}")
        self.backend = dist.get_backend(group)
        self.nccl = (NcclComm(dist, group, self.rank, self.n_workers, self.mode)
                     if self.backend == "nccl" else None)
        self._plans: dict = {}
        self._checked: set = set()
        self._ws = None

    @property
    def capturable(self) -> bool:
        """The exchange is stream-ordered (no host synchronisation)."""
        return self.nccl is not None

    def pad_to(self, n: int) -> int:
        return self.nccl.bucket_elems(n) if self.nccl is not None else n

    def exchange(self, plan: "BucketPlan", divide: bool, nonfinite_ptr, stream: int) -> None:
        """pack -> sum over ranks -> unpack q(sum / f32(n)) for one bucket."""
        if self.nccl is not None:
            need = int(_lib.lib().nnl_comm_workspace_size(self.nccl.handle, plan.total))
            if need and (self._ws is None or self._ws.numel() < need):
                self._ws = self.nccl.workspace(plan.total)
            self.nccl.allreduce_mean(plan, divide, nonfinite_ptr, stream, self._ws)
            return
        t = _lib.torch()
        world = self.n_workers if divide else 1
        plan.pack(stream)
        if self.mode == "exact":  # gather every rank's bucket, fold in rank order
            parts = [t.empty_like(plan.bucket) for _ in range(self.n_workers)]
            self._dist.all_gather(parts, plan.bucket, group=self.group)
            ptrs = t.tensor([q.data_ptr() for q in parts], dtype=t.int64, device=_lib.device())
            _lib.call("nnl_fold_f32", self.n_workers, ptrs.data_ptr(), plan.total,
                      plan.bucket.data_ptr(), stream)
            t.cuda.current_stream().synchronize()  # `parts`/`ptrs` die with this frame
        else:
            self._dist.all_reduce(plan.bucket, group=self.group)
        plan.unpack_mean(plan.bucket.data_ptr(), world, nonfinite_ptr, stream)

    def allreduce_sum_f32(self, tensor) -> None:
        if self.nccl is not None:
            self.nccl.allreduce_sum_f32(tensor, _lib.stream())
        else:
            self._dist.all_reduce(tensor, group=self.group)

    def barrier(self) -> None:
        self._dist.barrier(group=self.group)

    def _validate(self, signature) -> None:
        if signature in self._checked:
            return
        h = hashlib.sha256(repr(signature).encode()).digest()[:8]
        t = _lib.torch()
        mine = t.tensor([int.from_bytes(h, "little", signed=True)], dtype=t.int64,
                        device=_lib.device())
        allv = [t.empty_like(mine) for _ in range(self.n_workers)]
        self._dist.all_gather(allv, mine, group=self.group)
        if len({int(v.item()) for v in allv}) != 1:
            raise ShapeMismatchAcrossRanks("buffer lists differ across ranks")
        self._checked.add(signature)

    def plan(self, buffers: list[NdArray]) -> list[BucketPlan]:
        key = tuple(a.ptr for a in buffers)
        plans = self._plans.get(key)
        if plans is None:
            groups = plan_buckets([a.size for a in buffers], self.bucket_bytes)
            plans = []
            for g in groups:
                arrs = [buffers[i] for i in g]
                plans.append(BucketPlan(arrs, pad_to=self.pad_to(sum(a.size for a in arrs))))
            self._plans[key] = plans
        return plans

    def all_reduce(self, buffers: list[NdArray], division: bool = False,
                   nonfinite_ptr=None) -> None:
        """Reference API (communicator.py:69-105): every rank's buffers become
        the (mean, with division) sum over the ranks, rounded once."""
        self._validate(tuple((a.shape, a.dtype.value) for a in buffers))
        stream = _lib.stream()
        for p in self.plan(buffers):
            self.exchange(p, division, nonfinite_ptr, stream)


class BucketSchedule:
    """Which gradient buckets become complete as gradients turn final.

    Pure host logic (shared by the NCCL path and the gloo tests).  Buffers are
    grouped in the order their gradients are expected to become final
    (reverse creation order), ``plan_buckets`` style; ``ready(i)`` marks buffer
    i final and returns the buckets it completes, ``drain()`` the ones never
    completed (issued after backward).  Every rank derives the same schedule
    from the same graph, so collectives are issued in the same order
    everywhere (an NCCL requirement)."""

    def __init__(self, sizes: list[int], bucket_bytes: int):
        self.groups = plan_buckets(sizes, bucket_bytes)
        self.bucket_of = {i: b for b, g in enumerate(self.groups) for i in g}
        self.reset()

    def reset(self) -> None:
        self.left = [len(g) for g in self.groups]
        self.issued = [False] * len(self.groups)
        self.seen: set[int] = set()

    def ready(self, i: int) -> list[int]:
        if i in self.seen:
            return []
        self.seen.add(i)
        b = self.bucket_of[i]
        self.left[b] -= 1
        if self.left[b] == 0 and not self.issued[b]:
            self.issued[b] = True
            return [b]
        return []

    def drain(self) -> list[int]:
        out = [b for b in range(len(self.groups)) if not self.issued[b]]
        for b in out:
            self.issued[b] = True
        return out


class BucketedAllReduce:
    """Gradient all_reduce overlapped with backward.

    Parameters are bucketed in reverse creation order.  ``ready(v)`` (wired to
    ``backward(on_grad_ready=...)``) is called when v's gradient is final; when
    it completes a bucket, the communication stream waits for the compute
    stream at that point, packs the bucket (f32), runs the NCCL sum and
    unpacks q(sum / f32(n)) into the gradients, ORing the overflow flag —
    while backward continues on the compute stream.  ``finish()`` issues
    what is left and makes the compute stream wait for the communication
    stream (the update reads the reduced gradients)."""

    def __init__(self, comm: "DataParallelCommunicator", params: list[Variable],
                 nonfinite_ptr=None, bucket_bytes: int = 8 << 20):
        t = _lib.torch()
        self.comm = comm
        self.order = list(reversed(params))
        self.index = {id(p): i for i, p in enumerate(self.order)}
        self.schedule = BucketSchedule([p.grad.size for p in self.order], bucket_bytes)
        self.plans = []
        for g in self.schedule.groups:
            arrs = [self.order[i].grad for i in g]
            self.plans.append(BucketPlan(arrs, pad_to=comm.pad_to(sum(a.size for a in arrs))))
        self.nonfinite_ptr = nonfinite_ptr
        self.stream = t.cuda.Stream()
        self.world = comm.n_workers
        comm._validate(tuple((p.grad.shape, p.grad.dtype.value) for p in self.order))

    def begin(self) -> None:
        self.schedule.reset()

    def ready(self, v: Variable) -> None:
        i = self.index.get(id(v))
        if i is not None:
            for b in self.schedule.ready(i):
                self._issue(b)

    def _issue(self, b: int) -> None:
        t = _lib.torch()
        plan = self.plans[b]
        self.stream.wait_stream(t.cuda.current_stream())
        _lib.wait_aux(self.stream)  # gradients from the side / branch streams
        with t.cuda.stream(self.stream):
            self.comm.exchange(plan, True, self.nonfinite_ptr, _lib.stream())

    def finish(self) -> None:
        t = _lib.torch()
        for b in self.schedule.drain():
            self._issue(b)
        t.cuda.current_stream().wait_stream(self.stream)


MultiProcessDataParalellCommunicator = DataParallelCommunicator  # PAPER.md:88 spelling
MultiProcessDataParallelCommunicator = DataParallelCommunicator


# ---------------------------------------------------------------------------
# trainer (reference communicator.py:158-244)

@dataclass
class _Replica:
    registry: ParameterRegistry
    handles: dict[str, Variable]
    solver: SgdSolver
    scaler: DynamicLossScaler | None
    params: list[Variable] = field(default_factory=list)
    dscaler: DeviceLossScaler | None = None


def _wire_nonfinite(loss: Variable, params: list[Variable], flag_ptr: int) -> bool:
    """Point every param-gradient kernel at the scaler's overflow flag.

    Returns False if some trainable gradient is produced by a kind that does
    not report the flag (then the solver runs the explicit check pass)."""
    from .graph import _ancestors
    pids = {id(p) for p in params}
    covered: set[int] = set()
    for node in _ancestors(loss):
        hit = [v for v in node.inputs if id(v) in pids]
        if not hit:
            continue
        if node.kind not in ("Affine", "Convolution", "BatchNormalization"):
            return False
        node.state["nonfinite_ptr"] = flag_ptr
        if node.kind == "Convolution":
            # under the Convolution->BatchNormalization fusion (bias_by_bn) the
            # BN backward writes this convolution's bias gradient, so it must
            # flag overflow even when its own gamma/beta are frozen
            for c in node.outputs[0]._consumers:
                if c.kind == "BatchNormalization":
                    c.state["nonfinite_ptr"] = flag_ptr
        covered.update(id(v) for v in hit)
        if sum(1 for c in hit for cc in c._consumers) != len(hit):
            return False  # shared parameters: keep the explicit check
    return covered == pids


class PendingLoss:
    """Loss of a `step_async` step; `result()` waits for the step to finish."""

    __slots__ = ("_done", "_host", "_value")

    def __init__(self, done, host):
        self._done, self._host, self._value = done, host, None

    def result(self) -> float:
        if self._value is None:
            self._done.synchronize()
            self._value = float(self._host[0])
        return self._value


class DataParallelTrainer:
    """K lock-step replicas: shard the batch, mean-all-reduce grads, update.

    Same constructor and ``step`` as the reference.  Under torch.distributed
    (one process per GPU, world size == n_workers) each process holds one
    replica and gradients travel over NCCL; otherwise the K replicas are
    threads sharing the current GPU with the reference-exact in-process fold.

    ``step`` issues no host synchronisation except reading the loss back
    (the dynamic loss scale lives on the device).  Extensions: ``momentum``
    and ``weight_decay`` (NNabla Momentum SGD).
    """

    def __init__(self, n_workers: int, batch_size: int, build_fn, lr: float, seed: int,
                 loss_scaling=None, clip_norm: float | None = None, timeout: float = 60.0,
                 check_sync: bool = True, momentum: float = 0.0, weight_decay: float = 0.0,
                 bucket_bytes: int = 8 << 20, distributed: bool | None = None,
                 comm_mode: str | None = None):
        if n_workers < 1:
            raise InvalidWorkerCount(f"need at least one worker, got {n_workers}")
        if batch_size % n_workers != 0:
            raise InvalidWorkerCount(
                f"batch size {batch_size} not divisible by {n_workers} workers")
        import torch.distributed as dist
        # ``distributed=True`` forces the process-group path even at world
        # size 1 (tests the NCCL overlap path on a single GPU)
        up = dist.is_available() and dist.is_initialized()
        self.distributed = up and (dist.get_world_size() > 1 if distributed is None
                                   else bool(distributed))
        if self.distributed and dist.get_world_size() != n_workers:
            raise InvalidWorkerCount(
                f"n_workers={n_workers} but the process group has {dist.get_world_size()} ranks")
        self.n_workers = n_workers
        self.bucket_bytes = bucket_bytes
        self.batch_size = batch_size
        self.shard_size = batch_size // n_workers
        self.check_sync = check_sync
        self.static_scale = float(loss_scaling) if isinstance(loss_scaling, (int, float)) \
            and not isinstance(loss_scaling, bool) else None
        self.dynamic = isinstance(loss_scaling, DynamicLossScaler)
        self.replicas: list[_Replica] = []
        local = [dist.get_rank()] if self.distributed else list(range(n_workers))
        for _ in local:
            reg = ParameterRegistry(seed)
            with registry_scope(reg):
                handles = build_fn(self.shard_size)
            solver = SgdSolver(lr, clip_norm=clip_norm, momentum=momentum,
                               weight_decay=weight_decay).setup(reg.get_parameters())
            scaler = None
            dscaler = None
            if self.dynamic:
                scaler = DynamicLossScaler(loss_scaling.loss_scale, loss_scaling.scaling_factor,
                                           loss_scaling.interval, loss_scaling.counter)
                if clip_norm is None:
                    dscaler = DeviceLossScaler(scaler)
            rep = _Replica(reg, handles, solver, scaler, dscaler=dscaler)
            rep.params = list(reg.get_parameters().values())
            self.replicas.append(rep)
        self.ranks = local
        if self.distributed:
            self.comm = DataParallelCommunicator(mode=comm_mode)
            self.group = None
        else:
            self.comm = None
            self.group = CommunicatorGroup(n_workers, timeout)
        self._fused_flags = {}
        for rep in self.replicas:
            if rep.dscaler is not None:
                self._fused_flags[id(rep)] = _wire_nonfinite(rep.handles["loss"], rep.params,
                                                             rep.dscaler.nonfinite_ptr)

    @property
    def rank0(self) -> _Replica:
        return self.replicas[0]

    def _param_digest(self, rep: _Replica) -> bytes:
        h = hashlib.sha256()
        for p in rep.params:
            h.update(p.data.tobytes())
        return h.digest()

    def _overlap(self, rep: _Replica) -> "BucketedAllReduce":
        """The replica's bucketed all-reduce, issued from inside backward."""
        ov = getattr(rep, "_overlap", None)
        if ov is None:
            flag = rep.dscaler.nonfinite_ptr if rep.dscaler is not None else None
            ov = BucketedAllReduce(self.comm, rep.params, flag, self.bucket_bytes)
            rep._overlap = ov
        return ov

    def _work(self, rep: _Replica, rank: int, x_batch, label_batch, all_reduce) -> object:
        """One replica step.  ``all_reduce`` is a callable run after backward,
        or a ``BucketedAllReduce`` whose buckets are issued during backward."""
        lo = rank * self.shard_size
        if x_batch is not None:
            rep.handles["x"].d = x_batch[lo:lo + self.shard_size]
            rep.handles["label"].d = label_batch[lo:lo + self.shard_size]
        loss = rep.handles["loss"]
        loss.forward(clear_buffer=True)
        overlap = all_reduce if isinstance(all_reduce, BucketedAllReduce) else None
        hook = None
        if overlap is not None:
            overlap.begin()
            hook = overlap.ready
        if rep.dscaler is not None:
            seed = rep.dscaler.loss_scale_ptr
        elif rep.scaler is not None:
            seed = rep.scaler.loss_scale
        elif self.static_scale is not None:
            seed = self.static_scale
        else:
            seed = 1.0
        loss.backward(grad_seed=seed, clear_buffer=True, on_grad_ready=hook)
        if overlap is not None:
            overlap.finish()
        else:
            all_reduce(rep)
        if rep.dscaler is not None:
            rep.solver.dynamic_update(rep.dscaler, check=not self._fused_flags[id(rep)])
        elif rep.scaler is not None:
            dynamic_step(rep.scaler, rep.solver)
        elif self.static_scale is not None:
            rep.solver.scale_grad(1.0 / self.static_scale)
            rep.solver.clip_grad_by_norm()
            rep.solver.update()
        else:
            rep.solver.clip_grad_by_norm()
            rep.solver.update()
        return loss

    def _check_labels(self, rep: _Replica) -> None:
        """A replayed graph cannot raise from inside forward: surface the host
        label validation (`.d =` hook) before replay, as the reference raises
        LabelOutOfRange in forward (functions.py:337-339)."""
        from .errors import LabelOutOfRange
        for node in rep.handles["label"]._consumers:
            if node.state.get("labels_ok") is False:
                raise LabelOutOfRange(
                    f"labels must be integers in [0, {node.inputs[0].shape[1]})")

    def capture_graph(self) -> None:
        """Record one resident step into a CUDA graph; later `step_resident`
        calls replay it (removes the per-node launch overhead).

        Call after at least one warm-up step (all buffers, workspaces and
        tensor maps are then allocated at fixed addresses).  The warm-up run on
        the capture stream is a real training step on the resident batch.
        Under torch.distributed every rank calls this together: the recorded
        step contains the bucketed NCCL exchange issued from inside backward
        (libnnl's stream-ordered communicator), so N > 1 replays the same
        graph as N = 1.  Refused: several replicas in one process, the gloo
        transport, and the host-synchronous paths (clip_norm, host scaler)."""
        if self.n_workers != 1 and not self.distributed:
            raise NotImplementedError("graph capture needs one replica per process")
        if self.distributed and not self.comm.capturable:
            raise NotImplementedError(f"the {self.comm.backend} transport is host-synchronous")
        rep = self.replicas[0]
        if rep.dscaler is None and self.static_scale is None and rep.scaler is not None:
            raise NotImplementedError("host-synchronous loss scaling cannot be captured")
        t = _lib.torch()
        rank = self.ranks[0]
        reduce = self._overlap(rep) if self.distributed else (lambda r: None)
        side = t.cuda.Stream()
        side.wait_stream(t.cuda.current_stream())
        with t.cuda.stream(side):
            self._work(rep, rank, None, None, reduce)  # warm on the capture stream
        t.cuda.current_stream().wait_stream(side)
        g = t.cuda.CUDAGraph()
        before = _lib.lib().nnl_launch_count(0)
        with t.cuda.graph(g, stream=side):
            self._work(rep, rank, None, None, reduce)
        t.cuda.current_stream().wait_stream(side)
        self.graph_kernels = int(_lib.lib().nnl_launch_count(0) - before)  # libnnl kernels/step
        self._graph = g
        if getattr(self, "_feed", None) is not None:
            self._feed["graphs"] = [None, None]  # step_async re-records its I/O graphs

    def step_resident(self) -> None:
        """One step on the inputs already resident on the device: no host
        transfer and no loss read-back (the benchmark's device-side `value`)."""
        graph = getattr(self, "_graph", None)
        if graph is not None:
            graph.replay()
            return
        if self.distributed:
            rep = self.replicas[0]

            self._work(rep, self.ranks[0], None, None, self._overlap(rep))
        elif self.n_workers == 1:
            self._work(self.replicas[0], 0, None, None, lambda r: None)
        else:
            raise NotImplementedError("step_resident needs one replica per process")

    def save_checkpoint(self, path: str) -> None:
        """Parameters + solver masters/momentum + loss-scaler state of replica 0
        (all replicas are identical) in the NNP parameter.bin record format
        (checkpoint.py)."""
        from . import checkpoint
        rep = self.replicas[0]
        scaler = rep.dscaler if rep.dscaler is not None else rep.scaler
        checkpoint.save(path, rep.registry.get_parameters(grad_only=False), rep.solver, scaler)

    def load_checkpoint(self, path: str) -> None:
        """Restore `save_checkpoint` state into every replica, in place."""
        from . import checkpoint
        for rep in self.replicas:
            scaler = rep.dscaler if rep.dscaler is not None else rep.scaler
            checkpoint.load(path, rep.registry.get_parameters(grad_only=False), rep.solver,
                            scaler)

    def step_async(self, x_batch: np.ndarray, label_batch: np.ndarray) -> "PendingLoss":
        """Pipelined variant of `step` (extension, single process): the batch's
        host->device copy runs on a copy stream into one of two staging slots, so
        it overlaps the previous step's compute; the loss is read back
        asynchronously into pinned memory.  `PendingLoss.result()` waits for it.

        Same math as `step`: the device-side work of a step starts with the
        import of its inputs and ends with the loss read-back.  Pass pinned host
        arrays (e.g. `torch.empty(..., pin_memory=True).numpy()`) for an
        asynchronous copy.  After `capture_graph()`, each staging slot gets its
        own graph holding the input imports, the step and the loss export, so a
        step costs the host two copies, one replay and a read-back (the events
        and pinned loss slots are allocated once)."""
        if self.distributed or self.n_workers != 1:
            raise NotImplementedError("step_async is implemented for one replica per process")
        t = _lib.torch()
        rep = self.replicas[0]
        xv, lv = rep.handles["x"], rep.handles["label"]
        feed = getattr(self, "_feed", None)
        if feed is None:
            dev = _lib.device()
            feed = self._feed = {
                "stream": t.cuda.Stream(),
                "x": [t.empty(xv.shape, dtype=t.float32, device=dev) for _ in range(2)],
                "t": [t.empty(lv.shape, dtype=t.float32, device=dev) for _ in range(2)],
                "free": [t.cuda.Event() for _ in range(2)],   # slot's import consumed it
                "used": [False, False],
                "copied": [t.cuda.Event() for _ in range(2)],
                "slot": 0,
                "loss_dev": t.empty(1, dtype=t.float32, device=dev),
                # pinned loss slots + their events, reused round robin
                "host": [t.empty(1, dtype=t.float32, pin_memory=True) for _ in range(8)],
                "done": [t.cuda.Event() for _ in range(8)],
                "ring": 0,
                "graphs": [None, None],
            }
        x = np.asarray(x_batch, dtype=np.float32)[:self.shard_size]
        lab = np.asarray(label_batch, dtype=np.float32)[:self.shard_size]
        if x.shape != tuple(xv.shape) or lab.shape != tuple(lv.shape):
            raise ShapeMismatch(f"batch shapes {x.shape}/{lab.shape} != {xv.shape}/{lv.shape}")
        _note_host_values(lv, lab)  # label validation on the host, as `.d =` does
        slot = feed["slot"]
        feed["slot"] ^= 1
        cs, main = feed["stream"], t.cuda.current_stream()
        with t.cuda.stream(cs):
            if feed["used"][slot]:
                cs.wait_event(feed["free"][slot])
            hx, hl = t.from_numpy(np.ascontiguousarray(x)), t.from_numpy(np.ascontiguousarray(lab))
            feed["x"][slot].copy_(hx, non_blocking=hx.is_pinned())
            feed["t"][slot].copy_(hl, non_blocking=hl.is_pinned())
            feed["copied"][slot].record(cs)
        main.wait_event(feed["copied"][slot])
        graph = getattr(self, "_graph", None)
        if graph is not None:
            self._check_labels(rep)
            io = feed["graphs"][slot]
            if io is None:
                io = feed["graphs"][slot] = self._capture_io(rep, feed, slot)
            io.replay()
        else:
            self._import_and_export(rep, feed, slot, lambda: self._work(rep, 0, None, None,
                                                                          lambda r: None))
        feed["free"][slot].record(main)
        feed["used"][slot] = True
        k = feed["ring"]
        feed["ring"] = (k + 1) % len(feed["host"])
        host = feed["host"][k]
        host.copy_(feed["loss_dev"], non_blocking=True)
        done = feed["done"][k]
        done.record(main)
        return PendingLoss(done, host)

    def _import_and_export(self, rep, feed, slot, body) -> None:
        """The device part of one `step_async` step: import the staging slot's
        inputs, run `body` (the step), export the loss to `feed["loss_dev"]`."""
        rep.handles["x"].data.write_f32_device(feed["x"][slot])
        rep.handles["label"].data.write_f32_device(feed["t"][slot])
        body()
        loss = rep.handles["loss"]
        _lib.call("nnl_export_f32", loss.data.code, 1, 1, 1, loss.data.ptr,
                  feed["loss_dev"].data_ptr(), _lib.stream())

    def _capture_io(self, rep, feed, slot):
        """CUDA graph of `_import_and_export` for one staging slot (the step body
        recorded the same way as `capture_graph`)."""
        t = _lib.torch()
        side = t.cuda.Stream()
        side.wait_stream(t.cuda.current_stream())
        body = lambda: self._work(rep, 0, None, None, lambda r: None)  # noqa: E731
        # no warm-up run: capture_graph() already ran this step body, so every
        # buffer and workspace exists; recording executes nothing
        g = t.cuda.CUDAGraph()
        with t.cuda.graph(g, stream=side):
            self._import_and_export(rep, feed, slot, body)
        t.cuda.current_stream().wait_stream(side)
        return g

    def step(self, x_batch: np.ndarray, label_batch: np.ndarray, shard: bool = False) -> float:
        """One synchronised step; returns the batch loss (mean of shard losses).

        ``shard=True`` (extension): under torch.distributed the arrays are
        already this rank's shard, so no process materialises the global batch.
        """
        if self.distributed:
            rep = self.replicas[0]
            rank = self.ranks[0]
            if shard:
                xs, ls = x_batch, label_batch
            else:
                lo = rank * self.shard_size
                xs, ls = x_batch[lo:lo + self.shard_size], label_batch[lo:lo + self.shard_size]
            rep.handles["x"].d = xs
            rep.handles["label"].d = ls
            graph = getattr(self, "_graph", None)
            if graph is not None:  # the recorded step, buckets and NCCL included
                self._check_labels(rep)
                graph.replay()
                loss = rep.handles["loss"]
            else:
                loss = self._work(rep, rank, None, None, self._overlap(rep))
            t = _lib.torch()
            lv = t.empty(1, dtype=t.float32, device=_lib.device())
            _lib.call("nnl_export_f32", loss.data.code, 1, 1, 1, loss.data.ptr, lv.data_ptr(),
                      _lib.stream())
            self.comm.allreduce_sum_f32(lv)
            if self.check_sync and not shard:
                self._check_distributed(rep)
            return float(lv.item()) / self.n_workers
        if not self.distributed and self.n_workers == 1:
            graph = getattr(self, "_graph", None)
            if graph is not None:  # inputs through .d (H2D), then the recorded step
                rep = self.replicas[0]
                rep.handles["x"].d = x_batch[:self.shard_size]
                rep.handles["label"].d = label_batch[:self.shard_size]
                self._check_labels(rep)
                graph.replay()
                return float(rep.handles["loss"].d)
            loss = self._work(self.replicas[0], 0, x_batch, label_batch, lambda r: None)
            return float(loss.d)
        def work(comm: Communicator) -> float:
            rep = self.replicas[comm.rank]

            def ar(r):
                if self.n_workers > 1:
                    comm.all_reduce([p.grad for p in r.params], division=True)
                    if r.dscaler is not None and self._fused_flags[id(r)]:
                        # the fold rewrote every grad: recheck overflow on the mean
                        _lib.call("nnl_multi_nonfinite", *r.solver._args(),
                                  r.dscaler.nonfinite_ptr, _lib.stream())

            loss = self._work(rep, comm.rank, x_batch, label_batch, ar)
            return float(loss.d)

        losses = self.group.run(work)
        if self.check_sync and self.n_workers > 1:
            digests = {self._param_digest(r) for r in self.replicas}
            if len(digests) != 1:
                raise DivergedReplicas("parameter bytes differ across ranks after step")
        return float(np.mean(losses))

    def _check_distributed(self, rep: _Replica) -> None:
        t = _lib.torch()
        h = hashlib.sha256()
        for p in rep.params:
            h.update(p.data.raw_bytes())
        mine = t.tensor([int.from_bytes(h.digest()[:8], "little", signed=True)],
                        dtype=t.int64, device=_lib.device())
        allv = [t.empty_like(mine) for _ in range(self.n_workers)]
        self.comm._dist.all_gather(allv, mine)
        if len({int(v.item()) for v in allv}) != 1:
            raise DivergedReplicas("parameter bytes differ across ranks after step")


def data_parallel_step(trainer: DataParallelTrainer, x_batch, label_batch) -> float:
    return trainer.step(x_batch, label_batch)
