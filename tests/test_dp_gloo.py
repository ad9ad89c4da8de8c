"""world_size-2 CPU (gloo) test of the multi-process gradient exchange.

Each rank computes the oracle LeNet gradients of its contiguous shard
(communicator.py:216-218), packs them into f32 buckets with the package's
bucket planner, sums them with a real torch.distributed all_reduce, and
applies the unpack rule q(sum / f32(world)).  The result must equal the
reference's rank-ordered fold (communicator.py:99-105) bit for bit (for two
ranks the f32 sum is order-independent), and both ranks must agree.
"""

import os
import socket

import numpy as np
import pytest


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank_main(rank, world, port, out_q):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import torch
    import torch.distributed as dist
    from oracle import nnl_oracle as O
    from paper_2102_06725_b200.communicator import bucket_layout, plan_buckets

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        B = 8
        x = O.uniform(1, 0, (B, 1, 28, 28), 0, 1)
        lab = (np.arange(B) % 10).astype(np.float32)
        shard = B // world
        m = O.Model(0, half=True)
        xv = O.Var(x[rank * shard:(rank + 1) * shard], half=True)
        tv = O.Var(lab[rank * shard:(rank + 1) * shard], half=True)
        loss = m.sce(O.lenet(m, xv, 10), tv)
        O.backward(loss, 8.0)
        names = list(m.trainable())
        grads = [m.trainable()[k].grad for k in names]
        halves = [m.trainable()[k].half for k in names]
        sizes = [g.size for g in grads]
        result = [None] * len(grads)
        for group in plan_buckets(sizes, bucket_bytes=4096):
            offs = bucket_layout([sizes[i] for i in group])
            bucket = np.zeros(sum(sizes[i] for i in group), np.float32)
            for j, i in enumerate(group):
                bucket[offs[j]:offs[j] + sizes[i]] = grads[i].ravel()
            t = torch.from_numpy(bucket)
            dist.all_reduce(t)
            mean = t.numpy() / np.float32(world)
            for j, i in enumerate(group):
                v = mean[offs[j]:offs[j] + sizes[i]].reshape(grads[i].shape)
                result[i] = O.q16(v) if halves[i] else v
        out_q.put((rank, [r.copy() for r in result], [g.copy() for g in grads]))
    finally:
        dist.destroy_process_group()


def test_bucket_planner_covers_every_buffer_in_order():
    from paper_2102_06725_b200.communicator import bucket_layout, plan_buckets
    sizes = [10, 1000, 3, 5000, 7, 7, 9000]
    groups = plan_buckets(sizes, 4 * 1000)
    assert [i for g in groups for i in g] == list(range(len(sizes)))
    assert all(sum(sizes[i] for i in g) * 4 >= 4000 for g in groups[:-1])
    assert bucket_layout([3, 4, 5]) == [0, 3, 7]


def test_gloo_world2_mean_allreduce_matches_reference_fold():
    import torch.multiprocessing as mp
    from oracle import nnl_oracle as O
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(2):
        rank, reduced, local = q.get(timeout=240)
        res[rank] = (reduced, local)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = O.fold_mean([res[0][1], res[1][1]], [True] * len(res[0][1]))
    for a, b, w in zip(res[0][0], res[1][0], want):
        assert np.array_equal(a, b)           # replicas agree bitwise
        assert np.array_equal(a, w)           # == reference fold, bitwise


def _overlap_rank_main(rank, world, port, out_q):
    """Buckets released by BucketSchedule as gradients turn final (reverse
    creation order, the order backward finishes them) and reduced one by one
    with a real all_reduce; the leftovers go after "backward"."""
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import torch
    import torch.distributed as dist
    from oracle import nnl_oracle as O
    from paper_2102_06725_b200.communicator import BucketSchedule, bucket_layout

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        B = 8
        x = O.uniform(1, 0, (B, 1, 28, 28), 0, 1)
        lab = (np.arange(B) % 10).astype(np.float32)
        shard = B // world
        m = O.Model(0, half=True)
        xv = O.Var(x[rank * shard:(rank + 1) * shard], half=True)
        tv = O.Var(lab[rank * shard:(rank + 1) * shard], half=True)
        loss = m.sce(O.lenet(m, xv, 10), tv)
        O.backward(loss, 8.0)
        names = list(m.trainable())[::-1]          # readiness order
        grads = [m.trainable()[k].grad for k in names]
        halves = [m.trainable()[k].half for k in names]
        sizes = [g.size for g in grads]
        sched = BucketSchedule(sizes, bucket_bytes=8192)
        result = [None] * len(grads)
        issued = []

        def issue(b):
            group = sched.groups[b]
            offs = bucket_layout([sizes[i] for i in group])
            bucket = np.zeros(sum(sizes[i] for i in group), np.float32)
            for j, i in enumerate(group):
                bucket[offs[j]:offs[j] + sizes[i]] = grads[i].ravel()
            t = torch.from_numpy(bucket)
            dist.all_reduce(t)
            mean = t.numpy() / np.float32(world)
            for j, i in enumerate(group):
                assert result[i] is None                 # each buffer exactly once
                v = mean[offs[j]:offs[j] + sizes[i]].reshape(grads[i].shape)
                result[i] = O.q16(v) if halves[i] else v
            issued.append(b)

        # the last buffer is "never reached" by backward: it drains at the end
        for i in range(len(grads) - 1):
            for b in sched.ready(i):
                issue(b)
            assert sched.ready(i) == []                  # a second report is a no-op
        for b in sched.drain():
            issue(b)
        assert sorted(issued) == list(range(len(sched.groups)))
        out_q.put((rank, issued, [r.copy() for r in result], [g.copy() for g in grads]))
    finally:
        dist.destroy_process_group()


def test_bucket_schedule_releases_in_order():
    from paper_2102_06725_b200.communicator import BucketSchedule
    s = BucketSchedule([10, 1000, 3, 5000, 7], 4 * 1000)
    assert s.groups == [[0, 1], [2, 3], [4]]
    assert s.ready(2) == [] and s.ready(0) == [] and s.ready(3) == [1]
    assert s.ready(1) == [0] and s.drain() == [2] and s.drain() == []
    s.reset()
    assert s.ready(4) == [2] and s.drain() == [0, 1]


def test_gloo_world2_overlapped_buckets_match_reference_fold():
    import torch.multiprocessing as mp
    from oracle import nnl_oracle as O
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_overlap_rank_main, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(2):
        rank, issued, reduced, local = q.get(timeout=240)
        res[rank] = (issued, reduced, local)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res[0][0] == res[1][0]                  # same collective order on every rank
    want = O.fold_mean([res[0][2], res[1][2]], [True] * len(res[0][2]))
    for a, b, w in zip(res[0][1], res[1][1], want):
        assert np.array_equal(a, b)
        assert np.array_equal(a, w)
