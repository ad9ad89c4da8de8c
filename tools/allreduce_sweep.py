#!/usr/bin/env python
"""Gradient all_reduce bucket sweep (BASELINE.json config 5).

    python -m torch.distributed.run --nproc-per-node K --master-addr 127.0.0.1 \
        tools/allreduce_sweep.py [--min-mb 1] [--max-mb 1024] [--iters 20]

Per bucket size S (1 MB .. 1 GB of fp16 gradient, doubling) and per mode:

  nccl   fp16 buffer summed in place by NCCL, then q(sum / f32(K)) by torch
         (what a naive fp16 all-reduce does; partial sums can overflow where
         the reference's f32 fold does not)
  bucket the package's path (communicator.BucketPlan): nnl_bucket_pack to
         f32, NCCL f32 sum, nnl_bucket_unpack_mean (q(sum / f32(K)) + the
         overflow flag) -- the kernels the trainer runs per bucket

Values are RngState(seed=rank).next_uniform(n, -1, 1) rounded to fp16.  Each
timing is the max over ranks of the median of --iters CUDA-event-timed calls;
busbw = S * 2(K-1)/K / t (nccl-tests convention) against the 900 GB/s NVLink 5
per-direction peak.  Rank 0 prints one JSON line per (mode, size).
"""

import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

NVLINK_GBS = 900.0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--min-mb", type=int, default=1)
    ap.add_argument("--max-mb", type=int, default=1024)
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    args = ap.parse_args()

    import torch
    import torch.distributed as dist
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank, world = dist.get_rank(), dist.get_world_size()

    import paper_2102_06725_b200 as nn
    from paper_2102_06725_b200.communicator import BucketPlan
    from paper_2102_06725_b200.tensor import NdArray, Dtype

    def timed(fn) -> float:
        for _ in range(args.warmup):
            fn()
        ts = []
        for _ in range(args.iters):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            dist.barrier()
            s.record()
            fn()
            e.record()
            torch.cuda.synchronize()
            ts.append(s.elapsed_time(e))
        t = torch.tensor([statistics.median(ts)], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    mb = args.min_mb
    while mb <= args.max_mb:
        n = mb * (1 << 20) // 2
        vals = nn.RngState(rank).next_uniform_device((n,), -1.0, 1.0)
        half = vals.to(torch.float16)
        buf = half.clone()
        inv = 1.0 / world

        def plain():
            buf.copy_(half)
            dist.all_reduce(buf)
            buf.mul_(inv)

        grad = NdArray((n,), Dtype.F16)
        grad.write_f32_device(vals)
        plan = BucketPlan([grad])
        stream = torch.cuda.current_stream().cuda_stream

        def bucket():
            plan.pack(stream)
            dist.all_reduce(plan.bucket)
            plan.unpack_mean(plan.bucket.data_ptr(), world, None, stream)

        for mode, fn in (("nccl", plain), ("bucket", bucket)):
            ms = timed(fn)
            size = n * 2
            bus = size * 2 * (world - 1) / world / (ms / 1e3) / 1e9 if world > 1 else 0.0
            if rank == 0:
                print(json.dumps({"mode": mode, "bytes": size, "n_gpus": world,
                                  "ms": round(ms, 4), "busbw_gbs": round(bus, 1),
                                  "frac_nvlink": round(bus / NVLINK_GBS, 4)}), flush=True)
        del vals, half, buf, grad, plan
        torch.cuda.empty_cache()
        mb *= 2
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
