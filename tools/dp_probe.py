#!/usr/bin/env python
"""The data-parallel ResNet-50 step through the NCCL path with the bucketed
all-reduce overlapped with backward, at the world size torchrun gives (world 1
forced onto the process-group path): eager step time (device, max over ranks)
vs the same trainer without the collective.

    torchrun --nproc-per-node N tools/dp_probe.py [--steps 5] [--bucket-mb 8]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--bucket-mb", type=int, default=8)
    ap.add_argument("--batch", type=int, default=256)
    args = ap.parse_args()
    import torch
    import torch.distributed as dist
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    world, rank = dist.get_world_size(), dist.get_rank()
    import paper_2102_06725_b200 as nn
    import paper_2102_06725_b200.functions as F
    from paper_2102_06725_b200 import networks
    from paper_2102_06725_b200.communicator import DataParallelTrainer
    nn.set_default_context(nn.ExecutionContext(type_config=nn.TypeConfig.HALF))
    B = args.batch

    def build(bs):
        xv = nn.Variable((bs, 3, 224, 224))
        tv = nn.Variable((bs,))
        return {"x": xv, "label": tv,
                "loss": F.softmax_cross_entropy(networks.resnet50(xv, 1000), tv)}

    out = {"n_gpus": world, "batch_per_gpu": B, "bucket_mb": args.bucket_mb}
    for forced in (True, False):
        if not forced and world > 1:
            continue
        tr = DataParallelTrainer(world, B * world, build, lr=0.1, seed=0,
                                 loss_scaling=nn.DynamicLossScaler(8.0, 2.0, 2000),
                                 check_sync=False, momentum=0.9, weight_decay=1e-4,
                                 bucket_bytes=args.bucket_mb << 20, distributed=forced)
        rep = tr.rank0
        rep.handles["x"].data.write_f32_device(
            nn.RngState(1, counter=rank * B * 3 * 224 * 224).next_uniform_device((B, 3, 224, 224)))
        import numpy as np
        rep.handles["label"].d = ((np.arange(B) + rank * B) % 1000).astype(np.float32)
        for _ in range(3):
            tr.step_resident()
        torch.cuda.synchronize()
        dist.barrier()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(args.steps):
            tr.step_resident()
        e.record()
        torch.cuda.synchronize()
        t = torch.tensor([s.elapsed_time(e) / args.steps], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        key = "ms_per_step_nccl_overlap" if forced else "ms_per_step_local_eager"
        out[key] = round(float(t.item()), 3)
        if forced:
            out["buckets"] = len(rep._overlap.plans)
    if rank == 0:
        print(json.dumps(out), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
