"""One rank of a world-2 data-parallel LeNet run (tests/test_comm_gpu.py).

Both ranks share cuda:0 and talk over gloo (NCCL refuses two ranks on one
GPU), so this drives the real DataParallelTrainer -> DataParallelCommunicator
-> BucketedAllReduce -> device bucket pack/unpack path at world size 2 and
writes the run's losses and final weights to $OUT (rank 0)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)


def main():
    import torch
    import torch.distributed as dist
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    half = os.environ["HALF"] == "1"
    mode = os.environ.get("MODE", "nccl")
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2102_06725_b200 as nn
    import paper_2102_06725_b200.functions as F
    from paper_2102_06725_b200 import networks
    from paper_2102_06725_b200.communicator import DataParallelTrainer
    g = dict(np.load(os.path.join(ROOT, "tests", "golden", "lenet.npz")))
    tc = nn.TypeConfig.HALF if half else nn.TypeConfig.FLOAT
    nn.set_default_context(nn.ExecutionContext(type_config=tc))

    def build(bs):
        xv = nn.Variable((bs, 1, 28, 28))
        tv = nn.Variable((bs,))
        return {"x": xv, "label": tv,
                "loss": F.softmax_cross_entropy(networks.lenet(xv, 10), tv)}

    tr = DataParallelTrainer(world, 16, build, lr=0.05, seed=0, check_sync=True,
                             loss_scaling=nn.DynamicLossScaler(8.0, 2.0, 2000) if half else None,
                             bucket_bytes=16 << 10, comm_mode=mode)
    assert tr.distributed and tr.comm.backend == "gloo"
    losses = [tr.step(g["lenet_x"][i], g["lenet_labels"]) for i in range(2)]
    ov = tr.rank0._overlap
    assert len(ov.plans) >= 2 and all(ov.schedule.issued)   # buckets issued from backward
    out = {"losses": np.array(losses), "n_buckets": len(ov.plans)}
    for k, v in tr.rank0.registry.get_parameters().items():
        out[f"final__{k}"] = v.d
    if rank == 0:
        np.savez(os.environ["OUT"], **out)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
