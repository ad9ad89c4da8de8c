#!/usr/bin/env python
"""Training-step throughput on B200 for the BASELINE.json configs.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config resnet50|resnet18|lenet|mlp]

The default (what the driver runs) is C4: ResNet-50 mixed precision, batch
256 per GPU -- the BASELINE.json metric.  `--config` gives the C1-C3 lines
(MLP and LeNet are latency configs reported in us/step).

One process per GPU (torchrun for N>1; NCCL all-reduce of gradients).  Our
arm prints ONE JSON line on rank 0:

  value       img/s with inputs resident in HBM (device-timed, max over ranks)
  e2e         img/s through DataParallelTrainer.step() with the batch copied
              from pinned host memory every step and the loss read back
  roofline    the tcgen05 implicit-GEMM kernels (conv/affine fwd+bwd) from a
              CUDA-event-profiled step: algorithmic FLOPs / device time vs
              the measured bf16 peak (sustained) in MEASURED_PEAKS.json
  cpu_baseline  the oracle (numpy port of the reference path) on this host

``--impl reference`` times the reference path on the host CPU: the oracle
port (oracle/nnl_oracle.py) of nanonnl's training step, on a bounded sample
(1 image per step), with every host thread.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "ResNet-50 mixed-precision train images/sec at 1/2/4/8 B200; % of roofline"
UNIT = "img/s"


# BASELINE.json configs[0..3]; C4 (resnet50) is the headline line the driver runs,
# the others are `--config` lines (C5, the all-reduce sweep, is tools/allreduce_sweep.py)
CONFIGS = {
    "mlp": dict(
        metric="MLP 784-256-10 fp32 train step (fwd+bwd+Momentum SGD), batch 64: us/step",
        unit="us/step", higher_is_better=False, batch=64, shape=(784,), classes=10,
        half=False, scaler=None, lr=0.1, momentum=0.9, wd=0.0,
        workload="C1 MLP 784-256-10 (ReLU, softmax CE), fp32, momentum SGD 0.9, lr 0.1"),
    "lenet": dict(
        metric="LeNet 28x28 fp16 + dynamic loss scaling train step, batch 128: us/step",
        unit="us/step", higher_is_better=False, batch=128, shape=(1, 28, 28), classes=10,
        half=True, scaler=(8.0, 2.0, 2000), lr=0.01, momentum=0.0, wd=0.0,
        workload="C2 LeNet (conv5-pool2-relu x2, affine50-relu, affine10), fp16 storage + "
                 "dynamic loss scaling (8, x2, 2000), SGD lr 0.01"),
    "resnet18": dict(
        metric="ResNet-18 CIFAR-10 shape mixed-precision train images/sec (32x32, batch 128/GPU)",
        unit="img/s", higher_is_better=True, batch=128, shape=(3, 32, 32), classes=10,
        half=True, scaler=(8.0, 2.0, 2000), lr=0.1, momentum=0.9, wd=1e-4,
        workload="C3 ResNet-18 CIFAR (3x3 stem, [2,2,2,2] basic blocks), fp16 storage + dynamic "
                 "loss scaling (8, x2, 2000), momentum SGD 0.9, wd 1e-4, lr 0.1"),
    "resnet50": dict(
        metric=METRIC, unit=UNIT, higher_is_better=True, batch=256, shape=(3, 224, 224),
        classes=1000, half=True, scaler=(8.0, 2.0, 2000), lr=0.1, momentum=0.9, wd=1e-4,
        workload="ResNet-50 v1.5 224x224 train step: fp16 storage + dynamic loss scaling "
                 "(8, x2, 2000), momentum SGD 0.9, wd 1e-4, lr 0.1"),
}


def build_graph(nn, F, networks, name, bs):
    cf = CONFIGS[name]
    xv = nn.Variable((bs,) + cf["shape"])
    tv = nn.Variable((bs,))
    if name == "mlp":
        logits = networks.mlp(xv, 10, hidden=(256,))
    elif name == "lenet":
        logits = networks.lenet(xv, 10)
    elif name == "resnet18":
        logits = networks.resnet18_cifar(xv, 10)
    else:
        logits = networks.resnet50(xv, cf["classes"])
    return {"x": xv, "label": tv, "loss": F.softmax_cross_entropy(logits, tv)}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="resnet50", choices=sorted(CONFIGS))
    ap.add_argument("--batch", type=int, default=0, help="per-GPU batch (0: the config's)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--profile-only", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="eager steps (no CUDA graph)")
    return ap.parse_args()


def gemm_traffic() -> dict | None:
    """DRAM bytes of one step's tcgen05 GEMM launches (the implicit-GEMM kernel
    and the halo weight-gradient kernel) from the committed ncu capture
    (profiles/r02/traffic.json, tools/traffic_summary.py)."""
    try:
        with open(os.path.join(ROOT, "profiles", "r02", "traffic.json")) as f:
            ks = json.load(f)["kernels"]
    except (OSError, KeyError, ValueError):
        return None
    fams = [k for k in ("nnl::k_tc_gemm", "nnl::k_tc_wgrad3") if k in ks]
    if not fams:
        return None
    return {"bytes_per_step": sum(ks[k]["dram_bytes_per_launch"] * ks[k]["launches"] for k in fams),
            "launches": sum(ks[k]["launches"] for k in fams), "kernels": fams,
            "source": "profiles/r02/traffic.json (ncu dram__bytes, one step)"}


def peaks() -> dict:
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except OSError:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
                "fallback": True}


class Clocks:
    """SM clock and throttle-reason sampling during the timed region
    (B200_PROFILING.md's clocks line).  In-process NVML in a background thread
    every 2 ms, so even a sub-millisecond timed region (the C1/C2 latency
    configs) is sampled; nvidia-smi -lms 100 when NVML is unavailable."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    # nvmlClocksEventReason* bits (nvml.h)
    BITS = {"sw_power_cap": 0x4, "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20,
            "hw_thermal_slowdown": 0x40}

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.thread = None
        self.samples = []  # (sm_mhz, max_mhz, reasons bitmask)
        self.nvml = None
        self.path = tempfile.mktemp(suffix=".csv")

    def sample_now(self):
        """One synchronous sample: called inside the timed region after the
        steps are queued, while the GPU is still executing them."""
        if self.nvml is None:
            return
        try:
            n, h = self.nvml, self.handle
            self.samples.append((float(n.nvmlDeviceGetClockInfo(h, n.NVML_CLOCK_SM)),
                                 float(n.nvmlDeviceGetMaxClockInfo(h, n.NVML_CLOCK_SM)),
                                 int(n.nvmlDeviceGetCurrentClocksEventReasons(h))))
        except Exception:  # noqa: BLE001 -- sampling must never break the bench
            pass

    def _nvml_loop(self, stop):
        while not stop.is_set():
            self.sample_now()
            stop.wait(0.002)

    def __enter__(self):
        import threading
        try:
            import pynvml as nvml
            nvml.nvmlInit()
            self.handle = nvml.nvmlDeviceGetHandleByIndex(self.gpu)
            self.nvml = nvml
            self.stop = threading.Event()
            # a short GIL switch interval lets the sampler run inside sub-ms regions
            self.switch = sys.getswitchinterval()
            sys.setswitchinterval(0.0005)
            self.thread = threading.Thread(target=self._nvml_loop, args=(self.stop,), daemon=True)
            self.thread.start()
            return self
        except Exception:  # noqa: BLE001
            self.thread = None
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=self.f, stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.thread is not None:
            self.stop.set()
            self.thread.join()
            sys.setswitchinterval(self.switch)
        if self.proc is not None:
            self.proc.terminate()
            self.proc.wait()
            self.f.close()

    def summary(self) -> dict:
        sm, mx, reasons = [], [], set()
        for s_mhz, m_mhz, bits in self.samples:
            sm.append(s_mhz)
            mx.append(m_mhz)
            reasons.update(k for k, v in self.BITS.items() if bits & v)
        try:
            for line in open(self.path):
                parts = [p.strip() for p in line.split(",")]
                if len(parts) < 9:
                    continue
                try:
                    sm.append(float(parts[1]))
                    mx.append(float(parts[2]))
                except ValueError:
                    continue
                names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown",
                         "sw_power_cap"]
                for name, v in zip(names, parts[5:9]):
                    if v.lower() == "active":
                        reasons.add(name)
        except OSError:
            pass
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx),
                "reasons": sorted(reasons), "samples": len(sm),
                "source": "nvml" if self.samples else "nvidia-smi"}


def _oracle_builder(name):
    from oracle import nnl_oracle as O
    if name == "mlp":
        return lambda m, a, t: m.sce(O.mlp(m, a, 10, hidden=(256,)), t)
    if name == "lenet":
        return lambda m, a, t: m.sce(O.lenet(m, a, 10), t)
    if name == "resnet18":
        return lambda m, a, t: m.sce(O.resnet18_cifar(m, a, 10), t)
    return lambda m, a, t: m.sce(O.resnet50(m, a, CONFIGS["resnet50"]["classes"]), t)


# bounded CPU samples: images per oracle step (full batch where it takes < ~1 s)
CPU_SAMPLE = {"mlp": 64, "lenet": 128, "resnet18": 8, "resnet50": 1}


def oracle_rate(name: str, batch: int, steps: int, warmup: int) -> tuple[float, int, float]:
    """(img/s, host threads, s/step) of the oracle port (numpy) of the reference
    training step for config `name` on `batch` images."""
    import numpy as np
    from oracle import nnl_oracle as O
    cf = CONFIGS[name]
    x = O.uniform(1, 0, (batch,) + cf["shape"], 0.0, 1.0)
    lab = (np.arange(batch) % cf["classes"]).astype(np.float32)
    sc = O.Scaler(*cf["scaler"]) if cf["scaler"] else None
    tr = O.Trainer(_oracle_builder(name), 1, batch, cf["lr"], seed=0, half=cf["half"],
                   scaler=sc, momentum=cf["momentum"], weight_decay=cf["wd"])
    for _ in range(warmup):
        tr.step(x, lab)
    t0 = time.perf_counter()
    for _ in range(steps):
        tr.step(x, lab)
    dt = (time.perf_counter() - t0) / steps
    return batch / dt, len(os.sched_getaffinity(0)), dt


def _rate_value(name: str, img_s: float, batch: int) -> float:
    """The config's metric from an images/sec rate (us/step at `batch` for the
    latency configs)."""
    if CONFIGS[name]["unit"] == "us/step":
        return 1e6 * batch / img_s
    return img_s


def run_reference(args, rank: int, world: int) -> None:
    if rank != 0:
        return
    name = args.config
    cf = CONFIGS[name]
    steps, warmup = max(1, args.steps), max(0, args.warmup)
    sample = CPU_SAMPLE[name]
    if cf["unit"] == "us/step":  # the reference path on the full per-GPU batch
        sample = args.batch or cf["batch"]
    rate, cores, sps = oracle_rate(name, sample, steps, warmup)
    value = _rate_value(name, rate, sample)
    line = {
        "impl": "reference", "metric": cf["metric"], "value": round(value, 4), "unit": cf["unit"],
        "n_gpus": args.gpus, "steps": steps, "warmup": warmup, "ms_per_step": round(1000 * sps, 2),
        "higher_is_better": cf["higher_is_better"], "scaling": "weak", "vs_baseline": None,
        "dtype": "f16-storage/f32" if cf["half"] else "f32",
        "data": "synthetic (RngState seed 1)",
        "config": {"workload": cf["workload"] + " (oracle port of the reference path)",
                   "sample": f"{sample} image(s) per step", "parallelism": "host threads"},
        "cpu_baseline": {"value": round(value, 4), "unit": cf["unit"], "cores": cores,
                         "kind": "port",
                         "sample": f"{name} train step on {sample} image(s) (oracle/nnl_oracle.py)"},
        "e2e": {"value": round(value, 4), "unit": cf["unit"], "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import numpy as np
    import torch
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    import paper_2102_06725_b200 as nn
    import paper_2102_06725_b200.functions as F
    from paper_2102_06725_b200 import _lib, networks
    from paper_2102_06725_b200.communicator import DataParallelTrainer
    from paper_2102_06725_b200.profiler import PROFILER

    name = args.config
    cf = CONFIGS[name]
    B = args.batch or cf["batch"]
    nn.set_default_context(nn.ExecutionContext(
        type_config=nn.TypeConfig.HALF if cf["half"] else nn.TypeConfig.FLOAT))
    scaler = nn.DynamicLossScaler(*cf["scaler"]) if cf["scaler"] else None
    trainer = DataParallelTrainer(world, B * world, lambda bs: build_graph(nn, F, networks, name, bs),
                                  lr=cf["lr"], seed=0, loss_scaling=scaler, check_sync=False,
                                  momentum=cf["momentum"], weight_decay=cf["wd"])
    # this rank's shard of the global synthetic batch: counter offset = shard start
    per_img = int(np.prod(cf["shape"]))
    rng = nn.RngState(1, counter=rank * B * per_img)
    xdev = rng.next_uniform_device((B,) + cf["shape"], 0.0, 1.0)
    x_host = torch.empty(xdev.shape, dtype=torch.float32).pin_memory()
    x_host.copy_(xdev)
    del xdev
    lab_host = torch.empty(B, dtype=torch.float32).pin_memory()
    lab_host.copy_(torch.from_numpy(((np.arange(B) + rank * B) % cf["classes"]).astype(np.float32)))
    xs, ls = x_host.numpy(), lab_host.numpy()

    def e2e_step():
        return trainer.step(xs, ls, shard=True) if world > 1 else trainer.step(xs, ls)

    def e2e_run(k):
        """k end-to-end steps through the public API; single process: the
        pipelined `step_async` (step i+1's H2D overlaps step i's compute), each
        step still copies its inputs and reads its loss back."""
        if world > 1:
            out = None
            for _ in range(k):
                out = e2e_step()
            return out
        pend = None
        for _ in range(k):
            h = trainer.step_async(xs, ls)
            if pend is not None:
                pend.result()
            pend = h
        return pend.result()

    def sync():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()

    def max_over_ranks(v: float) -> float:
        if dist is None:
            return v
        t = torch.tensor([v], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for _ in range(args.warmup):
        e2e_step()
    sync()
    # host cost of issuing one eager step (Python engine + ctypes launches)
    t0 = time.perf_counter()
    trainer.step_resident()
    host_ms = (time.perf_counter() - t0) * 1000.0
    sync()
    graph = False
    if not args.no_graph:
        try:
            trainer.capture_graph()
            graph = True
        except Exception as exc:  # noqa: BLE001 - reported, eager path still valid
            print(f"# cuda graph capture failed, eager steps: {exc}", file=sys.stderr)
        for _ in range(2):
            trainer.step_resident()
        sync()

    # ---- device-resident throughput (value) ----
    K = args.steps
    _lib.lib().nnl_launch_count(1)
    with Clocks(local) as clk:
        sync()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(K):
            trainer.step_resident()
        e.record()
        # the queued steps are still running: sample the clocks while polling
        # for their end (NVML queries are ~10 us; the device events time the steps)
        clk.sample_now()
        while not e.query():
            clk.sample_now()
            time.sleep(0.001)
        sync()
        ms = max_over_ranks(s.elapsed_time(e))
    launches = int(_lib.lib().nnl_launch_count(1))
    if graph:  # replays issue no host launches: count the recorded libnnl kernels
        launches = trainer.graph_kernels * K
    img_s = B * world * K / (ms / 1000.0)
    value = ms * 1000.0 / K if cf["unit"] == "us/step" else img_s

    # ---- end-to-end through the public API (H2D from pinned memory + loss D2H) ----
    # untimed warm-up of the pipelined API (its first calls record the per-slot
    # input/loss graphs, one-time work like the resident graph's capture)
    e2e_run(max(2, args.warmup))
    sync()
    s2, e2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    w0 = time.perf_counter()
    s2.record()
    loss = e2e_run(K)
    e2.record()
    sync()
    ms_e2e = max_over_ranks(max(s2.elapsed_time(e2), (time.perf_counter() - w0) * 1000.0))
    e2e = ms_e2e * 1000.0 / K if cf["unit"] == "us/step" else B * world * K / (ms_e2e / 1000.0)

    # ---- roofline of the GEMM kernels from one profiled (eager) step ----
    saved_graph = getattr(trainer, "_graph", None)
    trainer._graph = None
    PROFILER.enabled = True
    PROFILER.gpu_lead_cycles = 400000  # ~0.2 ms: node timings free of host launch latency
    # one untimed profiled step first: the profiled (single-stream) order can reach a
    # kernel the graph never launched, whose first launch pays lazy module loading
    trainer.step_resident()
    PROFILER.reset()
    trainer.step_resident()
    PROFILER.enabled = False
    PROFILER.gpu_lead_cycles = 0
    trainer._graph = saved_graph
    prof = PROFILER.summary()
    gemm_ms = sum(v["ms"] for k, v in prof.items() if k.split(".")[0] in ("Convolution", "Affine"))
    gemm_fl = sum(v["flops"] for k, v in prof.items())
    total_ms = sum(v["ms"] for v in prof.values())
    pk = peaks()
    traffic = gemm_traffic() if name == "resnet50" else None
    achieved = gemm_fl / (gemm_ms / 1000.0) / 1e12 if gemm_ms > 0 else 0.0
    peak = pk.get("bf16_tflops_sustained", pk.get("bf16_tflops"))
    # the same GEMM node time against each pass's own roofline min(tensor, AI x HBM)
    # (the 1x1 layers are HBM-bound, so the tensor fraction alone understates them)
    layer_bound_ms = PROFILER.gemm_bound_ms(pk.get("bf16_tflops", peak), pk.get("hbm_gbs", 6541.5))

    if rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        return

    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        sample = CPU_SAMPLE[name]
        reps = 2 if name in ("resnet18", "resnet50") else 20
        rate, cores, _ = oracle_rate(name, sample, reps, 1 if reps > 2 else 0)
        cpu = {"value": round(_rate_value(name, rate, sample), 4), "unit": cf["unit"],
               "cores": cores, "kind": "port",
               "sample": f"oracle {name} train step, {sample} image(s) x {reps} steps"}

    h2d = int(x_host.numel() * 4 + lab_host.numel() * 4)
    latency = cf["unit"] == "us/step"
    line = {
        "metric": cf["metric"], "value": round(value, 2), "unit": cf["unit"], "n_gpus": world,
        "steps": K, "warmup": args.warmup, "ms_per_step": round(ms / K, 4),
        "higher_is_better": cf["higher_is_better"],
        "scaling": "weak", "vs_baseline": None, "dtype": "f16" if cf["half"] else "f32",
        "data": "synthetic (RngState seed 1, uniform [0,1)), random-init weights (registry seed 0)",
        "config": {"workload": cf["workload"], "name": name,
                   "global_batch": B * world, "per_gpu_batch": B, "input": list(cf["shape"]),
                   "parallelism": f"dp{world}", "cuda_graph": graph,
                   "host_ms_per_eager_step": round(host_ms, 3),
                   "l2": ("inputs+activations (~20 GB/step) far exceed the 126 MB L2"
                          if name == "resnet50" else
                          "working set fits in L2: steps run L2-warm (no flush)")},
        "e2e": {"value": round(e2e, 2), "unit": cf["unit"], "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": 4,
                "api": "DataParallelTrainer.step_async (H2D of step i+1 overlaps step i)"
                       if world == 1 else "DataParallelTrainer.step"},
        "gpu_launches": launches,
        "roofline": {"bound": "tensor", "kernel": "GEMM kernels (conv/affine fwd+dgrad+wgrad)",
                     "achieved": round(achieved, 2), "peak": peak, "unit": "TFLOP/s",
                     "frac": round(achieved / peak, 4) if peak else None,
                     "traffic": (traffic or {}).get("bytes_per_step"), "traffic_detail": traffic,
                     "peak_source": "MEASURED_PEAKS.json bf16_tflops_sustained",
                     "gemm_share_of_step": round(gemm_ms / total_ms, 3) if total_ms else None,
                     "gemm_ms": round(gemm_ms, 3),
                     "per_pass_bound_ms": round(layer_bound_ms, 3),
                     "frac_of_per_pass_bound": round(layer_bound_ms / gemm_ms, 4) if gemm_ms else None,
                     "gemm_tflop_per_step": round(gemm_fl / 1e12, 4)},
        "clocks": clk.summary(),
        "last_loss": loss,
        "profile_ms": {k: round(v["ms"], 3) for k, v in sorted(prof.items(),
                                                                key=lambda kv: -kv[1]["ms"])},
    }
    if latency:
        line["roofline"]["note"] = ("launch-latency bound: us/step (CUDA graph replay of "
                                    f"{trainer.graph_kernels if graph else '?'} kernels) is the "
                                    "figure of merit; the tensor fraction is informative only")
        line["images_per_s"] = round(img_s, 1)
    if cpu is not None:
        line["cpu_baseline"] = cpu
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
