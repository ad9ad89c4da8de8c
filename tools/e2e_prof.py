import cProfile, pstats, sys, os, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import bench
import paper_2102_06725_b200 as nn
import paper_2102_06725_b200.functions as F
from paper_2102_06725_b200 import networks
from paper_2102_06725_b200.communicator import DataParallelTrainer
name = sys.argv[1] if len(sys.argv) > 1 else "mlp"
cf = bench.CONFIGS[name]
nn.set_default_context(nn.ExecutionContext(type_config=nn.TypeConfig.HALF if cf["half"] else nn.TypeConfig.FLOAT))
B = cf["batch"]
sc = nn.DynamicLossScaler(*cf["scaler"]) if cf["scaler"] else None
tr = DataParallelTrainer(1, B, lambda bs: bench.build_graph(nn, F, networks, name, bs), lr=cf["lr"], seed=0,
                         loss_scaling=sc, check_sync=False, momentum=cf["momentum"], weight_decay=cf["wd"])
xh = torch.rand((B,) + cf["shape"]).pin_memory(); lh = torch.from_numpy((np.arange(B) % 10).astype(np.float32)).pin_memory()
xs, ls = xh.numpy(), lh.numpy()
for _ in range(3): tr.step(xs, ls)
tr.capture_graph()
def run(k):
    pend = None
    for _ in range(k):
        h = tr.step_async(xs, ls)
        if pend is not None: pend.result()
        pend = h
    pend.result()
run(20); torch.cuda.synchronize()
t0 = time.perf_counter(); run(200); torch.cuda.synchronize(); print("us/step", (time.perf_counter()-t0)/200*1e6)
pr = cProfile.Profile(); pr.enable(); run(200); pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)

# bare costs (host wall time per call, GPU work queued asynchronously)
torch.cuda.synchronize()
g = tr._graph
t0 = time.perf_counter()
for _ in range(200):
    g.replay()
t1 = time.perf_counter(); torch.cuda.synchronize(); t2 = time.perf_counter()
print(f"bare replay: host {(t1-t0)/200*1e6:.1f} us/call, drain {(t2-t1)*1e3:.2f} ms")
raw = g.__class__.__mro__[1].replay  # the C++ binding without torch's Python wrapper
t0 = time.perf_counter()
for _ in range(200):
    raw(g)
t1 = time.perf_counter(); torch.cuda.synchronize()
print(f"raw replay: host {(t1-t0)/200*1e6:.1f} us/call")
t0 = time.perf_counter()
for _ in range(200):
    h = tr.step_async(xs, ls)
t1 = time.perf_counter(); torch.cuda.synchronize()
print(f"step_async issue only: {(t1-t0)/200*1e6:.1f} us/call")
