"""Check the host->device input path used by DataParallelTrainer.step."""
import time
import numpy as np
import torch

x = torch.empty((256, 3, 224, 224), dtype=torch.float32).pin_memory()
x.normal_()
a = x.numpy()
t = torch.from_numpy(a)
print("from_numpy(pinned).is_pinned():", t.is_pinned())
for nb in (False, True):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(5):
        d = t.to("cuda", non_blocking=nb)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 5
    print(f"non_blocking={nb}: {dt*1e3:.2f} ms  {a.nbytes/dt/1e9:.1f} GB/s")
pag = np.random.rand(256, 3, 224, 224).astype(np.float32)
torch.cuda.synchronize(); t0 = time.perf_counter()
for _ in range(5):
    d = torch.from_numpy(pag).to("cuda")
torch.cuda.synchronize(); dt = (time.perf_counter() - t0) / 5
print(f"pageable: {dt*1e3:.2f} ms  {pag.nbytes/dt/1e9:.1f} GB/s")
