#!/usr/bin/env python
"""Time single SIMT-path GEMMs (affine / narrow convolutions of C1-C2) through
the C ABI with CUDA events: 200 back-to-back launches, mean us per call.

    python tools/simt_probe.py
"""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2102_06725_b200 import _lib  # noqa: E402


def timeit(fn, reps=50):
    """mean device time of one call: `reps` calls captured in a CUDA graph
    (no host launch overhead), the graph replayed 20 times"""
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(3):
            fn(s.cuda_stream)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(reps):
                fn(s.cuda_stream)
        g.replay()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        for _ in range(20):
            g.replay()
        b.record(s)
        torch.cuda.synchronize()
    return a.elapsed_time(b) * 1000 / (20 * reps)


def main():
    lib = _lib.lib()
    for dt, code in ((torch.float32, 0), (torch.float16, 1)):
        for (bs, fi, fo) in ((64, 784, 256), (64, 256, 10), (128, 256, 50), (128, 50, 10)):
            x = torch.rand(bs, fi, device="cuda", dtype=dt)
            w = torch.rand(fi, fo, device="cuda", dtype=dt)
            b = torch.rand(fo, device="cuda", dtype=dt)
            y = torch.empty(bs, fo, device="cuda", dtype=dt)
            dy = torch.rand(bs, fo, device="cuda", dtype=dt)
            dx = torch.empty(bs, fi, device="cuda", dtype=dt)
            dw = torch.empty(fi, fo, device="cuda", dtype=dt)
            db = torch.empty(fo, device="cuda", dtype=dt)
            wsz = max(lib.nnl_affine_workspace_size(code, bs, fi, fo, p) for p in range(3))
            ws = torch.empty(max(wsz, 16), device="cuda", dtype=torch.uint8)
            f = lambda st: _lib.call("nnl_affine_fwd", code, bs, fi, fi, fo, x.data_ptr(), w.data_ptr(),
                                  b.data_ptr(), y.data_ptr(), ws.data_ptr(), wsz, st)
            d = lambda st: _lib.call("nnl_affine_bwd_data", code, bs, fi, fi, fo, dy.data_ptr(),
                                  w.data_ptr(), dx.data_ptr(), 0, ws.data_ptr(), wsz, st)
            g = lambda st: _lib.call("nnl_affine_bwd_weight", code, bs, fi, fi, fo, x.data_ptr(),
                                  dy.data_ptr(), dw.data_ptr(), 0, db.data_ptr(), 0, None,
                                  ws.data_ptr(), wsz, st)
            print(f"{str(dt):14s} affine {bs}x{fi}->{fo}: fwd {timeit(f):7.2f} us  dgrad "
                  f"{timeit(d):7.2f} us  wgrad+bias {timeit(g):7.2f} us", flush=True)
    # empty-kernel floor: a tiny fill
    z = torch.empty(16, device="cuda")
    print(f"fill floor {timeit(lambda st: _lib.call('nnl_fill', 0, 16, z.data_ptr(), 0.0, st)):.2f} us")


if __name__ == "__main__":
    main()
