#!/usr/bin/env python
"""Mainloop-rate probe of the tcgen05 GEMM per operand-major combination, via
the affine entry points on a large square problem (no conv geometry):

    fwd   : A K-major  x B MN-major      y  = x . W
    dgrad : A K-major  x B K-major       gx = gy . W^T
    wgrad : A MN-major x B MN-major      gW = x^T . gy

    python tools/gemm_probe.py [--n 8192] [--iters 10]
"""
import argparse
import ctypes as C
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=8192)
    ap.add_argument("--shape", default="", help="M,N,K for the fwd mode (affine B x I -> O)")
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--once", action="store_true")
    args = ap.parse_args()
    import torch
    from paper_2102_06725_b200 import _lib
    n = args.n
    dev = torch.device("cuda")
    if args.shape:
        M, N, K = (int(v) for v in args.shape.split(","))
        x = torch.randn(M, K, device=dev, dtype=torch.float16)
        w = torch.randn(K, N, device=dev, dtype=torch.float16) * 0.01
        out = torch.empty(M, N, device=dev, dtype=torch.float16)
        b = torch.zeros(N, device=dev, dtype=torch.float16)
        ws = torch.empty(1 << 30, dtype=torch.uint8, device=dev)
        st = torch.cuda.current_stream().cuda_stream
        fn = lambda: _lib.call("nnl_affine_fwd", 1, M, K, K, N, x.data_ptr(), w.data_ptr(),
                               b.data_ptr(), out.data_ptr(), ws.data_ptr(), ws.numel(), st)
        fn()
        ts = []
        for _ in range(args.iters):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ms = statistics.median(ts)
        byts = 2.0 * (M * K + K * N + M * N)
        print(f"M={M} N={N} K={K}: {ms:8.3f} ms  {2.0 * M * N * K / ms / 1e9:8.1f} TF/s  "
              f"{byts / ms / 1e6:8.1f} GB/s")
        return
    x = torch.randn(n, n, device=dev, dtype=torch.float16)
    w = torch.randn(n, n, device=dev, dtype=torch.float16) * 0.01
    gy = torch.randn(n, n, device=dev, dtype=torch.float16)
    out = torch.empty(n, n, device=dev, dtype=torch.float16)
    b = torch.zeros(n, device=dev, dtype=torch.float16)
    flag = torch.zeros(1, dtype=torch.int32, device=dev)
    ws = torch.empty(1 << 30, dtype=torch.uint8, device=dev)
    st = torch.cuda.current_stream().cuda_stream
    calls = {
        "fwd": lambda: _lib.call("nnl_affine_fwd", 1, n, n, n, n, x.data_ptr(), w.data_ptr(),
                                 b.data_ptr(), out.data_ptr(), ws.data_ptr(), ws.numel(), st),
        "dgrad": lambda: _lib.call("nnl_affine_bwd_data", 1, n, n, n, n, gy.data_ptr(),
                                   w.data_ptr(), out.data_ptr(), 0, ws.data_ptr(), ws.numel(), st),
        "wgrad": lambda: _lib.call("nnl_affine_bwd_weight", 1, n, n, n, n, x.data_ptr(),
                                   gy.data_ptr(), out.data_ptr(), 0, None, 0, flag.data_ptr(),
                                   ws.data_ptr(), ws.numel(), st),
    }
    flops = 2.0 * n ** 3
    for name, fn in calls.items():
        if args.once:
            fn()
            torch.cuda.synchronize()
            continue
        fn()
        ts = []
        for _ in range(args.iters):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ms = statistics.median(ts)
        print(f"{name:6s} {ms:8.3f} ms  {flops / ms / 1e9:8.1f} TF/s")
    if not args.once:  # cuBLAS context (never used by the package)
        torch.matmul(x, w)
        ts = []
        for _ in range(args.iters):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            torch.matmul(x, w)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ms = statistics.median(ts)
        print(f"cublas {ms:8.3f} ms  {flops / ms / 1e9:8.1f} TF/s")


if __name__ == "__main__":
    main()
