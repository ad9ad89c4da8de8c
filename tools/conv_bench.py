#!/usr/bin/env python
"""Per-layer timing of the libnnl convolution kernels at ResNet-50 shapes.

    python tools/conv_bench.py [--layers all|i,j,..] [--passes fwd,dgrad,wgrad] [--cudnn]

Each pass is timed with CUDA events (median of --iters after --warmup), and
reported as TFLOP/s against the per-layer roofline bound
min(tensor peak, AI x HBM) from MEASURED_PEAKS.json.  --cudnn also times
torch/cuDNN on the same shapes for context (never used by the package).
"""

import argparse
import ctypes as C
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

# (batch, cin, cout, k, stride, pad, hw) -- the distinct ResNet-50 convolutions
LAYERS = [
    (256, 3, 64, 7, 2, 3, 224),
    (256, 64, 64, 1, 1, 0, 56),
    (256, 64, 64, 3, 1, 1, 56),
    (256, 64, 256, 1, 1, 0, 56),
    (256, 256, 64, 1, 1, 0, 56),
    (256, 256, 128, 1, 1, 0, 56),
    (256, 128, 128, 3, 2, 1, 56),
    (256, 256, 512, 1, 2, 0, 56),
    (256, 128, 512, 1, 1, 0, 28),
    (256, 512, 128, 1, 1, 0, 28),
    (256, 128, 128, 3, 1, 1, 28),
    (256, 512, 256, 1, 1, 0, 28),
    (256, 256, 256, 3, 2, 1, 28),
    (256, 512, 1024, 1, 2, 0, 28),
    (256, 256, 1024, 1, 1, 0, 14),
    (256, 1024, 256, 1, 1, 0, 14),
    (256, 256, 256, 3, 1, 1, 14),
    (256, 1024, 512, 1, 1, 0, 14),
    (256, 512, 512, 3, 2, 1, 14),
    (256, 1024, 2048, 1, 2, 0, 14),
    (256, 512, 2048, 1, 1, 0, 7),
    (256, 2048, 512, 1, 1, 0, 7),
    (256, 512, 512, 3, 1, 1, 7),
]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", default="all")
    ap.add_argument("--passes", default="fwd,dgrad,wgrad")
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--cudnn", action="store_true")
    ap.add_argument("--stats", action="store_true",
                    help="forward with the BN-statistics epilogue (as in the training step)")
    ap.add_argument("--once", action="store_true", help="one call per pass (for ncu)")
    ap.add_argument("--ab-pairs", action="store_true",
                    help="also time each pass with CTA pairs disabled (same process)")
    args = ap.parse_args()
    import torch
    from paper_2102_06725_b200 import _lib
    L = _lib.lib()
    pk = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    tpk = pk.get("bf16_tflops", 1683.5) * 1e12
    hbm = pk.get("hbm_gbs", 6541.5) * 1e9
    sel = range(len(LAYERS)) if args.layers == "all" else [int(i) for i in args.layers.split(",")]
    passes = args.passes.split(",")
    dev = torch.device("cuda")
    ws = torch.empty(1 << 31, dtype=torch.uint8, device=dev)
    flag = torch.zeros(1, dtype=torch.int32, device=dev)
    st = torch.cuda.current_stream().cuda_stream
    print(f"{'layer':34s} {'pass':6s} {'ms':>8s} {'TF/s':>8s} {'bound':>8s} {'%bnd':>6s}"
          + (f" {'cudnn':>8s}" if args.cudnn else ""))
    total = {"ours": 0.0, "bound": 0.0}
    for li in sel:
        b, c, k, r, s, p, hw = LAYERS[li]
        oh = (hw + 2 * p - r) // s + 1
        cs = _lib.ConvShape(b, hw, hw, c, k, r, r, s, s, p, p, oh, oh)
        x = torch.randn(b, hw, hw, c, device=dev, dtype=torch.float16)
        w = (torch.randn(k, r, r, c, device=dev, dtype=torch.float16) * 0.05)
        bias = torch.zeros(k, device=dev, dtype=torch.float16)
        y = torch.empty(b, oh, oh, k, device=dev, dtype=torch.float16)
        dy = torch.randn_like(y)
        dx = torch.empty_like(x)
        dw = torch.empty_like(w)
        flops = 2.0 * b * oh * oh * k * c * r * r
        for ps in passes:
            if ps == "fwd":
                sp, sh = None, None
                if args.stats:
                    rows = int(_lib.lib().nnl_conv2d_stat_rows(C.byref(cs), 1))
                    if rows > 0:
                        parts = torch.empty(rows * 2 * k, device=dev)
                        shift = torch.zeros(k, device=dev)
                        sp, sh = parts.data_ptr(), shift.data_ptr()
                fn = lambda: _lib.call("nnl_conv2d_fwd", C.byref(cs), 1, x.data_ptr(), w.data_ptr(),
                                       bias.data_ptr(), y.data_ptr(), sp, sh, ws.data_ptr(),
                                       ws.numel(), st)
                byts = 2.0 * (x.numel() + w.numel() + y.numel())
            elif ps == "dgrad":
                if c % 8:
                    continue
                fn = lambda: _lib.call("nnl_conv2d_bwd_data", C.byref(cs), 1, dy.data_ptr(),
                                       w.data_ptr(), dx.data_ptr(), 0, ws.data_ptr(), ws.numel(),
                                       st)
                byts = 2.0 * (dy.numel() + w.numel() + dx.numel())
            else:
                fn = lambda: _lib.call("nnl_conv2d_bwd_weight", C.byref(cs), 1, x.data_ptr(),
                                       dy.data_ptr(), dw.data_ptr(), 0, None, 0, flag.data_ptr(),
                                       ws.data_ptr(), ws.numel(), st)
                byts = 2.0 * (x.numel() + dy.numel() + w.numel())
            if args.once:
                fn()
                torch.cuda.synchronize()
                continue
            def timed():
                for _ in range(args.warmup):
                    fn()
                times = []
                for _ in range(args.iters):
                    e0 = torch.cuda.Event(enable_timing=True)
                    e1 = torch.cuda.Event(enable_timing=True)
                    e0.record()
                    fn()
                    e1.record()
                    torch.cuda.synchronize()
                    times.append(e0.elapsed_time(e1))
                return statistics.median(times)

            ms = timed()
            extra = ""
            if args.ab_pairs:
                prev = L.nnl_set_tc_pairs(0)
                ms_single = timed()
                L.nnl_set_tc_pairs(prev)
                extra += f" single {ms_single:8.3f}"
                total["single"] = total.get("single", 0.0) + ms_single
            bound_s = max(flops / tpk, byts / hbm)
            tf = flops / (ms / 1e3) / 1e12
            total["ours"] += ms
            total["bound"] += bound_s * 1e3
            if args.cudnn:
                xt = x.permute(0, 3, 1, 2)
                wt = w.permute(0, 3, 1, 2)
                dyt = dy.permute(0, 3, 1, 2)
                if ps == "fwd":
                    cf = lambda: torch.nn.functional.conv2d(xt, wt, None, s, p)
                elif ps == "dgrad":
                    cf = lambda: torch.nn.grad.conv2d_input(xt.shape, wt, dyt, s, p)
                else:
                    cf = lambda: torch.nn.grad.conv2d_weight(xt, wt.shape, dyt, s, p)
                for _ in range(2):
                    cf()
                ct = []
                for _ in range(args.iters):
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    cf()
                    e1.record()
                    torch.cuda.synchronize()
                    ct.append(e0.elapsed_time(e1))
                extra += f" cudnn {statistics.median(ct):8.3f}"
            name = f"{b}x{c}x{hw}x{hw}->{k} k{r}s{s}"
            print(f"{name:34s} {ps:6s} {ms:8.3f} {tf:8.1f} {bound_s * 1e3:8.3f} "
                  f"{100 * bound_s * 1e3 / ms:6.1f}{extra}", flush=True)
    if not args.once:
        print(f"TOTAL ours {total['ours']:.3f} ms, per-layer bound {total['bound']:.3f} ms "
              f"({100 * total['bound'] / max(total['ours'], 1e-9):.1f}% of roofline)"
              + (f"; without CTA pairs {total['single']:.3f} ms" if "single" in total else ""))


if __name__ == "__main__":
    main()
