#!/usr/bin/env python
"""Yardstick: every unique cfg4 layer through cuDNN (torch conv2d, channels_last bf16,
cudnn.benchmark autotuning) and -- for 1x1 stride-1 layers -- cuBLAS (torch.matmul on the
(N*H*W, C) x (C, K) view), against this library's conv_device, all timed the same way
(CUDA graph of `reps` launches, CUDA events, after warm-up).  Library kernels are the
comparison, never the product.

  python tools/cudnn_compare.py [--n 256] [--reps 5] [--json out.json]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402
import torch.nn.functional as F  # noqa: E402


def time_graph(fn, reps):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(3):
            fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(reps):
            fn()
    g.replay()
    torch.cuda.synchronize()
    best = None
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        torch.cuda.synchronize()
        t = a.elapsed_time(b) / reps
        best = t if best is None else min(best, t)
    return best


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=256)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--json", default=None)
    args = ap.parse_args()
    import paper_2110_03901_b200 as P
    from paper_2110_03901_b200._kernels import conv_device
    from paper_2110_03901_b200.traffic import plan
    torch.backends.cudnn.benchmark = True
    dev = torch.device("cuda", 0)
    rows = []
    seen = {}
    for layer in P.workloads.resnet50_layers(args.n):
        sp = layer.spec
        if sp in seen:
            seen[sp]["count"] += 1
            continue
        x = torch.randn((sp.n, sp.h_i, sp.w_i, sp.c_i), device=dev).bfloat16()
        w = (torch.randn((sp.h_f, sp.w_f, sp.c_i, sp.c_o), device=dev) * 0.05).bfloat16()
        y = torch.empty((sp.n, sp.h_o, sp.w_o, sp.c_o), device=dev, dtype=torch.bfloat16)
        flags = P._lib.FLAG_STATIC_FILTER
        t_ours = time_graph(lambda: conv_device(x, w, *sp.conv_args(), y=y, flags=flags), args.reps)
        # cuDNN: NCHW-shaped views of NHWC memory (channels_last), filter KCRS channels_last
        xc = x.permute(0, 3, 1, 2)
        wc = w.permute(3, 2, 0, 1).contiguous(memory_format=torch.channels_last)
        conv = lambda: F.conv2d(xc, wc, stride=(sp.stride_h, sp.stride_w), padding=(sp.pad_h, sp.pad_w),
                                dilation=(sp.dilation_h, sp.dilation_w))
        t_cudnn = time_graph(conv, args.reps)
        t_cublas = None
        if sp.h_f == 1 and sp.w_f == 1 and sp.stride_h == 1 and sp.stride_w == 1:
            a2 = x.view(-1, sp.c_i)
            b2 = w.view(sp.c_i, sp.c_o)
            o2 = y.view(-1, sp.c_o)
            t_cublas = time_graph(lambda: torch.matmul(a2, b2, out=o2), args.reps)
        row = {"layer": layer.name, "count": 1, "plan": plan(sp).branch, "gflop": sp.flops / 1e9,
               "ours_us": t_ours * 1e3, "cudnn_us": t_cudnn * 1e3,
               "cublas_us": None if t_cublas is None else t_cublas * 1e3}
        seen[sp] = row
        rows.append(row)
        del x, w, y
    tot = {"ours": 0.0, "cudnn": 0.0, "best_lib": 0.0}
    print("| layer | x | plan | ours us | cuDNN us | cuBLAS us | ours TFLOP/s | cuDNN TFLOP/s | ours/best lib |")
    print("|---|---|---|---|---|---|---|---|---|")
    for r in rows:
        best = min(v for v in (r["cudnn_us"], r["cublas_us"]) if v is not None)
        tot["ours"] += r["ours_us"] * r["count"]
        tot["cudnn"] += r["cudnn_us"] * r["count"]
        tot["best_lib"] += best * r["count"]
        print(f"| {r['layer']} | {r['count']} | {r['plan']} | {r['ours_us']:.1f} | {r['cudnn_us']:.1f} | "
              f"{'' if r['cublas_us'] is None else f'{r['cublas_us']:.1f}'} | "
              f"{r['gflop'] / r['ours_us'] * 1e3:.0f} | {r['gflop'] / r['cudnn_us'] * 1e3:.0f} | "
              f"{best / r['ours_us']:.2f} |")
    gf = sum(r["gflop"] * r["count"] for r in rows)
    print(f"\nstep (sum of per-layer times): ours {tot['ours']:.0f} us = {gf / tot['ours'] * 1e3:.0f} TFLOP/s; "
          f"cuDNN {tot['cudnn']:.0f} us = {gf / tot['cudnn'] * 1e3:.0f} TFLOP/s; best library per layer "
          f"{tot['best_lib']:.0f} us = {gf / tot['best_lib'] * 1e3:.0f} TFLOP/s")
    if args.json:
        with open(args.json, "w") as fh:
            json.dump({"n": args.n, "rows": rows, "totals_us": tot}, fh, indent=1)


if __name__ == "__main__":
    main()
