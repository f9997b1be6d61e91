#!/usr/bin/env python
"""Per-layer sweep of block-shape overrides (tile_n x flags) against the planner's own choice,
for the unique cfg4 layers at one per-GPU batch: where does an override beat the default?

  python tools/shape_sweep.py [--n 256] [--min-gain 0.03]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def timed(fn, reps=10):
    import torch
    fn()
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(reps):
            fn()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=256)
    ap.add_argument("--min-gain", type=float, default=0.03)
    args = ap.parse_args()
    import torch
    from paper_2110_03901_b200._kernels import conv_device
    from paper_2110_03901_b200.workloads import baseline_configs
    dev = torch.device("cuda", 0)
    seen = set()
    for L in baseline_configs()["cfg4"]:
        sp = L.spec.with_batch(args.n)
        key = (sp.h_i, sp.c_i, sp.c_o, sp.h_f, sp.stride_h)
        if key in seen or L.name == "stem":
            continue
        seen.add(key)
        x = torch.randn((sp.n, sp.h_i, sp.w_i, sp.c_i), device=dev).bfloat16()
        w = (torch.randn((sp.h_f, sp.w_f, sp.c_i, sp.c_o), device=dev) * 0.05).bfloat16()
        y = torch.empty((sp.n, sp.h_o, sp.w_o, sp.c_o), device=dev, dtype=torch.bfloat16)
        base = timed(lambda: conv_device(x, w, *sp.conv_args(), y=y))
        best = (base, 0, 0)
        for t in (0, 64, 128, 256):
            if t and t > max(64, sp.c_o + 63):
                continue
            for f in (0, 1, 2, 4, 8, 32):
                if (t, f) == (0, 0):
                    continue
                try:
                    us = timed(lambda: conv_device(x, w, *sp.conv_args(), y=y, tile_n=t, flags=f))
                except Exception:
                    continue
                if us < best[0]:
                    best = (us, t, f)
        gain = 1 - best[0] / base
        mark = "  <==" if gain >= args.min_gain else ""
        print(f"{L.name:12s} default {base:8.2f} us  best {best[0]:8.2f} us (tile_n {best[1]}, flags {best[2]})"
              f"  gain {gain * 100:5.1f}%{mark}", flush=True)


if __name__ == "__main__":
    main()
