#!/usr/bin/env python
"""What would launching the same-shape layers of the cfg4 sweep as ONE grouped convolution gain?
Emulation: every group of identical layer shapes (s4b1..b5 3x3, ...) becomes one convolution over
members x 256 images (same FLOP and activation bytes; one filter instead of `members`), and the sweep
of the grouped list is timed against the sweep of the 53 separate layers (CUDA graph, 20 replays).

  python tools/group_emulate.py [--n 256] [--jobs 0] [--only generic]
"""
import argparse
import collections
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=256)
    ap.add_argument("--jobs", type=float, default=0.0)
    ap.add_argument("--only", default="", help="comma list of layer-name substrings to group (default: all)")
    args = ap.parse_args()
    import torch
    import paper_2110_03901_b200 as P
    from paper_2110_03901_b200 import sweep as SW
    dev = torch.device("cuda", 0)
    layers = P.workloads.resnet50_layers(args.n)
    groups = collections.OrderedDict()
    for l in layers:
        key = l.spec if (not args.only or any(s in l.name for s in args.only.split(","))) else l.name
        groups.setdefault(key, []).append(l)

    def make(specs):
        convs = []
        for sp in specs:
            x = torch.randn((sp.n, sp.h_i, sp.w_i, sp.c_i), device=dev).bfloat16()
            w = (torch.randn((sp.h_f, sp.w_f, sp.c_i, sp.c_o), device=dev) * 0.05).bfloat16()
            y = torch.empty((sp.n, sp.h_o, sp.w_o, sp.c_o), device=dev, dtype=torch.bfloat16)
            convs.append((x, w, sp.conv_args(), y))
        return convs

    def timed(convs, flops):
        jobs = args.jobs or SW.default_jobs(flops, 53)
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            SW.conv_sweep(convs, jobs=jobs, order="mix")
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            SW.conv_sweep(convs, jobs=jobs, order="mix")
        best = 1e9
        for _ in range(3):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            g.replay()
            torch.cuda.synchronize()
            a.record()
            for _ in range(20):
                g.replay()
            b.record()
            torch.cuda.synchronize()
            best = min(best, a.elapsed_time(b) / 20)
        return best

    flops = float(sum(l.spec.flops for l in layers))
    sep = make([l.spec for l in layers])
    t_sep = timed(sep, flops)
    del sep
    torch.cuda.empty_cache()
    grp = make([ls[0].spec.with_batch(ls[0].spec.n * len(ls)) for ls in groups.values()])
    t_grp = timed(grp, flops)
    print(f"separate: {len(layers)} launches {t_sep * 1e3:.1f} us = {flops / t_sep / 1e9:.1f} TFLOP/s; "
          f"grouped: {len(groups)} launches {t_grp * 1e3:.1f} us = {flops / t_grp / 1e9:.1f} TFLOP/s "
          f"({t_grp / t_sep:.3f})")


if __name__ == "__main__":
    main()
