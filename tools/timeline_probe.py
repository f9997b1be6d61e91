#!/usr/bin/env python
"""Launch timeline of back-to-back conv launches (instrumented build, CTA 0):
globaltimer stamps of each launch's phases, and the gap between one launch's
exit and the next one's entry.

  python tools/timeline_probe.py [--layer s4b1_1x1b] [--n 1] [--reps 8]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layer", default="s4b1_1x1b")
    ap.add_argument("--n", type=int, default=1)
    ap.add_argument("--reps", type=int, default=8)
    args = ap.parse_args()
    import torch
    from paper_2110_03901_b200 import _lib
    _lib.use_instrumented()
    from paper_2110_03901_b200._kernels import conv_device
    from paper_2110_03901_b200.workloads import baseline_configs
    layers = {l.name: l for l in baseline_configs()["cfg4"]}
    dev = torch.device("cuda", 0)
    for name in args.layer.split(","):
        sp = layers[name].spec.with_batch(args.n)
        x = torch.randn((sp.n, sp.h_i, sp.w_i, sp.c_i), device=dev).to(torch.bfloat16)
        w = (torch.randn((sp.h_f, sp.w_f, sp.c_i, sp.c_o), device=dev) * 0.05).to(torch.bfloat16)
        y = torch.empty((sp.n, sp.h_o, sp.w_o, sp.c_o), device=dev, dtype=torch.bfloat16)
        dbg = torch.zeros(148 * 20 + 1 + 64 * 8, dtype=torch.int64, device=dev)
        conv_device(x, w, *sp.conv_args(), y=y)
        s = torch.cuda.Stream()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(args.reps):
                conv_device(x, w, *sp.conv_args(), y=y)
        g.replay()
        torch.cuda.synchronize()
        _lib.lib.imconv_debug_set_buffer(dbg.data_ptr())
        # the graph baked p.dbg at capture: re-capture with the buffer set
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(args.reps):
                conv_device(x, w, *sp.conv_args(), y=y)
        dbg.zero_()
        torch.cuda.synchronize()
        g.replay()
        torch.cuda.synchronize()
        _lib.lib.imconv_debug_set_buffer(None)
        t = dbg[148 * 20 + 1:].view(64, 8).cpu().tolist()
        n = int(dbg[148 * 20].item())
        print(f"{name} n={sp.n}: {n} launches (CTA 0 stamps, ns relative to the launch's entry)")
        print("  launch  wait-done  operands  last-commit  acc-ready  stores-done  exit   gap-to-next-entry")
        for i in range(min(n, 64)):
            e = t[i]
            rel = [(v - e[0]) if v else -1 for v in e[:7]]
            gap = (t[i + 1][0] - e[6]) if i + 1 < min(n, 64) and t[i + 1][0] and e[6] else 0
            print(f"  {i:5d}  " + "  ".join(f"{v:9d}" for v in rel[1:]) + f"  {gap:9d}")


if __name__ == "__main__":
    main()
