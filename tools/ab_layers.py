#!/usr/bin/env python
"""A/B of host-side planner switches (imconv_debug_set_flags bits 16+) on cfg4 layers:
each (layer, per-GPU batch) timed under switch set A and B, interleaved, each launch
sequence captured in a CUDA graph (reps launches, CUDA events, best of 7).  Also checks
that A and B produce identical outputs on integer-valued data (both must be exact).

  python tools/ab_layers.py --layers s5b0_3x3,s5b1_1x1a --n 256,32 --b 0x80000
  (0x80000 = no split-K, 0x200000 = no automatic CTA pairs; see imconv_api.cu kDbg*)
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", default="s5b0_3x3")
    ap.add_argument("--n", default="256")
    ap.add_argument("--a", type=lambda v: int(v, 0), default=0)
    ap.add_argument("--b", type=lambda v: int(v, 0), default=0)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--fa", type=lambda v: int(v, 0), default=0, help="imconv flags of arm A (block-shape overrides)")
    ap.add_argument("--fb", type=lambda v: int(v, 0), default=0, help="imconv flags of arm B")
    ap.add_argument("--data", default="int", choices=["int", "randn"],
                    help="int: integer-valued (outputs compared); randn: bench.py-like N(0,1) / Kaiming")
    args = ap.parse_args()
    import torch
    import paper_2110_03901_b200 as P
    from paper_2110_03901_b200 import _lib
    from paper_2110_03901_b200._kernels import conv_device
    from paper_2110_03901_b200.traffic import plan
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(0)
    flags = _lib.FLAG_STATIC_FILTER

    def timed(x, w, y, sp, host, cflags):
        _lib.lib.imconv_debug_set_flags(host)
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            conv_device(x, w, *sp.conv_args(), y=y, flags=flags | cflags)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(args.reps):
                conv_device(x, w, *sp.conv_args(), y=y, flags=flags | cflags)
        _lib.lib.imconv_debug_set_flags(0)
        g.replay()
        torch.cuda.synchronize()
        return g

    def best(g):
        ts = []
        for _ in range(7):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            g.replay()
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b) / args.reps * 1e3)
        return min(ts)

    print("| layer | n | plan A | plan B | A us | B us | B/A | outputs |")
    print("|---|---|---|---|---|---|---|---|")
    for n in [int(v) for v in args.n.split(",")]:
        layers = P.workloads.resnet50_layers(n)
        names = args.layers.split(",")
        if args.layers == "all":
            seen, names = set(), []
            for l in layers:
                if l.spec not in seen:
                    seen.add(l.spec)
                    names.append(l.name)
        by = {l.name: l for l in layers}
        for name in names:
            sp = by[name].spec
            g = torch.Generator(device=dev).manual_seed(5)
            if args.data == "int":
                x = torch.randint(-2, 3, (sp.n, sp.h_i, sp.w_i, sp.c_i), generator=g, device=dev).to(torch.bfloat16)
                w = torch.randint(-2, 3, (sp.h_f, sp.w_f, sp.c_i, sp.c_o), generator=g, device=dev).to(torch.bfloat16)
            else:
                x = torch.randn((sp.n, sp.h_i, sp.w_i, sp.c_i), generator=g, device=dev).to(torch.bfloat16)
                w = (torch.randn((sp.h_f, sp.w_f, sp.c_i, sp.c_o), generator=g, device=dev)
                     * (2.0 / (sp.c_i * sp.h_f * sp.w_f)) ** 0.5).to(torch.bfloat16)
            ya = torch.empty((sp.n, sp.h_o, sp.w_o, sp.c_o), device=dev, dtype=torch.bfloat16)
            yb = torch.empty_like(ya)
            _lib.lib.imconv_debug_set_flags(args.a)
            pa = plan(sp, flags=flags | args.fa).branch
            _lib.lib.imconv_debug_set_flags(args.b)
            pb = plan(sp, flags=flags | args.fb).branch
            _lib.lib.imconv_debug_set_flags(0)
            ga = timed(x, w, ya, sp, args.a, args.fa)
            gb = timed(x, w, yb, sp, args.b, args.fb)
            ta, tb = [], []
            for _ in range(3):
                ta.append(best(ga))
                tb.append(best(gb))
            same = torch.equal(ya, yb)
            print(f"| {name} | {n} | {pa} | {pb} | {min(ta):.2f} | {min(tb):.2f} | {min(tb) / min(ta):.3f} | "
                  f"{'identical' if same else ('DIFFER' if args.data == 'int' else 'differ (float sums)')} |", flush=True)
            del ga, gb, x, w, ya, yb


if __name__ == "__main__":
    main()
