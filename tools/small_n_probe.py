#!/usr/bin/env python
"""Per-layer kernel time vs per-GPU batch (the shard size of a strong-scaling
run): which layers keep a fixed floor when the batch shrinks.

  python tools/small_n_probe.py [--layers stem,s4b1_3x3,...] [--ns 1,8,32,64] [--flags 0]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", default="stem,s2b1_1x1a,s2b1_3x3,s2b1_1x1b,s3b1_1x1a,s3b1_3x3,s3b1_1x1b,"
                                        "s4b1_1x1a,s4b1_3x3,s4b1_1x1b,s5b1_1x1a,s5b1_3x3,s5b1_1x1b,s4b0_proj")
    ap.add_argument("--ns", default="1,8,16,32,64")
    ap.add_argument("--flags", default="0")
    ap.add_argument("--tile-n", default="0", help="comma list of tile_n values (0 = auto)")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--dbg", default="0", help="imconv_debug_set_flags value")
    args = ap.parse_args()
    import torch
    from paper_2110_03901_b200._kernels import conv_device
    from paper_2110_03901_b200.workloads import baseline_configs
    layers = {l.name: l for l in baseline_configs()["cfg4"]}
    dev = torch.device("cuda", 0)
    from paper_2110_03901_b200 import _lib
    _lib.lib.imconv_debug_set_flags(int(args.dbg, 0))
    ns = [int(v) for v in args.ns.split(",")]
    flag_set = [(int(f, 0), int(t)) for f in args.flags.split(",") for t in args.tile_n.split(",")]
    print("layer".ljust(12) + "".join(f"{'n=' + str(n) + ' f' + str(f) + ' t' + str(t):>18s}" for n in ns for f, t in flag_set))
    for name in args.layers.split(","):
        L = layers[name]
        cells = []
        for n in ns:
            sp = L.spec.with_batch(n)
            x = torch.randn((sp.n, sp.h_i, sp.w_i, sp.c_i), device=dev).to(torch.bfloat16)
            w = (torch.randn((sp.h_f, sp.w_f, sp.c_i, sp.c_o), device=dev) * 0.05).to(torch.bfloat16)
            y = torch.empty((sp.n, sp.h_o, sp.w_o, sp.c_o), device=dev, dtype=torch.bfloat16)
            for f, t in flag_set:
                conv_device(x, w, *sp.conv_args(), y=y, flags=f, tile_n=t)
                s = torch.cuda.Stream()
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=s):
                    for _ in range(args.reps):
                        conv_device(x, w, *sp.conv_args(), y=y, flags=f, tile_n=t)
                g.replay()
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                g.replay()
                e1.record()
                torch.cuda.synchronize()
                us = e0.elapsed_time(e1) / args.reps * 1e3
                cells.append(f"{us:9.2f}us {sp.flops / us / 1e6:5.0f}")
                del g
        print(name.ljust(12) + "".join(f"{c:>18s}" for c in cells), flush=True)


if __name__ == "__main__":
    main()
