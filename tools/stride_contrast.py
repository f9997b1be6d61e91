#!/usr/bin/env python
"""Channel-first vs channel-last implicit lowering as the stride grows (
the paper's Fig. 3 / Fig. 14a contrast), measured on B200.

  python tools/stride_contrast.py [--json out.json]

Both paths run the same tcgen05 pipeline; only operand generation differs:
channel-first = TMA im2col boxes (128-byte channel runs per tap), channel-last
= k ordered (c, r, s), every 2-byte A element gathered by threads.  The OUTPUT
is fixed (N x P x P x K) and the input grows with the 3x3 stride (H = s*P), so
both paths do identical work at every stride and only the input locality of
the operand gather changes.  CUDA-graph timing; reports TFLOP/s and CL/CF.
"""

import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=32)
    ap.add_argument("--c", type=int, default=128)
    ap.add_argument("--k", type=int, default=128)
    ap.add_argument("--p", type=int, default=28, help="output extent (fixed across strides)")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--json", default=None)
    args = ap.parse_args()
    import torch
    from paper_2110_03901_b200 import ConvSpec, _lib
    from paper_2110_03901_b200._kernels import conv_device

    torch.cuda.set_device(0)
    rows = []
    for stride in (1, 2, 3, 4):
        sp = ConvSpec.square(args.n, args.c, stride * args.p, args.k, 3, stride=stride, pad=1)
        x = torch.randn((sp.n, sp.h_i, sp.w_i, sp.c_i), device="cuda").bfloat16()
        w = (torch.randn((3, 3, sp.c_i, sp.c_o), device="cuda") * 0.05).bfloat16()
        res = {}
        for name, flags in (("channel_first", 0), ("channel_last", _lib.FLAG_CHANNEL_LAST)):
            run = lambda: conv_device(x, w, *sp.conv_args(), flags=flags)  # noqa: E731
            y = run()
            torch.cuda.synchronize()
            res[name + "_out"] = y.float()
            g = torch.cuda.CUDAGraph()
            s = torch.cuda.Stream()
            with torch.cuda.graph(g, stream=s):
                for _ in range(args.reps):
                    run()
            g.replay()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            g.replay()
            b.record()
            torch.cuda.synchronize()
            ms = a.elapsed_time(b) / args.reps
            res[name] = ms
        rel = float((res["channel_first_out"] - res["channel_last_out"]).abs().max() /
                    res["channel_first_out"].abs().max())
        row = {"stride": stride, "H": sp.h_i, "P": sp.h_o, "cf_ms": round(res["channel_first"], 4),
               "cl_ms": round(res["channel_last"], 4),
               "cf_tflops": round(sp.flops / (res["channel_first"] / 1e3) / 1e12, 1),
               "cl_tflops": round(sp.flops / (res["channel_last"] / 1e3) / 1e12, 1),
               "cl_over_cf": round(res["channel_last"] / res["channel_first"], 2), "max_rel_diff": rel}
        rows.append(row)
        print(json.dumps(row), flush=True)
    if args.json:
        json.dump({"n": args.n, "c": args.c, "k": args.k, "p": args.p, "rows": rows}, open(args.json, "w"), indent=1)


if __name__ == "__main__":
    main()
