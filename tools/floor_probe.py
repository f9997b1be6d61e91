#!/usr/bin/env python
"""Fixed per-launch cost of the conv kernels: back-to-back graph replays of a
one-tile convolution, with and without programmatic dependent launch, next to
a trivial torch kernel (the graph-node floor)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def timed(fn, reps=50):
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
    import torch
    from paper_2110_03901_b200 import _lib
    from paper_2110_03901_b200._kernels import conv_device
    dev = torch.device("cuda", 0)
    t = torch.zeros(1024, device=dev)
    print(f"torch add_ (1024 floats): {timed(lambda: t.add_(1)):.2f} us")
    cases = [("1x1 n1 8x8 c64 k64", (1, 8, 8, 64), (1, 1, 64, 64), (1, 1, 0, 0, 1, 1)),
             ("3x3 n1 8x8 c64 k64", (1, 8, 8, 64), (3, 3, 64, 64), (1, 1, 1, 1, 1, 1)),
             ("1x1 n1 8x8 c64 k256", (1, 8, 8, 64), (1, 1, 64, 256), (1, 1, 0, 0, 1, 1)),
             ("1x1 n1 8x8 c512 k256", (1, 8, 8, 512), (1, 1, 512, 256), (1, 1, 0, 0, 1, 1)),
             ("1x1 n1 8x8 c2048 k256", (1, 8, 8, 2048), (1, 1, 2048, 256), (1, 1, 0, 0, 1, 1)),
             ("3x3 n1 7x7 c512 k256", (1, 7, 7, 512), (3, 3, 512, 256), (1, 1, 1, 1, 1, 1))]
    for name, xs, ws, args in cases:
        x = torch.randn(xs, device=dev).to(torch.bfloat16)
        w = torch.randn(ws, device=dev).to(torch.bfloat16)
        row = []
        for dbg, lab in ((0, "pdl"), (1 << 18, "nopdl"), (1 << 19, "nosplitk")):
            _lib.lib.imconv_debug_set_flags(dbg)
            row.append(f"{lab} {timed(lambda: conv_device(x, w, *args)):7.2f} us")
        _lib.lib.imconv_debug_set_flags(0)
        print(f"{name:24s} " + "  ".join(row), flush=True)


if __name__ == "__main__":
    main()
