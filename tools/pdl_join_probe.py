#!/usr/bin/env python
"""Does a launch queued after a sweep of IMCONV_FLAG_INDEPENDENT convolutions see the output of
an EARLIER (slow) sweep member, not only of its immediate predecessor?  A slow first layer is
followed by fast independent layers; then (a) a flag-free conv and (b) a torch reduction read the
slow layer's output on the same stream.  Prints how often each consumer saw unfinished data."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import paper_2110_03901_b200 as P
    from paper_2110_03901_b200._kernels import conv_device
    from paper_2110_03901_b200.core import ConvSpec
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev).manual_seed(1)
    big = ConvSpec.square(64, 512, 14, 512, 3, stride=1, pad=1)   # slow
    small = ConvSpec.square(1, 64, 8, 64, 1)                      # fast
    xb = torch.randint(-2, 3, (big.n, big.h_i, big.w_i, big.c_i), device=dev, generator=g).bfloat16()
    wb = torch.randint(-2, 3, (3, 3, 512, 512), device=dev, generator=g).bfloat16()
    yb = torch.empty((big.n, big.h_o, big.w_o, big.c_o), device=dev, dtype=torch.bfloat16)
    xs = torch.randint(-2, 3, (1, 8, 8, 64), device=dev, generator=g).bfloat16()
    ws = torch.randint(-2, 3, (1, 1, 64, 64), device=dev, generator=g).bfloat16()
    ys = [torch.empty((1, 8, 8, 64), device=dev, dtype=torch.bfloat16) for _ in range(8)]
    w2 = torch.randint(-1, 2, (1, 1, 512, 64), device=dev, generator=g).bfloat16()
    ref_b = conv_device(xb, wb, 1, 1, 1, 1, 1, 1)
    ref_sum = ref_b.double().sum().item()
    ref_c = conv_device(ref_b, w2, 1, 1, 0, 0, 1, 1, out_dtype=torch.float32)
    torch.cuda.synchronize()
    IND = P._lib.FLAG_STATIC_FILTER | P._lib.FLAG_INDEPENDENT
    bad_conv = bad_sum = 0
    for it in range(50):
        yb.fill_(float("nan"))
        conv_device(xb, wb, 1, 1, 1, 1, 1, 1, y=yb, flags=P._lib.FLAG_STATIC_FILTER)  # sweep head (ordered)
        for y in ys:
            conv_device(xs, ws, 1, 1, 0, 0, 1, 1, y=y, flags=IND)
        c = conv_device(yb, w2, 1, 1, 0, 0, 1, 1, out_dtype=torch.float32)  # flag-free consumer
        s = yb.double().sum()                                               # torch consumer
        torch.cuda.synchronize()
        bad_conv += 0 if torch.equal(c, ref_c) else 1
        bad_sum += 0 if s.item() == ref_sum else 1
    print(f"flag-free conv saw unfinished data in {bad_conv}/50 runs; torch reduction in {bad_sum}/50")
    return 0 if bad_conv == 0 and bad_sum == 0 else 1


if __name__ == "__main__":
    sys.exit(main())
