#!/usr/bin/env python
"""One cfg4 layer through cuDNN (autotuned) and through this library, each launched once
inside a cudaProfilerStart/Stop range -- for `ncu --profile-from-start off` side-by-side
captures of the library kernel and cuDNN's choice on the same shape (yardstick only).

  ncu --profile-from-start off --set full -o rep python tools/cudnn_layer.py --layer s2b0_1x1b
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layer", default="s2b0_1x1b")
    ap.add_argument("--n", type=int, default=256)
    args = ap.parse_args()
    import torch
    import torch.nn.functional as F
    import paper_2110_03901_b200 as P
    from paper_2110_03901_b200._kernels import conv_device
    torch.backends.cudnn.benchmark = True
    dev = torch.device("cuda", 0)
    for name in args.layer.split(","):
        sp = {l.name: l for l in P.workloads.resnet50_layers(args.n)}[name].spec
        x = torch.randn((sp.n, sp.h_i, sp.w_i, sp.c_i), device=dev).bfloat16()
        w = (torch.randn((sp.h_f, sp.w_f, sp.c_i, sp.c_o), device=dev) * 0.05).bfloat16()
        xc = x.permute(0, 3, 1, 2)
        wc = w.permute(3, 2, 0, 1).contiguous(memory_format=torch.channels_last)

        def cudnn():
            return F.conv2d(xc, wc, stride=(sp.stride_h, sp.stride_w), padding=(sp.pad_h, sp.pad_w),
                            dilation=(sp.dilation_h, sp.dilation_w))

        def ours():
            return conv_device(x, w, *sp.conv_args(), flags=P._lib.FLAG_STATIC_FILTER)

        for _ in range(3):
            cudnn()
            ours()
        torch.cuda.synchronize()
        torch.cuda.cudart().cudaProfilerStart()
        ours()
        cudnn()
        torch.cuda.synchronize()
        torch.cuda.cudart().cudaProfilerStop()
        print(f"{name}: captured one launch of each")


if __name__ == "__main__":
    main()
