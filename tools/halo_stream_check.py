#!/usr/bin/env python
"""A/B of the streamed-filter halo kernel against the generic kernel on the layers it takes
(bit-exact on integer-valued data; timing per layer and batch)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from paper_2110_03901_b200 import _lib
    from paper_2110_03901_b200._kernels import conv_device
    dev = torch.device("cuda", 0)
    for (n, h, c, k, r) in [(2, 28, 128, 128, 3), (3, 17, 256, 64, 3), (2, 9, 192, 128, 5), (1, 30, 128, 128, 3)]:
        x = torch.randint(-2, 3, (n, h, h, c), device=dev).bfloat16()
        w = torch.randint(-2, 3, (r, r, c, k), device=dev).bfloat16()
        a = (1, 1, r // 2, r // 2, 1, 1)
        _lib.lib.imconv_debug_set_flags(0)
        y0 = conv_device(x, w, *a, out_dtype=torch.float32)
        y2 = conv_device(x, w, *a)
        _lib.lib.imconv_debug_set_flags(1 << 26)
        y1 = conv_device(x, w, *a, out_dtype=torch.float32)
        _lib.lib.imconv_debug_set_flags(0)
        torch.cuda.synchronize()
        print((n, h, c, k, r), torch.equal(y0, y1), torch.equal(y2, y1.bfloat16()), flush=True)


if __name__ == "__main__":
    main()
