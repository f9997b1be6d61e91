#!/usr/bin/env python
"""Soak: seeded random convolutions (tests/test_gpu_fuzz.py's generator, more seeds) through every
launch mode the sweep and the bench use -- default, IMCONV_FLAG_INDEPENDENT on 56 / 36 / 18 / 6 CTAs,
forced CTA pairs / single CTAs, no-halo -- integer-valued bf16 with fp32 output and int8, all
bit-exact against the oracle.  Prints the first mismatch and exits 1.

  python tools/soak.py [--seeds 40] [--start 5000] [--debug-build]
"""
import argparse
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seeds", type=int, default=40)
    ap.add_argument("--start", type=int, default=5000)
    ap.add_argument("--debug-build", action="store_true",
                    help="run through libimconv_debug.so (device invariant checks: mbarrier phases, tickets, ...)")
    args = ap.parse_args()
    import torch
    import paper_2110_03901_b200 as P
    from paper_2110_03901_b200 import _lib
    if args.debug_build:
        _lib.use_debug()
    from paper_2110_03901_b200._kernels import conv_device
    from oracle import oracle as O
    from test_gpu_fuzz import _random_case
    ind = _lib.FLAG_STATIC_FILTER | _lib.FLAG_INDEPENDENT
    modes = [("default", 0, 0), ("static", _lib.FLAG_STATIC_FILTER, 0), ("ind56", ind, 56), ("ind36", ind, 36),
             ("ind18", ind, 18), ("ind6", ind, 6), ("pair", _lib.FLAG_CTA_PAIR, 0), ("single", _lib.FLAG_SINGLE_CTA, 0),
             ("nohalo", _lib.FLAG_NO_HALO, 0), ("pair74", _lib.FLAG_CTA_PAIR | ind, 74)]
    t0 = time.time()
    cases = 0
    for seed in range(args.start, args.start + args.seeds):
        rng = np.random.default_rng(seed)
        for _ in range(6):
            n, h, w, c, k, r, s, st, ph, pw, dil = _random_case(rng)
            a = (st, st, ph, pw, dil, dil)
            x = rng.integers(-2, 3, size=(n, h, w, c)).astype(np.int8)
            f = rng.integers(-2, 3, size=(r, s, c, k)).astype(np.int8)
            want = O.conv2d_nhwc_exact_f64(x, f, *a)
            xb = torch.from_numpy(x).cuda().float().bfloat16()
            fb = torch.from_numpy(f).cuda().float().bfloat16()
            xi, fi = torch.from_numpy(x).cuda(), torch.from_numpy(f).cuda()
            wf = torch.from_numpy(want.astype(np.float32)).cuda()
            wi = torch.from_numpy(want.astype(np.int32)).cuda()
            for name, flags, ctas in modes:
                y = conv_device(xb, fb, *a, out_dtype=torch.float32, flags=flags, num_ctas=ctas)
                if not torch.equal(y, wf):
                    print("MISMATCH bf16", name, (n, h, w, c, k, r, s, a), "seed", seed,
                          "max err", (y - wf).abs().max().item())
                    return 1
                if c % 16 == 0 and k % 16 == 0:
                    yi = conv_device(xi, fi, *a, flags=flags, num_ctas=ctas)
                    if not torch.equal(yi, wi):
                        print("MISMATCH int8", name, (n, h, w, c, k, r, s, a), "seed", seed)
                        return 1
            cases += 1
    torch.cuda.synchronize()
    print(f"soak ok: {cases} shapes x {len(modes)} launch modes, bf16 and int8, {time.time() - t0:.0f} s")
    return 0


if __name__ == "__main__":
    sys.exit(main())
