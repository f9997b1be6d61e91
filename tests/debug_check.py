#!/usr/bin/env python
"""Run every kernel path of the library through the debug-invariant build
(libimconv_debug.so, -DIMCONV_DEBUG=1) and check the outputs against the CPU oracle.

The debug build traps on a violated pipeline invariant (mbarrier phase watchdog,
TMEM allocation range, split-K / stream-K ticket overrun, work-unit range,
staged vs stored epilogue chunk counts) and rejects a planner schedule whose waits
could deadlock (host check) -- the stand-in for compute-sanitizer, which this pool
does not offer.  Integer-valued operands: every checked image must be bit-exact.

  python tests/debug_check.py        (GPU; exit code 0 = every case ran clean and exact)

Test infrastructure (it checks against the oracle): run by tests/test_gpu_bench_batches.py.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

STREAM_K = 1 << 29  # imconv_api.cu kDbgStreamK (opt-in planner switch)


def cases():
    from paper_2110_03901_b200.core import ConvSpec
    sq = ConvSpec.square
    bf, i8 = "bf16", "int8"
    return [  # (label, spec, dtype, flags, host debug flags)
        ("1x1, filter slice resident", sq(256, 256, 14, 1024, 1), bf, 0, 0),
        ("1x1, CTA pairs", sq(256, 1024, 14, 256, 1), bf, 0, 0),
        ("3x3, CTA pairs + split tail", sq(256, 512, 7, 512, 3, stride=1, pad=1), bf, 0, 0),
        ("3x3, sub-wave split", sq(32, 512, 7, 512, 3, stride=1, pad=1), bf, 0, 0),
        ("3x3, CTA pairs stream-K", sq(256, 256, 14, 256, 3, stride=1, pad=1), bf, 0, STREAM_K),
        ("3x3, single-CTA stream-K", sq(128, 128, 28, 128, 3, stride=1, pad=1), bf, 0, STREAM_K),
        ("3x3 stride 2", sq(8, 128, 28, 128, 3, stride=2, pad=1), bf, 0, 0),
        ("3x3 dilation 2", sq(4, 128, 24, 128, 3, stride=1, pad=2, dilation=2), bf, 0, 0),
        ("small-C tap packing", sq(4, 32, 20, 64, 3, stride=1, pad=1), bf, 0, 0),
        ("channel-last baseline", sq(2, 64, 12, 64, 3, stride=2, pad=1), bf, 64, 0),
        ("7x7 stem (C = 8)", sq(4, 8, 224, 64, 7, stride=2, pad=3), bf, 0, 0),
        ("3x3 C=64 halo tiles", sq(8, 64, 56, 64, 3, stride=1, pad=1), bf, 0, 0),
        ("3x3 C=64 halo tiles, CTA pairs", sq(64, 64, 56, 64, 3, stride=1, pad=1), bf, 0, 0),
        ("3x3 C=128 streamed-filter halo", sq(64, 128, 28, 128, 3, stride=1, pad=1), bf, 0, 0),
        ("int8 3x3, CTA pairs", sq(64, 256, 28, 256, 3, stride=1, pad=1), i8, 0, 0),
        ("int8 3x3, CTA pairs + split tail", sq(128, 1024, 7, 1024, 3, stride=1, pad=1), i8, 0, 0),
        ("int8 3x3, sub-wave split", sq(16, 1024, 7, 1024, 3, stride=1, pad=1), i8, 0, 0),
        ("int8 3x3 stride 2", sq(16, 256, 28, 256, 3, stride=2, pad=1), i8, 0, 0),
    ]


def main():
    import numpy as np
    import torch
    from paper_2110_03901_b200 import _lib
    _lib.use_debug()
    from paper_2110_03901_b200._kernels import conv_device
    from paper_2110_03901_b200.traffic import plan
    from oracle import oracle as O
    dev = torch.device("cuda", 0)
    rng = np.random.default_rng(3)
    bad = 0
    for label, sp, dt, flags, host in cases():
        _lib.lib.imconv_debug_set_flags(host)
        pl = plan(sp, dtype=dt, flags=flags)
        lim = 42 if dt == "int8" else 2
        x = rng.integers(-lim, lim + 1, size=(sp.n, sp.h_i, sp.w_i, sp.c_i))
        w = rng.integers(-lim, lim + 1, size=(sp.h_f, sp.w_f, sp.c_i, sp.c_o))
        tdt = torch.int8 if dt == "int8" else torch.bfloat16
        odt = torch.int32 if dt == "int8" else torch.float32
        try:
            y = conv_device(torch.from_numpy(x).to(dev).to(tdt), torch.from_numpy(w).to(dev).to(tdt),
                            *sp.conv_args(), out_dtype=odt, flags=flags)
            torch.cuda.synchronize()
        except Exception as e:  # noqa: BLE001 -- a trap poisons the CUDA context: report and stop
            print(f"FAIL {label}: {type(e).__name__}: {e}", flush=True)
            return 2
        finally:
            _lib.lib.imconv_debug_set_flags(0)
        imgs = sorted({0, sp.n // 2, sp.n - 1})
        want = O.conv2d_nhwc_exact_f64(x[imgs], w, *sp.conv_args())
        got = y[imgs].cpu().numpy().astype(np.float64)
        ok = np.array_equal(got, want)
        bad += 0 if ok else 1
        print(f"{'ok  ' if ok else 'FAIL'} {label} (plan: {pl.branch})", flush=True)
    print("debug build: all cases clean and exact" if bad == 0 else f"debug build: {bad} case(s) differ")
    return 0 if bad == 0 else 1


if __name__ == "__main__":
    sys.exit(main())
