#!/usr/bin/env python
"""Run one BASELINE layer a few times on cuda:0 (for ncu / quick timing).

  python tools/run_layer.py --layer stem [--n 256] [--reps 5] [--tile-n 0] [--order reuse_aware]
"""

import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layer", default="stem")
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--tile-n", type=int, default=0)
    ap.add_argument("--order", default="reuse_aware")
    ap.add_argument("--flags", type=int, default=0, help="imconv flags: 1 = single CTA, 2 = CTA pair")
    ap.add_argument("--explicit", action="store_true", help="K3 im2col + K4 GEMM instead of the implicit kernel")
    ap.add_argument("--waits", action="store_true", help="print per-role wait-cycle instrumentation")
    ap.add_argument("--dbg-flags", type=int, default=0, help="instrumentation: disable kernel roles (wrong results)")
    ap.add_argument("--once", action="store_true", help="one launch, no timing (for ncu --set full)")
    ap.add_argument("--host-flags", type=lambda v: int(v, 0), default=0,
                    help="host-side A/B switches of imconv_debug_set_flags (bits 16+, experiments only)")
    ap.add_argument("--rps", type=int, default=0, help="row-band kernel: input rows per stage override (0 = auto)")
    args = ap.parse_args()
    import torch
    from paper_2110_03901_b200 import _lib
    if args.waits or args.dbg_flags:
        _lib.use_instrumented()
    from paper_2110_03901_b200._kernels import conv_device, gemm_device
    from paper_2110_03901_b200.workloads import baseline_configs
    import paper_2110_03901_b200._kernels as K

    layers = {l.name: l for cfg in baseline_configs().values() for l in cfg}
    for name in args.layer.split(","):  # several layers: one process (one ncu run covers them all)
        run_one(args, layers[name])


def run_one(args, layer):
    import torch
    from paper_2110_03901_b200 import _lib
    from paper_2110_03901_b200._kernels import conv_device, gemm_device
    import paper_2110_03901_b200._kernels as K

    sp = layer.spec if args.n is None else layer.spec.with_batch(args.n)
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    if layer.dtype == "int8":
        x = torch.randint(-128, 128, (sp.n, sp.h_i, sp.w_i, sp.c_i), device=dev, dtype=torch.int16).to(torch.int8)
        w = torch.randint(-128, 128, (sp.h_f, sp.w_f, sp.c_i, sp.c_o), device=dev, dtype=torch.int16).to(torch.int8)
    else:
        x = torch.randn((sp.n, sp.h_i, sp.w_i, sp.c_i), device=dev).to(torch.bfloat16)
        w = (torch.randn((sp.h_f, sp.w_f, sp.c_i, sp.c_o), device=dev) * 0.05).to(torch.bfloat16)
    order = {"reuse_aware": _lib.ORDER_REUSE_AWARE, "filter_major": _lib.ORDER_FILTER_MAJOR}[args.order]
    _lib.lib.imconv_debug_set_flags(args.dbg_flags | (args.rps << 8) | args.host_flags)
    def once():
        if args.explicit:
            low = K.im2col_nhwc(x, sp.h_f, sp.w_f, *sp.conv_args(), True)
            gemm_device(low, w.reshape(-1, sp.c_o))
        else:
            conv_device(x, w, *sp.conv_args(), tile_n=args.tile_n, order=order, flags=args.flags)

    once()
    torch.cuda.synchronize()
    if args.once:
        print(f"{layer.name}: launched once")
        return
    # the timed launches are replayed from a CUDA graph so host-side launch
    # latency (ctypes + tensor-map encoding) cannot starve short kernels
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(args.reps):
            once()
    g.replay()
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record()
    g.replay()
    ev[1].record()
    torch.cuda.synchronize()
    ms = ev[0].elapsed_time(ev[1]) / args.reps
    print(f"{layer.name} n={sp.n}: {ms:.4f} ms  {sp.flops / ms / 1e9:.1f} TFLOP/s")
    if args.waits:
        dbg = torch.zeros(148 * 20, dtype=torch.int64, device=dev)
        _lib.lib.imconv_debug_set_buffer(dbg.data_ptr())
        conv_device(x, w, *sp.conv_args(), tile_n=args.tile_n, order=order)
        torch.cuda.synchronize()
        _lib.lib.imconv_debug_set_buffer(None)
        d = dbg[:148 * 8].view(148, 8).double().mean(0).tolist()
        names = ["prod_total", "prod_wait_empty", "mma_total", "mma_wait_tempty", "mma_wait_full",
                 "epi_total", "epi_wait_tfull", "epi_tmem_ld"]
        print("  ".join(f"{nm}={v / 1e3:.1f}k" for nm, v in zip(names, d)))
        e = dbg[148 * 8:148 * 12].view(148, 4).double().mean(0).tolist()
        sk = dbg[148 * 12:].view(148, 8)
        if int(sk[:, 5].abs().sum()) > 0:
            used = sk[sk[:, 5] != 0].double()
            print(f"  split-K units ({used.shape[0]} CTAs, cycles, mean/max): " + "  ".join(
                f"{nm}={used[:, i].mean() / 1e3:.2f}k/{used[:, i].max() / 1e3:.2f}k" for i, nm in enumerate(
                    ["write_partials", "fence+bar", "arrive+spin", "bulk_wait", "reduce+stage", "start->tfull"])))
        print("  extra (generic: epi barriers+store waits, epi staging; row-band: issuer commit, issuer mma loop, "
              "producer fence+arrive, producer wait_group): " + "  ".join(f"{v / 1e3:.1f}k" for v in e))


if __name__ == "__main__":
    main()
