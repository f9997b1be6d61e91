#!/usr/bin/env python
"""Explicit im2col + GEMM vs the implicit kernel (north_star (d); paper §2.2,
PAPER.md:117-162): time and bytes of both paths per layer, on one GPU.

  python tools/overhead.py [--config cfg4] [--n 64] [--json out.json]

explicit = K3 (im2col_cf_vec16_kernel: lowered (NPQ, RSC) matrix written to
HBM) + K4 (the same tcgen05 kernel as a 1x1 GEMM over the lowered matrix);
implicit = the blocked implicit-im2col kernel.  Both are replayed from CUDA
graphs (host launch latency excluded).  Bytes: algorithmic traffic of each
path (explicit adds 2 x lowered bytes: write + read); the ncu-measured DRAM
bytes of both paths come from a separate ncu pass (see --ncu-csv).
"""

import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg4")
    ap.add_argument("--n", type=int, default=64, help="batch per layer (cfg4 default 64 keeps the lowered matrix "
                                                      "of the stem at 2.5 GB)")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--json", default=None)
    ap.add_argument("--once", action="store_true", help="single untimed pass of both paths (for ncu)")
    args = ap.parse_args()

    import torch
    from paper_2110_03901_b200 import _kernels as K
    from paper_2110_03901_b200._kernels import conv_device, gemm_device
    from paper_2110_03901_b200.lowering import lowered_memory_footprint, touched_pixels
    from paper_2110_03901_b200.workloads import baseline_configs

    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    seen = set()
    rows = []
    for layer in baseline_configs()[args.config]:
        sp = layer.spec.with_batch(min(args.n, layer.spec.n))
        if (sp, layer.dtype) in seen:
            continue
        seen.add((sp, layer.dtype))
        if layer.dtype == "int8":
            x = torch.randint(-128, 128, (sp.n, sp.h_i, sp.w_i, sp.c_i), device=dev, dtype=torch.int16).to(torch.int8)
            w = torch.randint(-128, 128, (sp.h_f, sp.w_f, sp.c_i, sp.c_o), device=dev, dtype=torch.int16).to(torch.int8)
        else:
            x = torch.randn((sp.n, sp.h_i, sp.w_i, sp.c_i), device=dev).to(torch.bfloat16)
            w = (torch.randn((sp.h_f, sp.w_f, sp.c_i, sp.c_o), device=dev) * 0.05).to(torch.bfloat16)
        wl = w.reshape(-1, sp.c_o)

        def implicit():
            return conv_device(x, w, *sp.conv_args())

        def explicit():
            low = K.im2col_nhwc(x, sp.h_f, sp.w_f, *sp.conv_args(), True)
            return gemm_device(low, wl)

        if args.once:
            implicit()
            explicit()
            torch.cuda.synchronize()
            continue
        # correctness of the explicit path against the implicit one
        yi, ye = implicit().float(), explicit().float().reshape(sp.n, sp.h_o, sp.w_o, sp.c_o)
        err = float((yi - ye).abs().max() / yi.abs().max().clamp_min(1e-30))
        times = {}
        for name, fn in (("implicit", implicit), ("explicit", explicit)):
            fn()
            torch.cuda.synchronize()
            s = torch.cuda.Stream()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                for _ in range(args.reps):
                    fn()
            g.replay()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            g.replay()
            e1.record()
            torch.cuda.synchronize()
            times[name] = e0.elapsed_time(e1) / args.reps
            del g
        e = 1 if layer.dtype == "int8" else 2
        eo = 4 if layer.dtype == "int8" else 2
        alg_impl = sp.n * touched_pixels(sp) * sp.c_i * e + sp.h_f * sp.w_f * sp.c_i * sp.c_o * e + \
            sp.gemm_m * sp.c_o * eo
        lowered = lowered_memory_footprint(sp, e)["lowered_bytes"]
        alg_expl = alg_impl + 2 * lowered
        rows.append({"layer": layer.name, "n": sp.n, "implicit_ms": round(times["implicit"], 5),
                     "explicit_ms": round(times["explicit"], 5),
                     "slowdown": round(times["explicit"] / times["implicit"], 3),
                     "lowered_MB": round(lowered / 1e6, 1),
                     "lowered_over_ifmap": round(lowered_memory_footprint(sp, e)["ratio"], 2),
                     "alg_bytes_implicit_MB": round(alg_impl / 1e6, 1),
                     "alg_bytes_explicit_MB": round(alg_expl / 1e6, 1), "max_rel_diff": err})
        print(json.dumps(rows[-1]), flush=True)
        del x, w, yi, ye
        torch.cuda.empty_cache()
    if rows:
        ti = sum(r["implicit_ms"] for r in rows)
        te = sum(r["explicit_ms"] for r in rows)
        print(json.dumps({"summary": args.config, "unique_layers": len(rows), "implicit_ms": round(ti, 4),
                          "explicit_ms": round(te, 4), "explicit_over_implicit": round(te / ti, 3)}))
        if args.json:
            json.dump({"config": args.config, "n": args.n, "layers": rows}, open(args.json, "w"), indent=1)


if __name__ == "__main__":
    main()
