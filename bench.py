#!/usr/bin/env python
"""Benchmark of the blocked implicit-im2col convolution on B200.

Default workload (BASELINE.json configs[3], "cfg4"): one step = the 53
convolution layers of ResNet-50 v1.5 at 224x224, batch 256 sharded evenly
over the ranks (strong scaling: the global batch is fixed, each GPU takes 256/N images), bf16 in / bf16 out, fp32
accumulation, synthetic N(0,1) activations and Kaiming weights.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg4] [--impl ours|reference]

Prints ONE JSON line on rank 0 (contract in the task statement):
  value       = whole-job conv TFLOP/s, inputs resident in HBM, device-timed
                (CUDA events, max over ranks), the step captured as a CUDA graph;
  e2e         = the same metric through the public API with pinned HOST
                buffers: H2D of every layer's input+filter, the kernel, D2H of
                every output, inside the timed region;
  roofline    = the conv kernel against the measured bf16 peak;
  cpu_baseline= the CPU oracle port (oracle/, numpy+OpenBLAS taps -- the
                reference's own float algorithm, _fallback.py:17-42) on a
                bounded sample of the same workload, rank 0 only.
--impl reference runs only that CPU implementation (rank 0; others exit 0).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}
METRIC = "conv TFLOP/s (2*N*K*C*R*S*P*Q/time)"


def committed_traffic(config: str):
    """DRAM bytes per step from the newest committed ncu launch list of this
    workload (profiles/r*/launches_*.csv: dram__bytes_read + write summed over
    the step's launches), or None."""
    import csv
    import glob
    if config != "cfg4":
        return None, None
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*", "launches_*.csv")))  # newest round / letter last
    for path in reversed(files):
        try:
            rows = [r for r in csv.reader(open(path)) if len(r) > 10]
            h = rows[0]
            im, iv, iid = h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
            ids = set()
            tot = 0.0
            for r in rows[1:]:
                ids.add(r[iid])
                if r[im] in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                    tot += float(r[iv].replace(",", ""))
            if len(ids) == 53 and tot > 0:
                return tot, os.path.relpath(path, ROOT)
        except Exception:
            continue
    return None, None


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
        return d, "measured"
    except Exception:
        return dict(PEAKS_FALLBACK), "fallback"


# ------------------------------------------------------------------ helpers

class ClockSampler:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md)."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []
        self._t = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self._t = threading.Thread(target=self._read, daemon=True)
        self._t.start()

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        if self._t:
            self._t.join(timeout=2)
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax = float(parts[2])
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_setup():
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 and not dist.is_initialized():
        dist.init_process_group("nccl" if torch.cuda.is_available() else "gloo")
    return world, rank, local


def shard_batch(n_total: int, world: int, rank: int):
    """Even N-sharding; ranks get contiguous image ranges."""
    from paper_2110_03901_b200.sharding import shard_range
    return shard_range(n_total, world, rank)


def cpu_threads():
    try:
        from threadpoolctl import threadpool_info
        info = threadpool_info()
        blas = [d.get("num_threads") for d in info if d.get("user_api") == "blas"]
        if blas:
            return int(blas[0])
    except Exception:
        pass
    return os.cpu_count() or 1


# ------------------------------------------------------------------ CPU arm

def cpu_reference_step(layers, n_sample: int, seed: int = 1):
    """The reference's CPU algorithm (oracle port: per-tap strided slice @
    w[r,s] through OpenBLAS, _fallback.py:17-42; int8 layers through the int64
    loop, _native.pyx:20-47) over every layer at batch n_sample.  Returns
    (seconds, flops)."""
    import numpy as np
    from oracle import oracle as O
    from paper_2110_03901_b200.workloads import synthetic_operands

    secs, flops = 0.0, 0
    for layer in layers:
        sp = layer.spec.with_batch(n_sample)
        x, w = synthetic_operands(layer, seed=seed, n=n_sample)
        if layer.dtype == "int8":
            xn, wn = x.numpy(), w.numpy()
            t0 = time.perf_counter()
            O.conv2d_nhwc_i64(xn, wn, *sp.conv_args(), threads=cpu_threads())
        else:
            xn, wn = x.float().numpy(), w.float().numpy()
            t0 = time.perf_counter()
            O.conv2d_nhwc_taps(xn, wn, *sp.conv_args())
        secs += time.perf_counter() - t0
        flops += sp.flops
        del x, w
    return secs, flops


def run_reference_arm(args, layers, world, rank):
    if rank != 0:
        return 0
    # torchrun exports OMP_NUM_THREADS=1 to every rank; the reference arm is rank 0 alone,
    # so it takes all host threads for OpenBLAS
    try:
        from threadpoolctl import threadpool_limits
        threadpool_limits(limits=os.cpu_count() or 1, user_api="blas")
    except Exception:
        pass
    n_sample = args.ref_sample
    for _ in range(args.warmup):
        cpu_reference_step(layers[:1], 1)
    times, flops = [], 0
    for _ in range(args.steps):
        s, flops = cpu_reference_step(layers, n_sample)
        times.append(s)
    mean_s = sum(times) / len(times)
    value = flops / mean_s / 1e12
    cores = cpu_threads()
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": mean_s * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": args.config, "sample_batch": n_sample, "layers": len(layers)},
        "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": cores, "kind": "port",
                         "sample": f"{args.config} all {len(layers)} layers at batch {n_sample} per step "
                                   f"(fp32 BLAS tap accumulation on bf16-rounded operands)"},
        "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ GPU arm

def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="cfg4", choices=["cfg1", "cfg2", "cfg3", "cfg4", "cfg5"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--ref-sample", type=int, default=4, help="batch per layer of one --impl reference step")
    ap.add_argument("--cpu-sample", type=int, default=32, help="batch per layer of the cpu_baseline sample")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--layers-json", default=None, help="write per-layer timings here (rank 0)")
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--emulate-world", type=int, default=0,
                    help="diagnostic (1 process): run rank 0's shard of a W-rank job and report W x its "
                         "throughput, i.e. what the W-GPU run measures when every rank matches rank 0")
    args = ap.parse_args(argv)

    from paper_2110_03901_b200.workloads import baseline_configs
    layers_full = baseline_configs()[args.config]
    world, rank, local = dist_setup()
    if args.impl == "reference":
        return run_reference_arm(args, layers_full, world, rank)

    import torch
    import torch.distributed as dist
    import paper_2110_03901_b200 as P
    from paper_2110_03901_b200 import _lib
    from paper_2110_03901_b200._kernels import conv_device
    from paper_2110_03901_b200.lowering import touched_pixels
    # the weights are written once at setup, never inside the step: every conv may start
    # its filter loads before its programmatic-launch wait (IMCONV_FLAG_STATIC_FILTER)
    STATIC = _lib.FLAG_STATIC_FILTER

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    peaks, peak_kind = load_peaks()

    # ---- per-rank shard of every layer (contiguous images; no collective) ----
    shard_world = world
    if args.emulate_world > 1:
        if world != 1:
            raise SystemExit("--emulate-world is a single-process diagnostic")
        shard_world = args.emulate_world
    work = []
    for li, layer in enumerate(layers_full):
        lo, hi = shard_batch(layer.spec.n, shard_world, rank)
        sp = layer.spec.with_batch(hi - lo)
        g = torch.Generator(device=dev).manual_seed(1000 + li)
        xs = (sp.n, sp.h_i, sp.w_i, sp.c_i)
        ws = (sp.h_f, sp.w_f, sp.c_i, sp.c_o)
        gw = torch.Generator(device=dev).manual_seed(2000 + li)  # identical weights on every rank
        if layer.dtype == "int8":
            x = torch.randint(-128, 128, xs, generator=g, device=dev, dtype=torch.int16).to(torch.int8)
            w = torch.randint(-128, 128, ws, generator=gw, device=dev, dtype=torch.int16).to(torch.int8)
            y = torch.empty((sp.n, sp.h_o, sp.w_o, sp.c_o), dtype=torch.int32, device=dev)
        else:
            x = torch.randn(xs, generator=g, device=dev, dtype=torch.float32)
            if layer.relu_input:
                x.clamp_(min=0)
            w = torch.randn(ws, generator=gw, device=dev, dtype=torch.float32) * (2.0 / (sp.c_i * sp.h_f * sp.w_f)) ** 0.5
            if layer.name == "stem":
                x[..., 3:] = 0
                w[:, :, 3:, :] = 0
            x, w = x.to(torch.bfloat16), w.to(torch.bfloat16)
            y = torch.empty((sp.n, sp.h_o, sp.w_o, sp.c_o), dtype=torch.bfloat16, device=dev)
        work.append((layer, sp, x, w, y))
    torch.cuda.synchronize()

    def step():
        for layer, sp, x, w, y in work:
            conv_device(x, w, *sp.conv_args(), y=y, flags=STATIC)

    total_flops_rank = sum(sp.flops for _, sp, *_ in work)
    e_in = {"int8": 1}
    bytes_alg_rank = 0
    for layer, sp, x, w, y in work:
        ei = e_in.get(layer.dtype, 2)
        bytes_alg_rank += sp.n * touched_pixels(sp) * sp.c_i * ei + sp.h_f * sp.w_f * sp.c_i * sp.c_o * ei \
            + sp.gemm_m * sp.c_o * y.element_size()

    # Consecutive timed steps must not find their inputs in L2: when one step's working set is
    # below twice the L2 size (the small parity configs), the step rotates over `copies`
    # independent sets of buffers (same values), so every step reads cold data.
    l2_bytes = int(getattr(torch.cuda.get_device_properties(dev), "L2_cache_size", 126 << 20))
    copies = 1 if bytes_alg_rank >= 2 * l2_bytes else -(-2 * l2_bytes // max(bytes_alg_rank, 1))
    work_sets = [work] + [[(layer, sp, x.clone(), w.clone(), torch.empty_like(y)) for layer, sp, x, w, y in work]
                          for _ in range(copies - 1)]
    l2_note = (f"inputs larger than L2: every layer has its own buffers, per-step working set "
               f"{bytes_alg_rank / 1e9:.1f} GB per GPU" if copies == 1 else
               f"steps rotate over {copies} copies of the {bytes_alg_rank / 1e6:.1f} MB working set "
               f"({copies * bytes_alg_rank / 1e6:.0f} MB > 2 x L2), so no step reads L2-resident inputs")

    def step_set(ws):
        for layer, sp, x, w, y in ws:
            conv_device(x, w, *sp.conv_args(), y=y, flags=STATIC)

    # launches per step (our kernels only)
    _lib.lib.imconv_reset_launch_count()
    step()
    torch.cuda.synchronize()
    launches_per_step = int(_lib.lib.imconv_launch_count())

    stream = torch.cuda.Stream()
    graphs = []
    if not args.no_graph:
        stream.wait_stream(torch.cuda.current_stream())
        for ws in work_sets:
            with torch.cuda.stream(stream):
                step_set(ws)  # warm caches outside capture
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=stream):
                step_set(ws)
            graphs.append(g)
        torch.cuda.synchronize()
    graph = graphs[0] if graphs else None
    step_ctr = [0]

    def run_step():
        i = step_ctr[0] % copies
        step_ctr[0] += 1
        if graphs:
            graphs[i].replay()
        else:
            step_set(work_sets[i])

    for _ in range(max(args.warmup, 3)):
        run_step()
    torch.cuda.synchronize()

    # ---- timed region: K back-to-back steps ----
    sampler = ClockSampler(local)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    sampler.start()
    time.sleep(0.3)  # let the sampler attach
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    cur = torch.cuda.current_stream()
    ev0.record(cur)
    for _ in range(args.steps):
        run_step()
    ev1.record(cur)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = sampler.stop()
    ms_rank = ev0.elapsed_time(ev1) / args.steps
    ms = ms_rank
    if world > 1:
        t = torch.tensor([ms_rank], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    total_flops = sum(l.spec.flops for l in layers_full)  # all ranks together
    if shard_world != world:  # emulated: every rank assumed as fast as rank 0
        total_flops = total_flops_rank * shard_world
    value = total_flops / (ms / 1e3) / 1e12

    # ---- per-layer kernel times (separate pass): each layer's `reps` launches
    # are replayed from their own CUDA graph, so host launch latency cannot
    # starve short kernels ----
    per_layer = []
    reps = 5
    side = torch.cuda.Stream()
    for layer, sp, x, w, y in work:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=side):
            for _ in range(reps):
                conv_device(x, w, *sp.conv_args(), y=y, flags=STATIC)
        g.replay()
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        evs[0].record()
        g.replay()
        evs[1].record()
        torch.cuda.synchronize()
        per_layer.append((layer, sp, evs[0].elapsed_time(evs[1]) / reps))
        del g
    kern_ms = sum(t for *_, t in per_layer)
    int8_peak = None
    if any(l.dtype == "int8" for l, *_ in work):
        # MEASURED_PEAKS.json has no int8 entry: measure cuBLAS int8 (torch._int_mm) here
        a8 = torch.randint(-128, 128, (8192, 8192), device=dev, dtype=torch.int8)
        b8 = torch.randint(-128, 128, (8192, 8192), device=dev, dtype=torch.int8)
        for _ in range(2):
            torch._int_mm(a8, b8)
        best = None
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            torch._int_mm(a8, b8)
            e1.record()
            torch.cuda.synchronize()
            t = e0.elapsed_time(e1)
            best = t if best is None else min(best, t)
        int8_peak = 2 * 8192 ** 3 / (best / 1e3) / 1e12
        del a8, b8
    dtype_peak = peaks.get("bf16_tflops_sustained", PEAKS_FALLBACK["bf16_tflops_sustained"])
    if int8_peak is not None and all(l.dtype == "int8" for l, *_ in work):
        dtype_peak = int8_peak
    hbm = peaks.get("hbm_gbs", PEAKS_FALLBACK["hbm_gbs"])
    # achieved: this rank's FLOP over its device time per step in the TIMED region (the step
    # is nothing but the conv kernels); the separate per-layer pass only apportions it
    achieved = total_flops_rank / (ms_rank / 1e3) / 1e12
    roof_ms = 0.0
    layer_rows = []
    for layer, sp, t_ms in per_layer:
        ei = e_in.get(layer.dtype, 2)
        eo = 4 if layer.dtype == "int8" else 2
        b = sp.n * touched_pixels(sp) * sp.c_i * ei + sp.h_f * sp.w_f * sp.c_i * sp.c_o * ei + sp.gemm_m * sp.c_o * eo
        pk = int8_peak if (layer.dtype == "int8" and int8_peak) else dtype_peak
        t_roof = max(sp.flops / (pk * 1e12), b / (hbm * 1e9)) * 1e3
        roof_ms += t_roof
        layer_rows.append({"layer": layer.name, "n": sp.n, "ms": round(t_ms, 5),
                           "tflops": round(sp.flops / (t_ms / 1e3) / 1e12, 2),
                           "gbs": round(b / (t_ms / 1e3) / 1e9, 1),
                           "roofline_frac": round(t_roof / t_ms, 3)})

    # ---- e2e through the public API with pinned host buffers ----
    e2e = None
    if not args.no_e2e:
        host = {}
        for layer, sp, x, w, y in work:
            key = (sp, layer.dtype)
            if key not in host:
                host[key] = (x.cpu().pin_memory(), w.cpu().pin_memory(),
                             torch.empty(y.shape, dtype=y.dtype, pin_memory=True))
        h2d = d2h = 0
        for layer, sp, x, w, y in work:
            hx, hw, hy = host[(sp, layer.dtype)]
            h2d += hx.numel() * hx.element_size() + hw.numel() * hw.element_size()
            d2h += hy.numel() * hy.element_size()

        def e2e_step():
            # the public API with pinned HOST tensors: upload, conv and download
            # of each layer (the pipelined host path of _kernels.conv2d_nhwc)
            for layer, sp, x, w, y in work:
                hx, hw, hy = host[(sp, layer.dtype)]
                P._kernels.conv2d_nhwc(hx, hw, *sp.conv_args(), out=hy)

        e2e_step()
        torch.cuda.synchronize()
        k_e2e = max(1, min(args.steps, 3))
        if world > 1:
            dist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(k_e2e):
            e2e_step()
        b.record()
        torch.cuda.synchronize()
        e_ms = a.elapsed_time(b) / k_e2e
        if world > 1:
            t = torch.tensor([e_ms], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e_ms = float(t.item())
        e2e = {"value": total_flops / (e_ms / 1e3) / 1e12, "unit": "TFLOP/s", "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "ms_per_step": e_ms}

    # ---- CPU baseline (rank 0, N=1 only) ----
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        s, f = cpu_reference_step(layers_full, args.cpu_sample)
        cpu = {"value": f / s / 1e12, "unit": "TFLOP/s", "cores": cpu_threads(), "kind": "port",
               "sample": f"{args.config}: all {len(layers_full)} layers at batch {args.cpu_sample} "
                         f"(oracle port of _fallback.conv2d_nhwc, fp32 OpenBLAS, {s:.1f} s)"}

    traffic, traffic_src = committed_traffic(args.config)
    # the stem executes C = 8 (3 image channels zero-padded, as BASELINE.json defines it);
    # the same run with only the 3 useful channels counted
    useful_value = None
    stem = [sp for layer, sp, *_ in work if layer.name == "stem" and sp.c_i == 8]
    if stem:
        useful_value = value * (total_flops_rank - stem[0].flops * 5 / 8) / total_flops_rank
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "bf16" if args.config != "cfg5" else "int8", "data": "synthetic",
            "config": {"workload": args.config + (" (ResNet-50 v1.5, 53 convs, 224x224)" if args.config == "cfg4" else ""),
                       "global_batch": layers_full[0].spec.n, "per_gpu_batch": work[0][1].n,
                       "parallelism": f"dp{world} (N-sharded, no collective)",
                       "l2": l2_note,
                       "cuda_graph": graph is not None,
                       **({"value_stem_c3": useful_value} if useful_value is not None else {})},
            **({"emulated_world": shard_world} if shard_world != world else {}),
            "pct_of_peak": {"measured_sustained": value / shard_world / dtype_peak,
                            "unit_peak": "int8 TOPS" if dtype_peak == int8_peak else "bf16 TFLOP/s",
                            "measured_burst": value / shard_world / (dtype_peak if dtype_peak == int8_peak
                                                               else peaks.get("bf16_tflops", 1648.9)),
                            "datasheet": value / shard_world / (4500.0 if dtype_peak == int8_peak else 2250.0)},
            "roofline": {"bound": "tensor", "achieved": achieved, "peak": dtype_peak, "unit": "TFLOP/s",
                         "frac": achieved / dtype_peak,
                         "traffic": None if traffic is None else traffic / world,
                         "traffic_unit": "DRAM bytes per step per GPU (ncu dram__bytes_read+write)",
                         "traffic_source": traffic_src,
                         "bytes_alg": bytes_alg_rank,
                         "peak_kind": (f"cuBLAS int8 (torch._int_mm 8192^3) measured in this run"
                                       if int8_peak is not None and dtype_peak == int8_peak
                                       else f"{peak_kind} bf16 sustained (MEASURED_PEAKS.json)"),
                         "kernel": "conv kernels (generic / row-band / halo), all layers of the step",
                         "achieved_source": "timed region: rank FLOP / device ms per step",
                         "roofline_limited_frac": roof_ms / ms_rank},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches_per_step * args.steps,
            "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
        if args.layers_json:
            with open(args.layers_json, "w") as fh:
                json.dump({"config": args.config, "world": world, "kernel_ms": kern_ms, "roofline_ms": roof_ms,
                           "layers": layer_rows}, fh, indent=1)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
