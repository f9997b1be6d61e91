#!/usr/bin/env python
"""Benchmark of the blocked implicit-im2col convolution on B200.

Default workload (BASELINE.json configs[3], "cfg4"): one step = the 53
convolution layers of ResNet-50 v1.5 at 224x224, batch 256 sharded evenly
over the ranks (strong scaling: the global batch is fixed, each GPU takes 256/N
images), bf16 in / bf16 out, fp32 accumulation, synthetic N(0,1) activations
and Kaiming weights.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg4] [--impl ours|reference]

``--gpus N`` (N > 1) without a torchrun environment re-launches this script
under ``torch.distributed.run`` with N ranks, one GPU each (NCCL); under
torchrun the ranks read RANK / LOCAL_RANK / WORLD_SIZE.

Prints ONE JSON line on rank 0 (contract in the task statement):
  value       = whole-job conv TFLOP/s, inputs resident in HBM, device-timed
                (CUDA events, max over ranks), the step captured as a CUDA graph;
  e2e         = the same metric through the public API with pinned HOST
                buffers: H2D of every layer's input+filter, the kernel, D2H of
                every output, inside the timed region;
  roofline    = the conv kernels against the measured bf16 peak (burst peak for
                a timed region under 1 s, sustained above);
  parity      = after the timed region every layer's output shards are
                all-gathered (NCCL) and the first and last image of every
                rank's shard are checked against the CPU oracle;
  cpu_baseline= the reference's own CPU kernels compiled from its sources
                (oracle/_ref: _fallback.conv2d_nhwc, _fallback.py:17-42, for
                floats; _native.conv2d_nhwc, _native.pyx:20-47, for ints), else
                the oracle port, on a bounded sample of the same workload,
                rank 0 only.
--impl reference runs only that CPU implementation (rank 0; others exit 0) on
the same workload and prints the same `config`.
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}
METRIC = "conv TFLOP/s (2*N*K*C*R*S*P*Q/time)"
L2_BYTES = 126 * 1024 * 1024       # B200 L2 (both dies): the rotation decision must not depend on the arm
BURST_REGION_MS = 1000.0           # timed regions shorter than this are compared with the burst peak
PARITY_TOL = 1e-2                  # north_star: normalised max error of bf16 output vs the fp32 oracle


# ------------------------------------------------------------------ helpers

def csrc_fingerprint() -> str:
    """sha256 over the kernel sources and the C ABI header: committed ncu traffic is
    reported only for the build it was captured from."""
    h = hashlib.sha256()
    csrc = os.path.join(ROOT, "paper_2110_03901_b200", "csrc")
    for name in sorted(os.listdir(csrc)):
        if name.endswith((".cu", ".cuh", ".h", ".cpp")):
            h.update(name.encode())
            with open(os.path.join(csrc, name), "rb") as fh:
                h.update(fh.read())
    with open(os.path.join(ROOT, "include", "imconv.h"), "rb") as fh:
        h.update(fh.read())
    return h.hexdigest()[:16]


def committed_traffic(config: str, world: int):
    """DRAM bytes per step per GPU from the committed ncu summary of this workload
    (profiles/traffic_<config>_w<world>.json, written by tools/traffic_summary.py from a
    launch list with dram__bytes_read/write).  Returns (bytes or None, note)."""
    path = os.path.join(ROOT, "profiles", f"traffic_{config}_w{world}.json")
    if not os.path.exists(path):
        return None, f"no committed ncu traffic for {config} at {world} GPU(s)"
    with open(path) as fh:
        d = json.load(fh)
    if d.get("csrc_sha") != csrc_fingerprint():
        return None, f"committed ncu traffic ({d.get('source')}) is from another build of the kernels: not reported"
    return float(d["dram_bytes_per_step"]), (f"committed ncu launch list {d.get('source')} of this build "
                                             f"(csrc {d['csrc_sha']}; not measured in this run)")


def measure_traffic(args, launches: int, timeout_s: float = 420.0):
    """DRAM bytes of one step measured in this run: a child process runs the same workload
    (one pass, eager launches) under `ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,
    gpu__time_duration.sum` and the bytes of that pass's `launches` conv kernels are summed
    (B200_PROFILING.md launch-list recipe).  The child's timings are never reported as a bench
    value; only its DRAM byte counters are.  Returns (bytes per step or None, note, rows)."""
    import csv
    import io
    import shutil
    ncu = shutil.which("ncu") or ("/usr/local/cuda/bin/ncu" if os.path.exists("/usr/local/cuda/bin/ncu") else None)
    if ncu is None:
        return None, "ncu not found", None
    log = os.path.join("/tmp", f"imconv_traffic_{os.getpid()}.csv")
    child = [sys.executable, os.path.abspath(__file__), "--config", args.config, "--traffic-child"]
    if args.emulate_world > 1:
        child += ["--emulate-world", str(args.emulate_world)]
    cmd = [ncu, "--metrics", "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum",
           "--clock-control", "none", "-k", "regex:conv_", "-s", str(launches), "-c", str(launches),
           "--csv", "--log-file", log] + child
    env = dict(os.environ)
    for k in ("RANK", "LOCAL_RANK", "WORLD_SIZE", "MASTER_ADDR", "MASTER_PORT"):
        env.pop(k, None)
    try:
        r = subprocess.run(cmd, stdout=subprocess.DEVNULL, stderr=subprocess.PIPE, text=True,
                           timeout=timeout_s, env=env)
        if r.returncode != 0:
            return None, f"ncu child failed (rc {r.returncode}): {r.stderr.strip()[-200:]}", None
        with open(log) as fh:
            rows = [row for row in csv.reader(io.StringIO(fh.read())) if len(row) > 10]
    except Exception as e:  # noqa: BLE001 -- the measurement is optional; say why it is absent
        return None, f"ncu child failed: {type(e).__name__}: {e}", None
    finally:
        if os.path.exists(log):
            os.remove(log)
    if len(rows) < 2:  # e.g. this bench itself runs under ncu (nested profiling is refused)
        return None, "ncu child produced no launch rows", None
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1.0, "usecond": 1e3,
             "msecond": 1e6}
    h = rows[0]
    iid, im, iu, iv, ik = (h.index("ID"), h.index("Metric Name"), h.index("Metric Unit"), h.index("Metric Value"),
                           h.index("Kernel Name"))
    per = {}
    for row in rows[1:]:
        d = per.setdefault(row[iid], {"kernel": row[ik].split("(")[0].replace("void ", "")})
        d[row[im]] = float(row[iv].replace(",", "")) * scale.get(row[iu], 1.0)
    if len(per) != launches:
        return None, f"ncu child profiled {len(per)} launches, expected {launches}", None
    total = sum(d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0) for d in per.values())
    return total, (f"measured in this run: ncu dram__bytes_read+write summed over the {launches} conv launches "
                   f"of one eager pass of the same workload in a child process"), list(per.values())


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
        return d, "measured"
    except Exception:
        return dict(PEAKS_FALLBACK), "fallback"


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


def free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def spawn_ranks(n: int, argv) -> int:
    """`--gpus N` outside torchrun: re-launch this script with N ranks (one GPU each).
    Rank 0's stdout carries the JSON line; the exit code is the launcher's."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__)] + list(argv)
    env = dict(os.environ)
    env.setdefault("OMP_NUM_THREADS", "1")
    return subprocess.call(cmd, env=env)


def dist_setup():
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 and not dist.is_initialized():
        if torch.cuda.is_available():
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
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


def use_all_host_threads():
    # torchrun exports OMP_NUM_THREADS=1 to every rank; the CPU legs run on rank 0 alone,
    # so they take every host thread for OpenBLAS
    try:
        from threadpoolctl import threadpool_limits
        threadpool_limits(limits=os.cpu_count() or 1, user_api="blas")
    except Exception:
        pass


def bytes_alg(sp, dtype: str, out_elem: int) -> int:
    """e_in*N*T*C + e_in*R*S*C*K + e_out*N*P*Q*K (T = distinct input pixels touched)."""
    from paper_2110_03901_b200.lowering import touched_pixels
    ei = 1 if dtype == "int8" else 2
    return sp.n * touched_pixels(sp) * sp.c_i * ei + sp.h_f * sp.w_f * sp.c_i * sp.c_o * ei \
        + sp.gemm_m * sp.c_o * out_elem


def rotation_copies(layers, world: int) -> int:
    """Copies of the working set a step rotates over so that no timed pass reads L2-resident
    inputs (1 when one pass already streams more than twice the L2)."""
    b = 0
    for li, layer in enumerate(layers):
        lo, hi = shard_batch(layer.spec.n, world, 0)
        b += bytes_alg(layer.spec.with_batch(hi - lo), layer.dtype, 4 if layer.dtype == "int8" else 2)
    return 1 if b >= 2 * L2_BYTES else -(-2 * L2_BYTES // max(b, 1))


def workload_config(name: str, layers, world: int) -> dict:
    """The `config` object both arms print (identical, so the driver compares like with like)."""
    lo, hi = shard_batch(layers[0].spec.n, world, 0)
    copies = rotation_copies(layers, world)
    per_gpu = 0
    for layer in layers:
        l0, h0 = shard_batch(layer.spec.n, world, 0)
        per_gpu += bytes_alg(layer.spec.with_batch(h0 - l0), layer.dtype, 4 if layer.dtype == "int8" else 2)
    l2 = (f"inputs larger than L2: every layer has its own buffers, per-step working set "
          f"{per_gpu / 1e9:.1f} GB per GPU" if copies == 1 else
          f"each timed pass reads L2-cold inputs: the captured step rotates over {copies} copies of the "
          f"{per_gpu / 1e6:.1f} MB working set ({copies * per_gpu / 1e6:.0f} MB > 2 x L2)")
    cfg = {"workload": name + (" (ResNet-50 v1.5, 53 convs, 224x224)" if name == "cfg4" else ""),
           "global_batch": layers[0].spec.n, "per_gpu_batch": hi - lo, "layers": len(layers),
           "parallelism": f"dp{world} (N-sharded, no collective)", "l2": l2}
    return cfg


def make_operands(layer, sp, li: int, lo: int, dev):
    """Operands of one rank's shard (images [lo, lo + sp.n) of the global batch): seeded by
    (layer, shard start) so any rank -- rank 0 when verifying -- can regenerate any shard;
    weights seeded by the layer alone (replicated on every rank)."""
    import torch
    g = torch.Generator(device=dev).manual_seed(1000 + 7919 * li + lo)
    gw = torch.Generator(device=dev).manual_seed(2000 + li)
    xs = (sp.n, sp.h_i, sp.w_i, sp.c_i)
    ws = (sp.h_f, sp.w_f, sp.c_i, sp.c_o)
    if layer.dtype == "int8":
        x = torch.randint(-128, 128, xs, generator=g, device=dev, dtype=torch.int16).to(torch.int8)
        w = torch.randint(-128, 128, ws, generator=gw, device=dev, dtype=torch.int16).to(torch.int8)
        return x, w
    x = torch.randn(xs, generator=g, device=dev, dtype=torch.float32)
    if layer.relu_input:
        x.clamp_(min=0)
    w = torch.randn(ws, generator=gw, device=dev, dtype=torch.float32) * (2.0 / (sp.c_i * sp.h_f * sp.w_f)) ** 0.5
    if layer.name == "stem":
        x[..., 3:] = 0
        w[:, :, 3:, :] = 0
    return x.to(torch.bfloat16), w.to(torch.bfloat16)


# ------------------------------------------------------------------ CPU legs

def cpu_impl():
    """(conv function, kind, description): the reference's kernels compiled from its
    sources (oracle/_ref) when present, else the oracle port."""
    from oracle import ref as R
    if R.available():
        return R.conv2d_nhwc, "reference", ("the reference's own kernels compiled from its sources "
                                            "(oracle/_ref: _fallback.conv2d_nhwc for floats, "
                                            "_native.conv2d_nhwc for ints)")
    from oracle import oracle as O
    return O.conv_reference, "port", "oracle port of the reference's kernels (oracle/oracle.py)"


def cpu_layer_operands(layer, sp, li: int):
    """Host operands in the reference's dtypes: bf16-rounded floats as fp32 (the GPU arm
    computes on the same bf16 values), ints as int64 (the reference's _norm)."""
    import torch
    x, w = make_operands(layer, sp, li, 0, torch.device("cpu"))
    if layer.dtype == "int8":
        return x.numpy().astype("int64"), w.numpy().astype("int64")
    return x.float().numpy(), w.float().numpy()


def cpu_time_layers(layers, n_sample, conv, reps: int = 1, budget_s: float | None = None):
    """Time `conv` over every layer at batch n_sample (or the full batch when None), `reps`
    passes, layer-outer so each layer's operands are generated once.  Returns the per-pass
    seconds list and the FLOP of one pass."""
    import numpy as np  # noqa: F401
    flops = 0
    per_pass = [0.0] * reps
    for li, layer in enumerate(layers):
        sp = layer.spec if n_sample is None else layer.spec.with_batch(n_sample)
        x, w = cpu_layer_operands(layer, sp, li)
        for r in range(reps):
            t0 = time.perf_counter()
            conv(x, w, *sp.conv_args())
            per_pass[r] += time.perf_counter() - t0
        flops += sp.flops
        del x, w
    return per_pass, flops


def run_reference_arm(args, layers, world, rank, config):
    if rank != 0:
        return 0
    use_all_host_threads()
    conv, kind, desc = cpu_impl()
    for _ in range(args.warmup):  # warm BLAS threads and page in the code: one image per layer
        cpu_time_layers(layers, 1, conv)
    # one full pass first: it sizes how many of the requested passes fit the time budget
    first, flops = cpu_time_layers(layers, None, conv)
    steps = max(1, min(args.steps, int(args.ref_budget_s // max(first[0], 1e-9))))
    times = first
    if steps > 1:
        more, _ = cpu_time_layers(layers, None, conv, reps=steps - 1)
        times = first + more
    mean_s = sum(times) / len(times)
    value = flops / mean_s / 1e12
    cores = cpu_threads() if kind == "port" or layers[0].dtype != "int8" else 1
    from oracle import ref as R
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world,
        "steps": steps, "warmup": args.warmup, "ms_per_step": mean_s * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "int64" if layers[0].dtype == "int8" else "f32",
        "data": "synthetic", "config": config,
        "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": cores, "kind": kind,
                         "sample": f"the whole {args.config} step (all {len(layers)} layers at the global batch "
                                   f"{layers[0].spec.n}) per timed step, {steps} of {args.steps} requested steps "
                                   f"within the {args.ref_budget_s:.0f} s budget; {desc}; bf16-rounded operands "
                                   f"in fp32"},
        "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "steps_requested": args.steps,
        "native_libs": sorted({ln.split()[-1] for ln in open("/proc/self/maps")
                               if ln.rstrip().endswith(".so") and ROOT in ln}),
        "ref_shared_objects": [os.path.relpath(p, ROOT) for p in R.shared_objects()],
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ parity of the benchmarked outputs

def verify_outputs(work, layers_full, world, rank, dev, shard_of, regen, reference_conv):
    """After the timed region: all-gather every layer's output shards (NCCL on GPUs, gloo
    on CPU; sharding.gather_shards) and, on rank 0, check the first and last image of every
    rank's shard against the CPU oracle (int8: bit-exact; bf16: normalised max error <=
    PARITY_TOL).  Mirrors the reference's verify loop (cli.py:230-248): every layer's
    kernel output against the direct convolution.  Returns the parity dict (rank 0) or None."""
    import numpy as np
    import torch
    from paper_2110_03901_b200.sharding import gather_shards
    max_err, checked, bad = 0.0, 0, []
    for li, (layer, sp, x, w, y) in enumerate(work):
        n_total = layers_full[li].spec.n
        y_full = gather_shards(y, n_total) if world > 1 else y
        if rank != 0:
            continue
        wf = w.float().cpu().numpy() if layer.dtype != "int8" else w.cpu().numpy().astype(np.int64)
        for r in range(world):
            lo, hi = shard_of(n_total, r)
            if hi <= lo:
                continue
            xr = x if r == rank else regen(layer, layers_full[li].spec.with_batch(hi - lo), li, lo)
            for i in sorted({lo, hi - 1}):
                xi = xr[i - lo:i - lo + 1]
                xi = xi.float().cpu().numpy() if layer.dtype != "int8" else xi.cpu().numpy().astype(np.int64)
                ref = np.asarray(reference_conv(xi, wf, *sp.conv_args()), dtype=np.float64)
                got = y_full[i:i + 1].float().cpu().numpy().astype(np.float64)
                if layer.dtype == "int8":
                    err = 0.0 if np.array_equal(got, ref) else float("inf")
                else:
                    err = float(np.abs(got - ref).max() / max(np.abs(ref).max(), 1e-30))
                max_err = max(max_err, err)
                checked += 1
                if not err <= PARITY_TOL:
                    bad.append(f"{layer.name}[{i}]")
        del y_full
    if rank != 0:
        return None
    return {"ok": not bad, "checked_images": checked, "layers": len(work), "max_norm_err": max_err,
            "tol": PARITY_TOL if layers_full[0].dtype != "int8" else 0.0,
            "bar": "bit-exact" if layers_full[0].dtype == "int8" else "max|y-ref|/max|ref| (bf16 out vs fp32 oracle)",
            "failures": bad[:10],
            "how": "outputs of the timed steps all-gathered over ranks (sharding.gather_shards); first and last "
                   "image of every rank's shard vs oracle.conv2d_nhwc_taps / exact int path"}


# ------------------------------------------------------------------ GPU arm

def main(argv=None):
    argv = sys.argv[1:] if argv is None else argv
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="cfg4", choices=["cfg1", "cfg2", "cfg3", "cfg4", "cfg5"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--ref-budget-s", type=float, default=1000.0,
                    help="--impl reference: time budget of the timed full-size steps (fewer steps if exceeded)")
    ap.add_argument("--cpu-sample", type=int, default=64, help="batch per layer of the cpu_baseline sample")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--layers-json", default=None, help="write per-layer timings here (rank 0)")
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--no-overlap", action="store_true",
                    help="launch the layers serialised (each waits for the previous grid) instead of with "
                         "IMCONV_FLAG_INDEPENDENT; by default both are timed and the overlapped step is the "
                         "headline")
    ap.add_argument("--no-traffic", action="store_true",
                    help="skip the in-run ncu DRAM-traffic measurement (report the committed figure if any)")
    ap.add_argument("--traffic-child", action="store_true", help=argparse.SUPPRESS)
    ap.add_argument("--sweep-jobs", type=float, default=0.0,
                    help="convolutions in flight in the overlapped step (paper_2110_03901_b200.sweep; "
                         "0 = the library default for the step's work)")
    ap.add_argument("--launch-order", default="mix", choices=["sweep", "lpt", "reverse", "mix"],
                    help="order of the layers' launches inside the timed step (diagnostic)")
    ap.add_argument("--planner-debug", type=lambda v: int(v, 0), default=0,
                    help="diagnostic A/B only: host planner switches (imconv_debug_set_flags bits 16+); "
                         "reported in the line's `run` object")
    ap.add_argument("--emulate-world", type=int, default=0,
                    help="diagnostic (1 process): run rank 0's shard of a W-rank job and report W x its "
                         "throughput, i.e. what the W-GPU run measures when every rank matches rank 0")
    args = ap.parse_args(argv)

    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(args.gpus, argv)

    from paper_2110_03901_b200.workloads import baseline_configs
    layers_full = baseline_configs()[args.config]
    world, rank, local = dist_setup()
    if world > 1 and args.gpus not in (1, world):
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; running {world} ranks", file=sys.stderr)
    shard_world = world
    if args.emulate_world > 1:
        if world != 1:
            raise SystemExit("--emulate-world is a single-process diagnostic")
        shard_world = args.emulate_world
    config = workload_config(args.config, layers_full, shard_world)
    if args.impl == "reference":
        return run_reference_arm(args, layers_full, world, rank, config)

    import torch
    import torch.distributed as dist
    import paper_2110_03901_b200 as P
    from paper_2110_03901_b200 import _lib
    from paper_2110_03901_b200._kernels import conv_device
    # The weights are written once at setup, never inside the step: every conv may start its
    # filter loads before its programmatic-launch wait (IMCONV_FLAG_STATIC_FILTER).  The cfg4
    # workload is a SWEEP of independent convolutions (BASELINE.json: every layer gets its own
    # N(0,1) input), each over its own buffers, so by default every launch also carries
    # IMCONV_FLAG_INDEPENDENT: it never waits for the preceding grid, and layer i+1's CTAs start
    # on the SMs layer i's last wave leaves idle.  The serialised step (every layer waiting for
    # the previous one, as a chained network would) is timed in the same run and reported beside.
    SERIAL_FLAGS = _lib.FLAG_STATIC_FILTER
    STATIC = SERIAL_FLAGS | (0 if args.no_overlap else _lib.FLAG_INDEPENDENT)

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    peaks, peak_kind = load_peaks()
    if args.planner_debug:
        if args.planner_debug & 0xffff:
            raise SystemExit("--planner-debug takes host planner switches only (bits 16+)")
        _lib.lib.imconv_debug_set_flags(args.planner_debug)

    # ---- per-rank shard of every layer (contiguous images; no collective) ----
    work = []
    for li, layer in enumerate(layers_full):
        lo, hi = shard_batch(layer.spec.n, shard_world, rank)
        sp = layer.spec.with_batch(hi - lo)
        x, w = make_operands(layer, sp, li, lo, dev)
        odt = torch.int32 if layer.dtype == "int8" else torch.bfloat16
        y = torch.empty((sp.n, sp.h_o, sp.w_o, sp.c_o), dtype=odt, device=dev)
        work.append((layer, sp, x, w, y))
    torch.cuda.synchronize()

    total_flops_rank = sum(sp.flops for _, sp, *_ in work)
    bytes_alg_rank = sum(bytes_alg(sp, layer.dtype, y.element_size()) for layer, sp, x, w, y in work)

    # Consecutive timed passes must not find their inputs in L2: when one pass's working set
    # is below twice the L2 size (the small parity configs), the captured step runs the pass
    # over `copies` independent sets of buffers (same values), so every pass reads cold data.
    copies = rotation_copies(layers_full, shard_world)
    work_sets = [work] + [[(layer, sp, x.clone(), w.clone(), torch.empty_like(y)) for layer, sp, x, w, y in work]
                          for _ in range(copies - 1)]

    from paper_2110_03901_b200 import sweep as SW
    sweep_jobs = args.sweep_jobs or SW.default_jobs(float(sum(sp.flops for _, sp, *_ in work)), len(work))
    # (a replay that rotates over several buffer sets runs them all as one sweep)
    sweep_jobs_all = args.sweep_jobs or SW.default_jobs(float(sum(sp.flops for _, sp, *_ in work)) * copies,
                                                        len(work) * copies)

    def one_pass(ws, flags=None):
        order = ws[::-1] if args.launch_order == "reverse" else ws
        if flags is None and STATIC != SERIAL_FLAGS:
            # the overlapped step: the layers as one sweep of independent convolutions, about
            # `sweep_jobs` of them in flight at a time (paper_2110_03901_b200.sweep)
            SW.conv_sweep([(x, w, sp.conv_args(), y) for layer, sp, x, w, y in order], jobs=sweep_jobs,
                          check=True, order=args.launch_order if args.launch_order in ("lpt", "mix") else "given")
            return
        for layer, sp, x, w, y in order:
            conv_device(x, w, *sp.conv_args(), y=y, flags=STATIC if flags is None else flags)

    def all_passes(flags=None):
        if flags is None and STATIC != SERIAL_FLAGS and len(work_sets) > 1:
            # the rotation copies hold independent buffers too: one sweep over all of them
            convs = []
            for ws in work_sets:
                order = ws[::-1] if args.launch_order == "reverse" else ws
                convs += [(x, w, sp.conv_args(), y) for layer, sp, x, w, y in order]
            SW.conv_sweep(convs, jobs=sweep_jobs_all, check=True,
                          order=args.launch_order if args.launch_order in ("lpt", "mix") else "given")
            return
        for ws in work_sets:
            one_pass(ws, flags)

    # launches per pass (our kernels only)
    _lib.lib.imconv_reset_launch_count()
    one_pass(work)
    torch.cuda.synchronize()
    launches_per_pass = int(_lib.lib.imconv_launch_count())
    if args.traffic_child:  # ncu child of measure_traffic: the profiled pass, then exit
        one_pass(work)
        torch.cuda.synchronize()
        return 0

    graph = None
    if not args.no_graph:
        stream = torch.cuda.Stream()
        stream.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(stream):
            all_passes()  # warm caches outside capture
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=stream):
            all_passes()  # one replay = `copies` passes, one per buffer set
        torch.cuda.synchronize()

    def run_replay():
        if graph is not None:
            graph.replay()
        else:
            all_passes()

    replays = -(-args.steps // copies)  # timed passes = replays * copies >= steps
    passes = replays * copies
    for _ in range(max(-(-max(args.warmup, 3) // copies), 1)):
        run_replay()
    torch.cuda.synchronize()

    # ---- timed region: back-to-back passes ----
    sampler = ClockSampler(local)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    sampler.start()
    time.sleep(0.3)  # let the sampler attach
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    cur = torch.cuda.current_stream()
    ev0.record(cur)
    for _ in range(replays):
        run_replay()
    ev1.record(cur)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = sampler.stop()
    region_ms_rank = ev0.elapsed_time(ev1)
    ms_rank = region_ms_rank / passes
    ms = ms_rank
    if world > 1:
        t = torch.tensor([ms_rank], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    # ---- the same step with the layers serialised (no IMCONV_FLAG_INDEPENDENT), same replays ----
    serial_ms = None
    if STATIC != SERIAL_FLAGS and graph is not None:
        g_ser = torch.cuda.CUDAGraph()
        with torch.cuda.stream(stream):
            all_passes(SERIAL_FLAGS)
        torch.cuda.synchronize()
        with torch.cuda.graph(g_ser, stream=stream):
            all_passes(SERIAL_FLAGS)
        g_ser.replay()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(cur)
        for _ in range(replays):
            g_ser.replay()
        e1.record(cur)
        torch.cuda.synchronize()
        serial_ms = e0.elapsed_time(e1) / passes
        if world > 1:
            t = torch.tensor([serial_ms], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            serial_ms = float(t.item())
        del g_ser
    total_flops = sum(l.spec.flops for l in layers_full)  # all ranks together
    if shard_world != world:  # emulated: every rank assumed as fast as rank 0
        total_flops = total_flops_rank * shard_world
    value = total_flops / (ms / 1e3) / 1e12

    # ---- parity of what was just timed ----
    parity = None
    if not args.no_parity and shard_world == world:
        from oracle import oracle as O
        ref_conv = O.conv2d_nhwc_taps if layers_full[0].dtype != "int8" else O.conv2d_nhwc_exact_f64
        parity = verify_outputs(work, layers_full, world, rank, dev,
                                lambda n, r: shard_batch(n, world, r),
                                lambda layer, sp, li, lo: make_operands(layer, sp, li, lo, dev)[0], ref_conv)

    # ---- per-layer kernel times (separate pass): each layer's `reps` launches
    # are replayed from their own CUDA graph, so host launch latency cannot
    # starve short kernels ----
    per_layer = []
    reps = 5
    side = torch.cuda.Stream()
    for layer, sp, x, w, y in work:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=side):
            for _ in range(reps):  # (each layer alone: repeated launches share y, so never overlapped)
                conv_device(x, w, *sp.conv_args(), y=y, flags=_lib.FLAG_STATIC_FILTER)
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
    burst = region_ms_rank < BURST_REGION_MS
    bf16_peak = peaks.get("bf16_tflops" if burst else "bf16_tflops_sustained",
                          PEAKS_FALLBACK["bf16_tflops" if burst else "bf16_tflops_sustained"])
    dtype_peak = bf16_peak
    if int8_peak is not None and all(l.dtype == "int8" for l, *_ in work):
        dtype_peak = int8_peak
    hbm = peaks.get("hbm_gbs", PEAKS_FALLBACK["hbm_gbs"])
    # achieved: this rank's FLOP over its device time per pass in the TIMED region (the step
    # is nothing but the conv kernels); the separate per-layer pass only apportions it
    achieved = total_flops_rank / (ms_rank / 1e3) / 1e12
    roof_ms = 0.0
    layer_rows = []
    # per roofline bound: the layers whose tensor time exceeds their HBM time, and the rest --
    # each group's bound time over its measured time (the kernels' quality, apart from the mix)
    groups = {"tensor": [0, 0.0, 0.0], "hbm": [0, 0.0, 0.0]}
    for layer, sp, t_ms in per_layer:
        eo = 4 if layer.dtype == "int8" else 2
        b = bytes_alg(sp, layer.dtype, eo)
        pk = int8_peak if (layer.dtype == "int8" and int8_peak) else bf16_peak
        t_tc, t_mem = sp.flops / (pk * 1e12) * 1e3, b / (hbm * 1e9) * 1e3
        t_roof = max(t_tc, t_mem)
        gr = groups["tensor" if t_tc >= t_mem else "hbm"]
        gr[0] += 1
        gr[1] += t_ms
        gr[2] += t_roof
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

    # ---- CPU baseline (rank 0, N=1 only): the reference's kernels on a bounded sample ----
    cpu = None
    if rank == 0 and world == 1 and shard_world == 1 and not args.no_cpu:
        use_all_host_threads()
        conv, kind, desc = cpu_impl()
        n_s = min(args.cpu_sample, layers_full[0].spec.n)
        cpu_time_layers(layers_full[:1], 1, conv)  # warm-up
        secs, f = cpu_time_layers(layers_full, n_s, conv)
        cores = 1 if (layers_full[0].dtype == "int8" and kind == "reference") else cpu_threads()
        cpu = {"value": f / secs[0] / 1e12, "unit": "TFLOP/s", "cores": cores, "kind": kind,
               "sample": f"{args.config}: all {len(layers_full)} layers at batch {n_s} of {layers_full[0].spec.n} "
                         f"({desc}; {secs[0]:.1f} s)"}

    traffic, traffic_note, traffic_rows = None, "not measured (--no-traffic)", None
    if rank == 0 and world == 1 and not args.no_traffic:
        traffic, traffic_note, traffic_rows = measure_traffic(args, launches_per_pass)
    if traffic is None:
        committed, note = committed_traffic(args.config, shard_world)
        if committed is not None:
            traffic, traffic_note = committed, note
        else:
            traffic_note += f"; {note}"
    # the stem executes C = 8 (3 image channels zero-padded, as BASELINE.json defines it);
    # the same run with only the 3 useful channels counted
    useful_value = None
    stem = [sp for layer, sp, *_ in work if layer.name == "stem" and sp.c_i == 8]
    if stem:
        useful_value = value * (total_flops_rank - stem[0].flops * 5 / 8) / total_flops_rank
    if rank == 0:
        peak_name = "int8 TOPS (cuBLAS torch._int_mm, this run)" if dtype_peak == int8_peak else (
            f"{peak_kind} bf16 {'burst' if burst else 'sustained'} (MEASURED_PEAKS.json; timed region "
            f"{region_ms_rank:.0f} ms {'<' if burst else '>='} {BURST_REGION_MS:.0f} ms)")
        line = {
            "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": passes,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "bf16" if layers_full[0].dtype != "int8" else "int8", "data": "synthetic",
            "config": config,
            **({"emulated_world": shard_world} if shard_world != world else {}),
            "run": {"cuda_graph": graph is not None, "passes_per_replay": copies, "replays": replays,
                    "timed_region_ms": region_ms_rank,
                    "layer_overlap": STATIC != SERIAL_FLAGS,
                    **({"planner_debug": hex(args.planner_debug)} if args.planner_debug else {}),
                    **({"sweep_jobs": round(sweep_jobs_all if copies > 1 else sweep_jobs, 3),
                        "sweep_ctas_per_launch": SW.sweep_grid(sweep_jobs_all if copies > 1 else sweep_jobs, dev),
                        "sweep_launch_order": args.launch_order}
                       if STATIC != SERIAL_FLAGS else {}),
                    **({"value_layers_serialized": total_flops / (serial_ms / 1e3) / 1e12,
                        "ms_per_step_layers_serialized": serial_ms} if serial_ms else {}),
                    **({"value_stem_c3": useful_value} if useful_value is not None else {})},
            "pct_of_peak": {"measured_burst": value / shard_world / (dtype_peak if dtype_peak == int8_peak
                                                                     else peaks.get("bf16_tflops", 1648.9)),
                            "measured_sustained": value / shard_world / (
                                dtype_peak if dtype_peak == int8_peak else peaks.get("bf16_tflops_sustained", 1400.0)),
                            "datasheet": value / shard_world / (4500.0 if dtype_peak == int8_peak else 2250.0),
                            "unit_peak": "int8 TOPS" if dtype_peak == int8_peak else "bf16 TFLOP/s"},
            "roofline": {"bound": "tensor", "achieved": achieved, "peak": dtype_peak, "unit": "TFLOP/s",
                         "frac": achieved / dtype_peak,
                         "traffic": traffic,
                         "traffic_unit": "DRAM bytes per step per GPU (ncu dram__bytes_read+write)",
                         "traffic_source": traffic_note,
                         **({"traffic_over_alg": traffic / bytes_alg_rank} if traffic else {}),
                         **({"ncu_pass_us": sum(d.get("gpu__time_duration.sum", 0.0) for d in traffic_rows) / 1e3,
                             "ncu_top_launch": max(({"kernel": d["kernel"][:60], "us": d.get("gpu__time_duration.sum", 0.0) / 1e3,
                                                     "dram_bytes": d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)}
                                                    for d in traffic_rows), key=lambda e: e["us"])}
                            if traffic_rows else {}),
                         "bytes_alg": bytes_alg_rank,
                         "peak_kind": peak_name,
                         "kernel": "conv kernels (generic / row-band / halo), all layers of the step",
                         "achieved_source": "timed region: rank FLOP / device ms per pass",
                         "roofline_limited_frac": roof_ms / ms_rank,
                         "by_bound": {k: {"layers": v[0], "ms_per_step": round(v[1], 4),
                                          "frac": round(v[2] / v[1], 3) if v[1] else None,
                                          "of": ("tensor peak" if k == "tensor" else "HBM copy bandwidth")}
                                      for k, v in groups.items()},
                         "by_bound_source": "separate per-layer pass (each layer alone, 5 launches per CUDA graph)"},
            "parity": parity,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches_per_pass * passes,
            "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
        if args.layers_json:
            with open(args.layers_json, "w") as fh:
                json.dump({"config": args.config, "world": shard_world, "kernel_ms": kern_ms,
                           "roofline_ms": roof_ms, "layers": layer_rows}, fh, indent=1)
    rc = 0 if (parity is None or rank != 0 or parity["ok"]) else 1
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return rc


if __name__ == "__main__":
    sys.exit(main())
