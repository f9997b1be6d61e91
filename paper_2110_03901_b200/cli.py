"""Command line front end: ``python -m paper_2110_03901_b200 {verify,simulate,overhead}``.

Mirrors the reference CLI's commands for the convolution path (cli.py:117-153,
:209-248), driving the B200 kernels instead of the
systolic-array model:

* ``verify [--count N] [--seed S]`` -- the reference's randomized validation:
  the same ``random_spec`` case sequence and ``default_operands``, every
  functional method's OFMap (channel-first implicit kernel, channel-last and
  channel-first explicit im2col + GEMM) checked against ``direct_conv`` and
  against an independent host int64 tap loop (the checker, not a compute
  path).  Prints ``k/N match``; mismatches exit 1 with
  ``<prog>: error: VerifyMismatch: case<i>/<method>,...``.
* ``simulate --workload FILE [--method M] [--verify] [--out CSV]`` -- every
  layer of a workload JSON (the reference's schema: ``layers`` with
  n/c_i/h_i/w_i/c_o/h_f/w_f and stride|stride_h/_w, pad, dilation; optional
  ``methods``, ``seed``, ``elem_bytes``, ``model``) runs on the GPU; rows give
  the measured device time and TFLOP/s and the predicted DRAM bytes
  (``traffic.predict``) in the reference's ``# sasim-csv v1`` CSV format.
* ``overhead --workload FILE`` -- the explicit-lowering memory footprint per
  layer (``lowering.lowered_memory_footprint``) with a TOTAL row.

Errors follow the reference convention: ``<prog>: error: <Type>: <msg>``,
exit status 2.
"""

from __future__ import annotations

import argparse
import csv
import json
import os
import sys
from contextlib import nullcontext

import numpy as np

from .core import ConvSpec, ShapeError, direct_conv
from .functional import ALL_METHODS, Method, functional_ofmap
from .lowering import lowered_memory_footprint
from .workloads import default_operands, random_spec

PROG = "paper_2110_03901_b200"
CSV_SCHEMA = "# sasim-csv v1"
SPEC_COLUMNS = ["n", "c_i", "h_i", "w_i", "c_o", "h_f", "w_f", "stride_h", "stride_w", "pad_h", "pad_w",
                "dilation_h", "dilation_w"]
SIM_COLUMNS = ["name", "method"] + SPEC_COLUMNS + ["kernel", "gpu_ms", "tflops", "dram_read_bytes",
                                                   "dram_write_bytes", "verified", "error"]
OVERHEAD_COLUMNS = ["name"] + SPEC_COLUMNS[:12] + ["original_bytes", "lowered_bytes", "ratio"]


class WorkloadError(ValueError):
    """A workload file is malformed."""


class VerifyMismatch(RuntimeError):
    """A kernel disagreed with the oracle."""


def _axis_pair(d: dict, key: str, default: int):
    if key in d and (f"{key}_h" in d or f"{key}_w" in d):
        raise WorkloadError(f"give either {key} or {key}_h/{key}_w, not both")
    if key in d:
        return int(d[key]), int(d[key])
    return int(d.get(f"{key}_h", default)), int(d.get(f"{key}_w", default))


def layer_spec(d: dict) -> ConvSpec:
    sh, sw = _axis_pair(d, "stride", 1)
    ph, pw = _axis_pair(d, "pad", 0)
    dh, dw = _axis_pair(d, "dilation", 1)
    try:
        return ConvSpec(n=int(d["n"]), c_i=int(d["c_i"]), h_i=int(d["h_i"]), w_i=int(d["w_i"]), c_o=int(d["c_o"]),
                        h_f=int(d["h_f"]), w_f=int(d["w_f"]), stride_h=sh, stride_w=sw, pad_h=ph, pad_w=pw,
                        dilation_h=dh, dilation_w=dw)
    except KeyError as exc:
        raise WorkloadError(f"layer is missing required key {exc}") from None


def load_workload(path: str) -> dict:
    if not os.path.exists(path):
        raise WorkloadError(f"workload file not found: {path}")
    try:
        with open(path) as fh:
            doc = json.load(fh)
    except json.JSONDecodeError as exc:
        raise WorkloadError(f"{path}:{exc.lineno}: {exc.msg}") from None
    layers, names = [], set()
    for idx, entry in enumerate(doc.get("layers", [])):
        name = entry.get("name", f"layer{idx}")
        if name in names:
            raise WorkloadError(f"{path}: duplicate layer name {name!r}")
        names.add(name)
        try:
            layers.append((name, layer_spec(entry)))
        except (WorkloadError, ShapeError) as exc:
            raise WorkloadError(f"{path}: layer {name!r}: {exc}") from None
    methods = [Method.parse(m) for m in doc.get("methods", ["channel_first"])]
    return {"model": doc.get("model", os.path.basename(path)), "layers": layers, "methods": methods,
            "elem_bytes": int(doc.get("elem_bytes", 2)), "seed": int(doc.get("seed", 0))}


def _fmt(v):
    if isinstance(v, float):
        return f"{v:.10g}"
    return "" if v is None else v


def _write_csv(out, columns, rows):
    ctx = nullcontext(sys.stdout) if out in (None, "-") else open(out, "w", newline="")
    with ctx as fh:
        fh.write(CSV_SCHEMA + "\n")
        w = csv.writer(fh, lineterminator="\n")
        w.writerow(columns)
        for row in rows:
            w.writerow([_fmt(row.get(c)) for c in columns])


def _spec_cells(name, sp: ConvSpec) -> dict:
    return {"name": name, "n": sp.n, "c_i": sp.c_i, "h_i": sp.h_i, "w_i": sp.w_i, "c_o": sp.c_o, "h_f": sp.h_f,
            "w_f": sp.w_f, "stride_h": sp.stride_h, "stride_w": sp.stride_w, "pad_h": sp.pad_h, "pad_w": sp.pad_w,
            "dilation_h": sp.dilation_h, "dilation_w": sp.dilation_w}


def _host_check(x: np.ndarray, w: np.ndarray, sp: ConvSpec) -> np.ndarray:
    """Independent int64 tap-loop convolution on the host -- the verify
    command's checker (never a result path)."""
    xp = np.zeros((sp.n, sp.h_i + 2 * sp.pad_h, sp.w_i + 2 * sp.pad_w, sp.c_i), dtype=np.int64)
    xp[:, sp.pad_h:sp.pad_h + sp.h_i, sp.pad_w:sp.pad_w + sp.w_i, :] = x
    y = np.zeros((sp.n, sp.h_o, sp.w_o, sp.c_o), dtype=np.int64)
    for r in range(sp.h_f):
        for s in range(sp.w_f):
            h0, w0 = r * sp.dilation_h, s * sp.dilation_w
            win = xp[:, h0:h0 + (sp.h_o - 1) * sp.stride_h + 1:sp.stride_h,
                     w0:w0 + (sp.w_o - 1) * sp.stride_w + 1:sp.stride_w, :]
            y += np.tensordot(win, w[r, s].astype(np.int64), axes=([3], [0]))
    return y


def _mismatches(tag, sp, x, w, methods):
    want = _host_check(np.asarray(x.data).reshape(sp.n, sp.h_i, sp.w_i, sp.c_i),
                       np.asarray(w.data).reshape(sp.h_f, sp.w_f, sp.c_i, sp.c_o), sp)
    bad = []
    ref = np.asarray(direct_conv(x, w, sp).data).reshape(want.shape)
    if not np.array_equal(ref, want):
        bad.append(f"{tag}/direct_conv")
    for m in methods:
        got = np.asarray(functional_ofmap(sp, m, x, w).data).reshape(want.shape)
        if not np.array_equal(got, want):
            bad.append(f"{tag}/{m.value}")
    return bad


def cmd_verify(args) -> int:
    rng = np.random.default_rng(args.seed if args.seed is not None else 0)
    failures = []
    for i in range(args.count):
        sp = random_spec(rng)
        x, f = default_operands(sp, int(rng.integers(0, 2**31)))
        failures += _mismatches(f"case{i}", sp, x, f, ALL_METHODS)
    ok = args.count - len({fl.split("/")[0] for fl in failures})
    print(f"{ok}/{args.count} match")
    if failures:
        print(f"{PROG}: error: VerifyMismatch: " + ",".join(failures), file=sys.stderr)
        return 1
    return 0


def _time_layer(sp: ConvSpec, method: Method, x, w, reps: int = 5) -> float:
    import torch
    from ._kernels import conv_device
    from .functional import explicit_im2col
    from .lowering import ColumnOrdering
    if method is Method.CHANNEL_FIRST_IMPLICIT:
        xd = torch.as_tensor(np.asarray(x.data)).reshape(sp.n, sp.h_i, sp.w_i, sp.c_i).float().cuda().bfloat16()
        wd = torch.as_tensor(np.asarray(w.data)).reshape(sp.h_f, sp.w_f, sp.c_i, sp.c_o).float().cuda().bfloat16()
        run = lambda: conv_device(xd, wd, *sp.conv_args())  # noqa: E731
    else:
        order = ColumnOrdering.CHANNEL_LAST if method is Method.CHANNEL_LAST_IMPLICIT else \
            ColumnOrdering.CHANNEL_FIRST
        run = lambda: explicit_im2col(sp, x, w, order)  # noqa: E731
    run()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        run()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def cmd_simulate(args) -> int:
    from .traffic import predict
    wl = load_workload(args.workload)
    methods = [Method.parse(args.method)] if args.method else wl["methods"]
    seed = args.seed if args.seed is not None else wl["seed"]
    rows, mismatched = [], []
    for name, sp in wl["layers"]:
        for m in methods:
            row = _spec_cells(name, sp) | {"method": m.value}
            try:
                x, f = default_operands(sp, seed)
                if args.verify:
                    bad = _mismatches(name, sp, x, f, [m])
                    mismatched += bad
                    row["verified"] = 0 if bad else 1
                ms = _time_layer(sp, m, x, f)
                row["gpu_ms"] = ms
                row["tflops"] = sp.flops / (ms / 1e3) / 1e12
                try:
                    t = predict(sp)
                    row.update(kernel=t.kernel, dram_read_bytes=t.dram_read_bytes,
                               dram_write_bytes=t.dram_write_bytes + t.resident_dirty_bytes)
                except Exception as exc:  # (CTA-pair shapes are not modelled)
                    row["kernel"] = f"unmodelled: {exc}"
            except Exception as exc:
                row["error"] = f"{type(exc).__name__}: {exc}"
            rows.append(row)
    _write_csv(args.out, SIM_COLUMNS, rows)
    if args.verify:
        total = len(rows)
        print(f"{total - len(mismatched)}/{total} match", file=sys.stderr if args.out in (None, "-") else sys.stdout)
        if mismatched:
            print(f"{PROG}: error: VerifyMismatch: " + ",".join(mismatched), file=sys.stderr)
            return 1
    return 0


def cmd_overhead(args) -> int:
    wl = load_workload(args.workload)
    rows, tot_orig, tot_low = [], 0, 0
    for name, sp in wl["layers"]:
        fp = lowered_memory_footprint(sp, wl["elem_bytes"])
        tot_orig += fp["original_bytes"]
        tot_low += fp["lowered_bytes"]
        rows.append(_spec_cells(name, sp) | fp)
    if wl["layers"]:
        rows.append({"name": "TOTAL", "original_bytes": tot_orig, "lowered_bytes": tot_low,
                     "ratio": tot_low / tot_orig})
    _write_csv(args.out, OVERHEAD_COLUMNS, rows)
    return 0


def build_parser() -> argparse.ArgumentParser:
    p = argparse.ArgumentParser(prog=PROG, description="B200 implicit-im2col convolution: verify / simulate / overhead")
    sub = p.add_subparsers(dest="command", required=True)

    def common(sp, workload=True):
        if workload:
            sp.add_argument("--workload", required=True, help="workload JSON (the reference's schema)")
        sp.add_argument("--out", default="-", help="output CSV path (- = stdout)")
        sp.add_argument("--seed", type=int, default=None)

    sp = sub.add_parser("simulate", help="run every workload layer on the GPU")
    common(sp)
    sp.add_argument("--method", help="override workload methods")
    sp.add_argument("--verify", action="store_true", help="check OFMaps against the host int64 checker")
    sp.set_defaults(func=cmd_simulate)
    sp = sub.add_parser("overhead", help="explicit-lowering memory overhead")
    common(sp)
    sp.set_defaults(func=cmd_overhead)
    sp = sub.add_parser("verify", help="randomized validation of every method")
    common(sp, workload=False)
    sp.add_argument("--count", type=int, default=30)
    sp.set_defaults(func=cmd_verify)
    return p


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    try:
        return args.func(args)
    except Exception as exc:
        msg = str(exc).replace("\n", " ")
        print(f"{PROG}: error: {type(exc).__name__}: {msg}", file=sys.stderr)
        return 2


if __name__ == "__main__":
    sys.exit(main())
