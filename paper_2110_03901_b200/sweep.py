"""Independent convolutions run concurrently -- the B200 counterpart of the reference's
``sweep(specs, ..., jobs=N)`` (/root/reference/pkg/src/sasim/simulator.py:550-576), which
evaluates independent specs on N worker threads.

Here the N "jobs" are convolutions in flight on the GPU at the same time, on one stream:

* every launch carries ``IMCONV_FLAG_INDEPENDENT`` (include/imconv.h): it does not wait for
  the preceding grid, so its CTAs start on whatever SMs are free;
* the first launch of a sweep carries ``IMCONV_FLAG_BARRIER`` instead: it waits for all work
  queued before the sweep and only then lets the rest of the sweep start;
* each launch runs on ``sms // jobs`` persistent CTAs, so about ``jobs`` convolutions share the
  GPU: a memory-bound layer's stream overlaps a compute-bound layer's MMAs, and each layer's
  fixed costs overlap other layers' work.  The planner's throughput mode applies (no split-K,
  CTA pairs below one wave: the SMs a launch leaves idle run the others).

Measured on the cfg4 sweep (53 ResNet-50 layers, profiles/r2/README.md): 1 / 2 / 4 / 8-GPU
shards (256 / 128 / 64 / 32 images) 876 -> 916, 1662 -> 1813, 2956 -> 3521, 4724 -> 6553
TFLOP/s against one launch at a time on every SM.

The buffers of a sweep must be disjoint: no convolution may write memory another one (or any
kernel still in flight) reads or writes.  ``conv_sweep`` checks the outputs against every
operand of the sweep and raises ``ValueError`` on overlap.
"""

from __future__ import annotations

from typing import Iterable, Sequence

import torch

from . import _lib

# per-GPU work (FLOP per sweep) above which fewer, larger launches run side by side
_BIG_SWEEP_FLOP = 1.5e12


def default_jobs(flop: float, count: int | None = None) -> float:
    """Convolutions in flight for a sweep of ``count`` convolutions and ``flop`` total work.

    A heuristic fitted to measurements on B200 (profiles/r2/README.md, "sweep concurrency"):
    * convolutions of >= 100 GFLOP each fill the GPU alone: 1 (cfg3, 2 x 309 GFLOP);
    * a handful (<= 8) of them: 2 (cfg5 int8 / cfg2);
    * many tiny ones (< 4 GFLOP each): 8 (cfg1's 41 copies of a 1.85 GFLOP layer: 344 -> 569
      TFLOP/s against one at a time);
    * otherwise ~8/3 for >= 1.5 TFLOP in total (56 CTAs each on 148 SMs: the cfg4 sweep at 256
      images) and 4 below (37 CTAs each: its 128 / 64 / 32-image shards).
    """
    count = count or 64
    avg = flop / count
    if avg >= 100e9:
        return 1.0
    if count <= 8:
        return float(min(2, count))
    if avg < 4e9:
        return 8.0
    return 8.0 / 3.0 if flop >= _BIG_SWEEP_FLOP else 4.0


def sweep_grid(jobs: float, device: torch.device | None = None) -> int:
    """Persistent CTAs per launch when ``jobs`` launches share the device's SMs."""
    sms = torch.cuda.get_device_properties(device or torch.cuda.current_device()).multi_processor_count
    # even: CTA-pair launches run whole clusters (an odd 55 measured 895-903 against 917-919 for 56)
    return max(2, 2 * round(sms / jobs / 2))


def _span(t: torch.Tensor):
    start = t.data_ptr()
    return start, start + t.numel() * t.element_size()


def _check_disjoint(convs) -> None:
    for i, (x, w, _args, y) in enumerate(convs):
        for what, t in (("x", x), ("w", w), ("y", y)):
            if not t.is_contiguous():
                raise ValueError(f"sweep convolution {i}: {what} must be contiguous (a copy would serialise the sweep)")
    spans = []
    for i, (x, w, _args, y) in enumerate(convs):
        spans.append((i, "x", _span(x)))
        spans.append((i, "w", _span(w)))
    for i, (x, w, _args, y) in enumerate(convs):
        ylo, yhi = _span(y)
        for j, what, (lo, hi) in spans:
            if lo < yhi and ylo < hi:
                raise ValueError(f"sweep output {i} overlaps {what} of convolution {j}")
        for j, (_x2, _w2, _a2, y2) in enumerate(convs):
            if j != i:
                lo, hi = _span(y2)
                if lo < yhi and ylo < hi:
                    raise ValueError(f"sweep outputs {i} and {j} overlap")


def _est_us2(x, w, y) -> tuple:
    """(tensor time, memory time) of one convolution in us at the measured B200 peaks
    (1650 TFLOP/s bf16 / 3000 TOPS int8, 6500 GB/s)."""
    flop = 2.0 * y.numel() * w.shape[0] * w.shape[1] * w.shape[2]
    peak = 3000e12 if x.dtype == torch.int8 else 1650e12
    nbytes = x.numel() * x.element_size() + w.numel() * w.element_size() + y.numel() * y.element_size()
    return flop / peak * 1e6, nbytes / 6500e9 * 1e6


def _est_us(x, w, y) -> float:
    """Roofline time estimate of one convolution: max(tensor time, time to move its operands
    and output)."""
    return max(_est_us2(x, w, y))


def mixed_order(convs: Sequence) -> list:
    """Launch order that keeps the mix of memory and tensor work in flight balanced: with
    ~jobs launches in flight, a memory-bound layer then runs beside compute-bound ones instead
    of beside other memory-bound layers.  (A memory-bound layer on a third of the SMs is limited
    by the per-SM store rate, ~52 GB/s (tools/store_bench.cu), not by HBM, so it costs fewer
    SM-microseconds there than alone on every SM -- provided the others in flight leave it the
    HBM bandwidth.)

    The convolutions whose memory share m / (m + t) exceeds the sweep's are merged with the
    others so that the running surplus of memory time stays near zero; each side goes from its
    most extreme member to its most balanced one, except that long poles (estimate >= twice the
    median) lead their side, so the sweep does not end on one long launch."""
    est = [_est_us2(x, w, y) for x, w, _a, y in convs]
    goal = sum(m for _t, m in est) / max(sum(t + m for t, m in est), 1e-30)
    tot = sorted(max(e) for e in est)
    long_pole = 2.0 * tot[len(tot) // 2]
    surplus = [m - goal * (t + m) for t, m in est]   # > 0: more memory time than the sweep's mix
    share = [m / max(t + m, 1e-30) for t, m in est]
    heavy = sorted((i for i in range(len(est)) if surplus[i] > 0),
                   key=lambda i: (max(est[i]) < long_pole, -share[i], i))
    light = sorted((i for i in range(len(est)) if surplus[i] <= 0),
                   key=lambda i: (max(est[i]) < long_pole, share[i], i))
    out, a, b, run = [], 0, 0, 0.0
    while a < len(heavy) or b < len(light):
        if b >= len(light) or (a < len(heavy) and run <= 0.0):
            run += surplus[heavy[a]]
            out.append(heavy[a])
            a += 1
        else:
            run += surplus[light[b]]
            out.append(light[b])
            b += 1
    return out


def conv_sweep(convs: Sequence, jobs: float | None = None, flops: float | None = None,
               check: bool = True, flags: int = 0, order: str = "given") -> list:
    """Run independent convolutions concurrently on the current stream.

    ``convs``: sequence of ``(x, w, (sh, sw, ph, pw, dh, dw), y)`` with CUDA tensors in the
    compute dtype (``y`` preallocated, contiguous, the output dtype).  ``jobs``: convolutions
    in flight (default: :func:`default_jobs` of the sweep's FLOP, given or computed).  Returns
    the outputs.  Capturable into a CUDA graph like any launch of the library.
    """
    from ._kernels import conv_device
    convs = list(convs)
    if not convs:
        return []
    if check:
        _check_disjoint(convs)
    if jobs is None:
        jobs = default_jobs(sweep_flops(convs) if flops is None else flops, len(convs))
    grid = sweep_grid(jobs, convs[0][0].device)
    base = flags | _lib.FLAG_STATIC_FILTER | _lib.FLAG_INDEPENDENT
    # launch order: "given" = as listed (default), "lpt" = longest estimated first, "mix" =
    # memory and tensor work balanced (mixed_order); outputs are returned as listed.  On the cfg4
    # sweep at 256 images: given (ResNet order, which already alternates memory- and compute-bound
    # layers) 925-928 TFLOP/s, mix 929-936, lpt 899-902 against given 909-920 on another box,
    # reverse 851; 32-image shard x 8: given 6448-6488, mix 6526-6594.  Per-launch grids snapped
    # to whole waves (e.g. 50 instead of 56 CTAs for the 98 pair blocks of a stage-5 layer)
    # measured no gain: the SMs a short last wave leaves idle already run the next launch.
    idx = list(range(len(convs)))
    if order == "lpt":
        idx.sort(key=lambda i: -_est_us(convs[i][0], convs[i][1], convs[i][3]))
    elif order == "mix":
        idx = mixed_order(convs)
    elif order != "given":
        raise ValueError(f"unknown sweep order {order!r}")
    out = [None] * len(convs)
    for pos, i in enumerate(idx):
        x, w, args, y = convs[i]
        f = base | (_lib.FLAG_BARRIER if pos == 0 else 0)
        out[i] = conv_device(x, w, *args, y=y, out_dtype=y.dtype, flags=f, num_ctas=grid)
    return out


def sweep_flops(convs: Iterable) -> float:
    """2 * N*P*Q*K * R*S*C summed over ``(x, w, args, y)`` tuples."""
    total = 0.0
    for x, w, args, y in convs:
        total += 2.0 * y.numel() * w.shape[0] * w.shape[1] * w.shape[2]
    return total
