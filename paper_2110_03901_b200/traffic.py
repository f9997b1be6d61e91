"""DRAM-traffic prediction for the kernel's B200 raster.

The reference scores block orders with an LRU replay of the gathered element
stream (``blocksched.reuse_traffic``, blocksched.py:102-151; keys are (h, w, c)
without the image index, so every image replays the same stream).  Here the
same idea is applied to what actually runs on the GPU: ``predict`` calls the
host C++ replay ``imconv_predict_traffic`` (include/imconv.h), which walks the
generic kernel's persistent schedule -- block shape, CTA round-robin,
REUSE_AWARE / FILTER_MAJOR k-subtile order, B-stationary and split-K
decisions, all from the launcher's own planner -- as 128-byte line accesses
(batch-aware NHWC keys) through a write-back LRU the size of L2.  Host code:
no GPU needed.  ``tools/traffic_validate.py`` compares the prediction with
the DRAM bytes ncu measures.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

from . import _lib
from .core import ConvSpec

L2_BYTES_B200 = 126 * 1024 * 1024  # B200 L2 (both dies)
KERNELS = {0: "generic", 1: "row-band", 2: "halo", 3: "halo-stream"}


@dataclass(frozen=True)
class TrafficPrediction:
    dram_read_bytes: int
    dram_write_bytes: int           # dirty output lines evicted during the kernel
    resident_dirty_bytes: int       # output still in L2 when the kernel ends
    line_requests: int
    compulsory_read_bytes: int      # every distinct input / filter line once
    tiles: int
    bn: int
    mt: int
    grid: int
    k_subtiles: int
    kernel: str                     # kernel conv2d_nhwc picks (the replay models the generic raster)


@dataclass(frozen=True)
class LaunchPlan:
    """What imconv_conv2d_nhwc launches for one layer (imconv_plan)."""

    kernel: str
    grid: int
    bn: int
    mt: int
    ksub: int
    cta_pair: bool
    b_resident: bool
    sk_split: int
    tiles: int
    sk_tail: int
    sk_mode: int = 0

    @property
    def branch(self) -> str:
        """Short label of the planner branch (tests and tools group layers by it)."""
        if self.kernel != "generic":
            return self.kernel
        parts = [f"{128 * self.mt * (2 if self.cta_pair else 1)}x{self.bn}"]
        if self.cta_pair:
            parts.append("pair")
        if self.b_resident:
            parts.append("b-stationary")
        if self.sk_split > 1:
            parts.append(f"split{self.sk_split}")
        if self.sk_mode == 2:
            parts.append("stream-k")
        if self.ksub > 1:
            parts.append(f"ksub{self.ksub}")
        return "generic " + " ".join(parts)


def _args(spec: ConvSpec, dtype: str, out_dtype: str | None, order: str, flags: int):
    from ._device import aligned_channels, aligned_k
    in_code = {"bf16": _lib.BF16, "f16": _lib.F16, "int8": _lib.I8}[dtype]
    e = 1 if dtype == "int8" else 2
    if out_dtype is None:
        out_dtype = "int32" if dtype == "int8" else dtype
    out_code = {"bf16": _lib.BF16, "f16": _lib.F16, "f32": _lib.F32, "int32": _lib.I32}[out_dtype]
    a = _lib.ImconvArgs()
    a.in_dtype, a.out_dtype = in_code, out_code
    a.n, a.h, a.w_ = spec.n, spec.h_i, spec.w_i
    a.c, a.k = aligned_channels(spec.c_i, e), aligned_k(spec.c_o, e)
    a.r, a.s = spec.h_f, spec.w_f
    a.stride_h, a.stride_w, a.pad_h, a.pad_w, a.dil_h, a.dil_w = spec.conv_args()
    a.order = {"reuse_aware": _lib.ORDER_REUSE_AWARE, "filter_major": _lib.ORDER_FILTER_MAJOR}[order]
    a.flags = flags
    return a


def plan(spec: ConvSpec, dtype: str = "bf16", sms: int = 148, out_dtype: str | None = None, flags: int = 0,
         order: str = "reuse_aware") -> LaunchPlan:
    """The launch ``conv2d_nhwc`` issues for ``spec`` on a ``sms``-SM device (host code)."""
    a = _args(spec, dtype, out_dtype, order, flags)
    t = _lib.ImconvPlanInfo()
    _lib.check(_lib.lib.imconv_plan(ctypes.byref(a), int(sms), ctypes.byref(t)), "imconv_plan")
    return LaunchPlan(KERNELS.get(t.kernel, "?"), t.grid, t.bn, t.mt, t.ksub, bool(t.cta_pair), bool(t.b_resident),
                      t.sk_split, t.tiles, t.sk_tail, t.sk_mode)


def predict(spec: ConvSpec, dtype: str = "bf16", order: str = "reuse_aware", l2_bytes: int = L2_BYTES_B200,
            sms: int = 148, out_dtype: str | None = None, flags: int = 0) -> TrafficPrediction:
    """Predicted DRAM traffic of one ``conv2d_nhwc`` launch of ``spec``.

    ``dtype`` is the compute type (bf16 / f16 / int8); channels are padded the
    way the device path pads them (16-byte rows).
    """
    a = _args(spec, dtype, out_dtype, order, flags)
    t = _lib.ImconvTraffic()
    _lib.check(_lib.lib.imconv_predict_traffic(ctypes.byref(a), int(l2_bytes), int(sms), ctypes.byref(t)),
               "imconv_predict_traffic")
    return TrafficPrediction(t.dram_read_bytes, t.dram_write_bytes, t.resident_dirty_bytes, t.line_requests,
                             t.compulsory_read_bytes, t.tiles, t.bn, t.mt, t.grid, t.k_subtiles,
                             KERNELS.get(t.kernel, "?"))
