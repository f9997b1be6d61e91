"""Functional (OFMap-producing) halves of the reference simulator's methods
(simulator.py:286-293, :354-364, :417-421, :527-532), on the GPU.

The reference's cycle model (``simulate``'s timing half, ``sweep``) models a
700 MHz 128x128 systolic array and is out of scope: on B200 the kernels are
timed for real (bench.py).  What remains is the numerics of each lowering
method, all of which must equal ``direct_conv``:

* CHANNEL_FIRST_IMPLICIT -- the paper's method: the implicit-im2col kernel;
* CHANNEL_LAST_IMPLICIT  -- channel-last lowering (CL im2col @ CL filter);
* EXPLICIT_IM2COL        -- materialised CF lowering (K3) + GEMM (K4);
* GEMM                   -- same lowering product, 1x1-conv view.
"""

from __future__ import annotations

from enum import Enum

from .core import ConvSpec, Layout, Tensor, _as_filter_hwcn, _as_nhwc, direct_conv, gemm
from .core import ShapeError
from .lowering import ColumnOrdering, im2col_explicit, lower_filter


class Method(Enum):
    CHANNEL_FIRST_IMPLICIT = "cf_implicit"
    CHANNEL_LAST_IMPLICIT = "cl_implicit"
    EXPLICIT_IM2COL = "explicit"
    GEMM = "gemm"

    @classmethod
    def parse(cls, name: str) -> "Method":
        """Method from a name or alias (simulator.py:42-58's spellings)."""
        key = name.strip().lower().replace("-", "_")
        aliases = {
            "cf": cls.CHANNEL_FIRST_IMPLICIT, "channel_first": cls.CHANNEL_FIRST_IMPLICIT,
            "channel_first_implicit": cls.CHANNEL_FIRST_IMPLICIT, "cf_implicit": cls.CHANNEL_FIRST_IMPLICIT,
            "cl": cls.CHANNEL_LAST_IMPLICIT, "channel_last": cls.CHANNEL_LAST_IMPLICIT,
            "channel_last_implicit": cls.CHANNEL_LAST_IMPLICIT, "cl_implicit": cls.CHANNEL_LAST_IMPLICIT,
            "explicit": cls.EXPLICIT_IM2COL, "explicit_im2col": cls.EXPLICIT_IM2COL,
            "gemm": cls.GEMM, "plain_gemm": cls.GEMM,
        }
        if key not in aliases:
            raise ShapeError(f"unknown method {name!r}")
        return aliases[key]


Method.PLAIN_GEMM = Method.GEMM  # the reference's member name


ALL_METHODS = tuple(Method)


def channel_first_implicit(spec: ConvSpec, ifmap: Tensor, filters: Tensor, **kw) -> Tensor:
    """Σ over taps of gather(tap) @ f[r, s] without materialising any gather
    (simulator._functional_cf, simulator.py:286-293)."""
    return direct_conv(ifmap, filters, spec, **kw)


def channel_last_implicit(spec: ConvSpec, ifmap: Tensor, filters: Tensor, **kw) -> Tensor:
    """The channel-last baseline (simulator.py:300-364): reduction
    order k = (c, r, s), A operands gathered element by element by the kernel's
    producer threads (IMCONV_FLAG_CHANNEL_LAST) -- the lowering whose cost grows
    with the stride, kept to reproduce the paper's contrast (tools/stride_contrast.py).
    Integer operands (int8 tensor cores; the baseline gathers 2-byte elements) use
    the explicit channel-last im2col + GEMM, which computes the same OFMap."""
    from . import _device as D, _lib
    xd = ifmap.data if hasattr(ifmap, "data") else ifmap
    if D.is_integer_dtype(D.torch_dtype_of(xd)):
        return explicit_im2col(spec, ifmap, filters, ColumnOrdering.CHANNEL_LAST, **kw)
    kw["flags"] = kw.get("flags", 0) | _lib.FLAG_CHANNEL_LAST
    return direct_conv(ifmap, filters, spec, **kw)


def explicit_im2col(spec: ConvSpec, ifmap: Tensor, filters: Tensor,
                    ordering: ColumnOrdering = ColumnOrdering.CHANNEL_FIRST, **kw) -> Tensor:
    """Materialise the lowered matrix in HBM, then GEMM (simulator.py:527-532)."""
    low = im2col_explicit(ifmap, spec, ordering)
    flt = lower_filter(filters, spec, ordering)
    out = gemm(low, flt, **kw)
    return Tensor.from_array(out.view().reshape(spec.n, spec.h_o, spec.w_o, spec.c_o), Layout.NHWC)


def functional_ofmap(spec: ConvSpec, method: Method, ifmap: Tensor, filters: Tensor, **kw) -> Tensor:
    """The OFMap ``simulate(spec, arch, method, ifmap=, filters=)`` returns."""
    _as_nhwc(ifmap, spec)
    _as_filter_hwcn(filters, spec)
    if method is Method.CHANNEL_FIRST_IMPLICIT:
        return channel_first_implicit(spec, ifmap, filters, **kw)
    if method is Method.CHANNEL_LAST_IMPLICIT:
        return channel_last_implicit(spec, ifmap, filters, **kw)
    return explicit_im2col(spec, ifmap, filters, ColumnOrdering.CHANNEL_FIRST, **kw)


__all__ = ["ALL_METHODS", "Method", "channel_first_implicit", "channel_last_implicit", "explicit_im2col",
           "functional_ofmap"]
