"""Kernel plug-in surface -- the drop-in for ``sasim._kernels``
(/root/reference/pkg/src/sasim/_kernels/__init__.py).

Same names and argument meaning as the reference:

* :func:`conv2d_nhwc`      (reference __init__.py:37-46)
* :func:`tile_gather_nhwc` (reference __init__.py:49-50)
* :func:`im2col_nhwc`      (reference __init__.py:53-54)
* :func:`lru_simulate`     (reference __init__.py:57-59)
* ``BACKEND``              (reference __init__.py:16-26)

Differences, by design (BASELINE.json north_star):

* One backend only -- hand-written sm_100a CUDA behind ``libimconv.so``.
  There is no ``SASIM_PURE_PYTHON`` switch and no CPU fallback; without a
  CUDA device every compute call raises ``RuntimeError``.
* Arithmetic types are the tensor-core ones.  Integer operands run as
  int8 x int8 -> int32 (bit-exact; values must lie in [-128, 127] and the
  accumulator bound R*S*C*2**14 must stay below 2**31, else ``ValueError``).
  Floating operands run as bf16 (or fp16) x bf16 -> fp32 accumulate.
  Numpy in -> numpy out (ints come back int64 like the reference's
  ``_norm``, floats in the input's float dtype); CUDA tensors in -> CUDA
  tensor out (bf16/fp16 in -> same dtype out unless ``out_dtype``).
* Shape checks happen here (the reference kernel level silently accepts a
  channel mismatch on its int path); mismatches raise
  ``ValueError``.
"""

from __future__ import annotations

import numpy as np
import torch

from .. import _device as D
from .. import _lib

BACKEND = "sm_100a"


def _out_extent(size, f, stride, pad, dil):
    return (size + 2 * pad - dil * (f - 1) - 1) // stride + 1


def _plan_dtypes(x, w, compute, out_dtype):
    """Decide (compute torch dtype, output torch dtype, numpy result dtype)."""
    xd, wd = D.torch_dtype_of(x), D.torch_dtype_of(w)
    if D.is_integer_dtype(xd) and D.is_integer_dtype(wd):
        if compute not in (None, "int8"):
            raise ValueError(f"integer operands compute as int8, not {compute!r}")
        np_res = None if isinstance(x, torch.Tensor) else np.int64
        return torch.int8, torch.int32, np_res
    if compute is None:
        compute = "f16" if (xd == torch.float16 and wd == torch.float16) else "bf16"
    cdt = {"bf16": torch.bfloat16, "f16": torch.float16}.get(compute)
    if cdt is None:
        raise ValueError(f"unsupported compute type {compute!r} (bf16, f16, int8)")
    if out_dtype is None:
        if xd in (torch.bfloat16, torch.float16) and xd == cdt:
            odt = cdt
        else:
            odt = torch.float32
    else:
        odt = out_dtype
    if odt not in (cdt, torch.float32):
        raise ValueError(f"output dtype {odt} not supported for {cdt} inputs")
    np_res = None
    if not isinstance(x, torch.Tensor):  # numpy in -> numpy out
        np_res = np.float64 if np.asarray(x).dtype == np.float64 or np.asarray(w).dtype == np.float64 \
            else np.float32
    return cdt, odt, np_res


def _check_int8(t: torch.Tensor, what: str):
    if t.dtype == torch.int8 or t.numel() == 0:
        return
    lo, hi = torch.aminmax(t)
    if int(lo) < -128 or int(hi) > 127:
        raise ValueError(f"{what} values outside int8 range [-128, 127]; the tensor-core integer "
                         "path is int8 x int8 -> int32")


def conv_device(xd: torch.Tensor, wd: torch.Tensor, sh=1, sw=1, ph=0, pw=0, dh=1, dw=1, *,
                out_dtype: torch.dtype | None = None, tile_n: int = 0, num_ctas: int = 0,
                order: int = _lib.ORDER_REUSE_AWARE, y: torch.Tensor | None = None,
                flags: int = 0) -> torch.Tensor:
    """Core device call: CUDA tensors already in the compute dtype
    (bf16 / f16 / int8), x (N,H,W,C), w (R,S,C,K) -> y (N,P,Q,K)."""
    if xd.dim() != 4 or wd.dim() != 4:
        raise ValueError("x must be (N,H,W,C) and w (R,S,C,K)")
    n, h, wi, c = xd.shape
    r, s, c2, k = wd.shape
    if c != c2:
        raise ValueError(f"input channels {c} != filter channels {c2}")
    if min(sh, sw, dh, dw) < 1 or min(ph, pw) < 0:
        raise ValueError("stride/dilation must be >= 1 and padding >= 0")
    p, q = _out_extent(h, r, sh, ph, dh), _out_extent(wi, s, sw, pw, dw)
    if dh * (r - 1) + 1 > h + 2 * ph or dw * (s - 1) + 1 > wi + 2 * pw or p < 1 or q < 1:
        raise ValueError("effective filter extent exceeds the padded input")
    code = D._TORCH_CODE[xd.dtype]
    if wd.dtype != xd.dtype:
        raise ValueError("x and w must share the compute dtype")
    if out_dtype is None:
        out_dtype = torch.int32 if code == _lib.I8 else xd.dtype
    ocode = D._TORCH_CODE[out_dtype]
    e = D._ELEM[code]
    c_pad, k_pad = D.aligned_channels(c, e), D.aligned_k(k, e)
    if code == _lib.I8 and r * s * c >= (1 << 17):
        raise ValueError("int8 reduction length R*S*C >= 2**17 could overflow the int32 accumulator")
    xp = D.pad_nhwc(xd.contiguous(), c_pad)
    wp = D.pad_hwcn(wd.contiguous(), c_pad, k_pad)
    direct = (k_pad == k)
    if y is None or not direct:
        yk = torch.empty((n, p, q, k_pad), dtype=out_dtype, device=xd.device)
    else:
        if tuple(y.shape) != (n, p, q, k) or y.dtype != out_dtype or not y.is_contiguous():
            raise ValueError("preallocated y has the wrong shape/dtype/layout")
        yk = y
    a = _lib.ImconvArgs()
    a.x, a.w, a.y = xp.data_ptr(), wp.data_ptr(), yk.data_ptr()
    a.in_dtype, a.out_dtype = code, ocode
    a.n, a.h, a.w_, a.c = n, h, wi, c_pad
    a.k, a.r, a.s = k_pad, r, s
    a.stride_h, a.stride_w, a.pad_h, a.pad_w, a.dil_h, a.dil_w = sh, sw, ph, pw, dh, dw
    a.tile_n, a.num_ctas, a.order, a.flags = tile_n, num_ctas, order, flags
    _lib.check(_lib.lib.imconv_conv2d_nhwc(a, D.stream_handle()), "imconv_conv2d_nhwc")
    if k_pad != k:
        yk = yk[..., :k].contiguous()
        if y is not None:
            y.copy_(yk)
            return y
    return yk


_COPY_STREAMS: dict = {}


def _copy_streams(dev: torch.device):
    """(host->device, device->host) copy streams of a device, created once."""
    key = dev.index
    if key not in _COPY_STREAMS:
        _COPY_STREAMS[key] = (torch.cuda.Stream(dev), torch.cuda.Stream(dev))
    return _COPY_STREAMS[key]


def _conv_host(x: torch.Tensor, w: torch.Tensor, args, cdt, odt, out, **kw) -> torch.Tensor:
    """Host tensors in, host tensor out, with the transfers pipelined.

    The batch is split into up to four chunks: chunk i+1 is uploaded on a
    copy stream while chunk i computes on the caller's current stream and
    chunk i-1 is downloaded on a second copy stream, so the two PCIe
    directions and the tensor cores overlap (a serial upload -> conv ->
    download pays them one after another); uploads wait for no GPU work, so
    consecutive calls overlap too.  The result is ordered before later work
    on the caller's stream.  With ``out`` (pinned CPU tensor) the call
    is asynchronous like a CUDA copy; without it, a pinned result is
    allocated and the call returns once it is ready.
    """
    dev = D.require_cuda()
    if cdt == torch.int8 and x.dtype != torch.int8:
        _check_int8(x, "input")
        x = x.to(torch.int8)
    if cdt == torch.int8 and w.dtype != torch.int8:
        _check_int8(w, "filter")
        w = w.to(torch.int8)
    x, w = x.contiguous(), w.contiguous()
    n, h, wi, c = x.shape
    r, s_, _, k = w.shape
    sh, sw, ph, pw, dh, dw = args
    shape = (n, _out_extent(h, r, sh, ph, dh), _out_extent(wi, s_, sw, pw, dw), k)
    sync = out is None
    if out is None:
        out = torch.empty(shape, dtype=odt, pin_memory=True)
    elif out.is_cuda or tuple(out.shape) != shape or out.dtype != odt or not out.is_contiguous():
        raise ValueError(f"out must be a contiguous CPU tensor {shape} of {odt}")
    cur = torch.cuda.current_stream(dev)
    s_in, s_out = _copy_streams(dev)
    # uploads read host memory into fresh device buffers, so they wait for no GPU
    # work: the next call's upload overlaps this call's download (full-duplex PCIe)
    chunks = max(1, min(4, n, x.numel() * x.element_size() // (8 << 20)))  # >= 8 MB per chunk
    bounds = [(i * n // chunks, (i + 1) * n // chunks) for i in range(chunks)]
    with torch.cuda.stream(s_in):
        wd = w.to(dev, non_blocking=True)
        wd = wd if wd.dtype == cdt else wd.to(cdt)
    for a, b in bounds:
        with torch.cuda.stream(s_in):
            xd = x[a:b].to(dev, non_blocking=True)
            xd = xd if xd.dtype == cdt else xd.to(cdt)
            landed = torch.cuda.Event()
            landed.record(s_in)
        cur.wait_event(landed)
        xd.record_stream(cur)
        wd.record_stream(cur)
        y = conv_device(xd, wd, *args, out_dtype=odt, **kw)
        done = torch.cuda.Event()
        done.record(cur)
        s_out.wait_event(done)
        with torch.cuda.stream(s_out):
            out[a:b].copy_(y, non_blocking=True)
        y.record_stream(s_out)
    fin = torch.cuda.Event()
    fin.record(s_out)
    cur.wait_event(fin)
    if sync:
        cur.synchronize()
    return out


def conv2d_nhwc(x, w, sh, sw, ph, pw, dh, dw, *, compute: str | None = None, out_dtype=None,
                tile_n: int = 0, num_ctas: int = 0, order: str = "reuse_aware", flags: int = 0, out=None):
    """Direct convolution NHWC x HWCN -> NHWC with virtual zero padding.

    Drop-in for the reference's ``conv2d_nhwc(x, w, sh, sw, ph, pw, dh, dw)``
    (_kernels/__init__.py:37-46).  Computed by the sm_100a implicit-im2col
    tcgen05 kernel; see the module docstring for dtype routing.  CPU torch
    tensors take the pipelined host path (:func:`_conv_host`; ``out`` = a
    pinned CPU result tensor makes the call asynchronous).
    """
    cdt, odt, np_res = _plan_dtypes(x, w, compute, out_dtype)
    ordc = {"reuse_aware": _lib.ORDER_REUSE_AWARE, "filter_major": _lib.ORDER_FILTER_MAJOR}[order]
    if isinstance(x, torch.Tensor) and isinstance(w, torch.Tensor) and not x.is_cuda and not w.is_cuda:
        if x.dim() != 4 or w.dim() != 4 or x.shape[3] != w.shape[2]:
            raise ValueError(f"x (N,H,W,C) and w (R,S,C,K) expected, got {tuple(x.shape)} x {tuple(w.shape)}")
        return _conv_host(x, w, (sh, sw, ph, pw, dh, dw), cdt, odt, out, tile_n=tile_n, num_ctas=num_ctas,
                          order=ordc, flags=flags)
    if out is not None:
        raise ValueError("out= is for CPU (host) tensors; device calls return a new tensor")
    xd = D.to_device(x)
    wd = D.to_device(w)
    if cdt == torch.int8:
        _check_int8(xd, "input")
        _check_int8(wd, "filter")
    xd, wd = xd.to(cdt), wd.to(cdt)
    y = conv_device(xd, wd, sh, sw, ph, pw, dh, dw, out_dtype=odt, tile_n=tile_n, num_ctas=num_ctas, order=ordc,
                    flags=flags)
    if np_res is not None and not D.is_device_array(x):
        return D.to_host(y, np_res)
    return y


def tile_gather_nhwc(x, r, s, sh, sw, ph, pw, dh, dw, ho, wo):
    """One decomposed 1x1 tile's (n*ho*wo, c) operand, zeros at padding.

    Drop-in for the reference's tile_gather_nhwc (_kernels/__init__.py:49-50,
    _native.pyx:50-69).  Inside the implicit kernel this gather is done by
    the TMA engine straight into shared memory and never stored; this entry
    point materialises it for the reference API's callers.
    """
    host = not D.is_device_array(x)
    xd = D.to_device(x)
    if xd.dim() != 4:
        raise ValueError("x must be (N,H,W,C)")
    n, h, wi, c = xd.shape
    out = torch.empty((n * ho * wo, c), dtype=xd.dtype, device=xd.device)
    if out.numel():
        _lib.check(_lib.lib.imconv_tile_gather_nhwc(xd.data_ptr(), out.data_ptr(), xd.element_size(), n, h, wi, c,
                                                    r, s, sh, sw, ph, pw, dh, dw, ho, wo, D.stream_handle()),
                   "imconv_tile_gather_nhwc")
    return D.to_host(out, np.asarray(x).dtype) if host else out


def im2col_nhwc(x, hf, wf, sh, sw, ph, pw, dh, dw, channel_first):
    """Explicit lowering to (n*ho*wo, hf*wf*c); drop-in for the reference's
    im2col_nhwc (_kernels/__init__.py:53-54, _native.pyx:72-99)."""
    host = not D.is_device_array(x)
    xd = D.to_device(x)
    if xd.dim() != 4:
        raise ValueError("x must be (N,H,W,C)")
    n, h, wi, c = xd.shape
    ho, wo = _out_extent(h, hf, sh, ph, dh), _out_extent(wi, wf, sw, pw, dw)
    out = torch.empty((n * ho * wo, hf * wf * c), dtype=xd.dtype, device=xd.device)
    if out.numel():
        _lib.check(_lib.lib.imconv_im2col_nhwc(xd.data_ptr(), out.data_ptr(), xd.element_size(), n, h, wi, c, hf, wf,
                                               sh, sw, ph, pw, dh, dw, int(bool(channel_first)),
                                               D.stream_handle()), "imconv_im2col_nhwc")
    return D.to_host(out, np.asarray(x).dtype) if host else out


def gemm_device(a: torch.Tensor, b: torch.Tensor, out_dtype=None) -> torch.Tensor:
    """(m, kd) @ (kd, n) on the tcgen05 kernel (1x1 stride-1 convolution)."""
    m, kd = a.shape
    kd2, n = b.shape
    if kd != kd2:
        raise ValueError(f"inner dims mismatch: {tuple(a.shape)} x {tuple(b.shape)}")
    y = conv_device(a.reshape(1, 1, m, kd), b.reshape(1, 1, kd, n), out_dtype=out_dtype)
    return y.reshape(m, n)


def lru_simulate(keys, capacity):
    """Fully-associative LRU replay -> (hits, misses); drop-in for the
    reference's lru_simulate (_kernels/__init__.py:57-59).  Host C++."""
    import ctypes

    k = np.ascontiguousarray(np.asarray(keys, dtype=np.int64))
    h, m = ctypes.c_int64(0), ctypes.c_int64(0)
    _lib.check(_lib.lib.imconv_lru_simulate(k.ctypes.data, k.size, int(capacity), ctypes.byref(h),
                                            ctypes.byref(m)), "imconv_lru_simulate")
    return int(h.value), int(m.value)
