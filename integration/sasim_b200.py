"""sasim/_kernels/_b200.py -- the reference's kernel plug-in backed by libimconv.so.

This file is what a maintainer of the reference (``sasim``) drops in next to
``_native`` and ``_fallback``: it exports the four functions of the plug-in
surface with the reference's signatures and semantics
(/root/reference/pkg/src/sasim/_kernels/__init__.py:37-58):

    conv2d_nhwc(x, w, sh, sw, ph, pw, dh, dw)                        -> new (N, P, Q, K)
    tile_gather_nhwc(x, r, s, sh, sw, ph, pw, dh, dw, ho, wo)        -> new (N*ho*wo, C)
    im2col_nhwc(x, hf, wf, sh, sw, ph, pw, dh, dw, channel_first)    -> new (N*P*Q, R*S*C)
    lru_simulate(keys, capacity)                                     -> (hits, misses)

and is selected in ``_kernels/__init__.py:16-26``.  It
binds the C ABI of include/imconv.h with ctypes only -- no code of the
``paper_2110_03901_b200`` package is imported -- so it is exactly what the
reference would ship.  Arrays in and out are numpy (as the reference's
callers expect); the library computes on the GPU:

  * integer inputs whose values fit int8 run the int8 -> int32 tensor-core
    path (bit-exact; the result is returned as int64 like ``_native``);
  * float inputs run the bf16 path with fp32 accumulation and fp32 output
    (integer-valued floats up to |x| <= 256 are exact in bf16; other values
    carry bf16 input rounding -- BASELINE.json's 1e-2 tolerance);
  * integers outside int8 cannot run on the tensor cores: ``ValueError``
    (the reference keeps ``_native`` for them; this plug-in has no CPU path).

Channels are zero-padded to 16-byte rows on the device (exact: padded
channels contribute 0).  Errors from the library raise ``ValueError`` with
``imconv_strerror``'s text, matching the reference's exception type for bad
arguments.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

LIB_PATH = os.environ.get("SASIM_B200_LIB") or os.path.join(
    os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2110_03901_b200", "libimconv.so")

_BF16, _I8, _F32, _I32 = 0, 2, 3, 4


class _Args(ctypes.Structure):
    """imconv_conv_args (include/imconv.h)."""

    _fields_ = [("x", ctypes.c_void_p), ("w", ctypes.c_void_p), ("y", ctypes.c_void_p),
                ("in_dtype", ctypes.c_int32), ("out_dtype", ctypes.c_int32),
                ("n", ctypes.c_int64), ("h", ctypes.c_int64), ("w_", ctypes.c_int64), ("c", ctypes.c_int64),
                ("k", ctypes.c_int64), ("r", ctypes.c_int64), ("s", ctypes.c_int64),
                ("stride_h", ctypes.c_int32), ("stride_w", ctypes.c_int32),
                ("pad_h", ctypes.c_int32), ("pad_w", ctypes.c_int32),
                ("dil_h", ctypes.c_int32), ("dil_w", ctypes.c_int32),
                ("tile_n", ctypes.c_int32), ("num_ctas", ctypes.c_int32),
                ("order", ctypes.c_int32), ("flags", ctypes.c_int32)]


_L = None


def _lib():
    global _L
    if _L is None:
        L = ctypes.CDLL(LIB_PATH)
        vp, i32, i64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
        L.imconv_conv2d_nhwc.argtypes = [ctypes.POINTER(_Args), vp]
        L.imconv_conv2d_nhwc.restype = ctypes.c_int
        L.imconv_out_extent.argtypes = [i64] * 5
        L.imconv_out_extent.restype = i64
        L.imconv_tile_gather_nhwc.argtypes = [vp, vp, i32, i64, i64, i64, i64] + [i32] * 8 + [i64, i64, vp]
        L.imconv_tile_gather_nhwc.restype = ctypes.c_int
        L.imconv_im2col_nhwc.argtypes = [vp, vp, i32, i64, i64, i64, i64] + [i32] * 9 + [vp]
        L.imconv_im2col_nhwc.restype = ctypes.c_int
        L.imconv_lru_simulate.argtypes = [vp, i64, i64, ctypes.POINTER(i64), ctypes.POINTER(i64)]
        L.imconv_lru_simulate.restype = ctypes.c_int
        L.imconv_strerror.argtypes = [ctypes.c_int]
        L.imconv_strerror.restype = ctypes.c_char_p
        _L = L
    return _L


def _check(rc: int) -> None:
    if rc != 0:
        raise ValueError(_lib().imconv_strerror(rc).decode())


def _stream(torch):
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _device_operand(arr, torch):
    """numpy -> (device tensor in the kernel's element type, is_int)."""
    a = np.ascontiguousarray(np.asarray(arr))
    if np.issubdtype(a.dtype, np.integer):
        if a.size and (a.min() < -128 or a.max() > 127):
            raise ValueError("integer operands outside int8 cannot run on the int8 tensor-core path")
        return torch.from_numpy(a.astype(np.int8)).cuda(), True
    return torch.from_numpy(a.astype(np.float32)).cuda().to(torch.bfloat16), False


def _pad_last(t, mult_elems, torch):
    extra = (-t.shape[-1]) % mult_elems
    return torch.nn.functional.pad(t, (0, extra)) if extra else t.contiguous()


def conv2d_nhwc(x, w, sh, sw, ph, pw, dh, dw):
    """_kernels/__init__.py:37-46: (N,H,W,C) x (R,S,C,K) -> new (N,P,Q,K)."""
    import torch
    xd, ints = _device_operand(x, torch)
    wd, w_ints = _device_operand(w, torch)
    if ints != w_ints:  # the reference promotes to a common dtype (__init__.py:39-41): float wins
        xd, wd, ints = xd.float().to(torch.bfloat16), wd.float().to(torch.bfloat16), False
    n, h, wi, c = xd.shape
    r, s, c2, k = wd.shape
    if c2 != c:
        raise ValueError(f"filter has {c2} input channels, input has {c}")
    e = 1 if ints else 2
    xd = _pad_last(xd, 16 // e, torch)                                    # C to 16-byte rows
    wd = torch.nn.functional.pad(wd, (0, 0, 0, xd.shape[-1] - c))         # filter C alike
    wd = _pad_last(wd, 16 // e, torch)                                    # K to 16-byte rows
    cp, kp = xd.shape[-1], wd.shape[-1]
    L = _lib()
    p = L.imconv_out_extent(h, r, sh, ph, dh)
    q = L.imconv_out_extent(wi, s, sw, pw, dw)
    if p < 1 or q < 1:
        raise ValueError("effective filter extent exceeds the padded input")
    y = torch.empty((n, p, q, kp), device="cuda", dtype=torch.int32 if ints else torch.float32)
    a = _Args(xd.data_ptr(), wd.data_ptr(), y.data_ptr(), _I8 if ints else _BF16, _I32 if ints else _F32,
              n, h, wi, cp, kp, r, s, sh, sw, ph, pw, dh, dw, 0, 0, 0, 0)
    _check(L.imconv_conv2d_nhwc(ctypes.byref(a), _stream(torch)))
    out = y[..., :k].cpu().numpy()
    if ints:
        return out.astype(np.int64)
    dt = np.result_type(np.asarray(x).dtype, np.asarray(w).dtype)
    return out.astype(dt if np.issubdtype(dt, np.floating) else np.float64)


def tile_gather_nhwc(x, r, s, sh, sw, ph, pw, dh, dw, ho, wo):
    """_native.pyx:50-69: one tap's (N*ho*wo, C) operand, zeros at padding."""
    import torch
    a = np.ascontiguousarray(np.asarray(x))
    xd = torch.from_numpy(a).cuda()
    n, h, w, c = a.shape
    out = torch.empty((n * ho * wo, c), dtype=xd.dtype, device="cuda")
    _check(_lib().imconv_tile_gather_nhwc(xd.data_ptr(), out.data_ptr(), a.itemsize, n, h, w, c,
                                          r, s, sh, sw, ph, pw, dh, dw, ho, wo, _stream(torch)))
    return out.cpu().numpy()


def im2col_nhwc(x, hf, wf, sh, sw, ph, pw, dh, dw, channel_first):
    """_native.pyx:72-99: the explicit lowered matrix (CF or CL column order)."""
    import torch
    a = np.ascontiguousarray(np.asarray(x))
    xd = torch.from_numpy(a).cuda()
    n, h, w, c = a.shape
    L = _lib()
    p = L.imconv_out_extent(h, hf, sh, ph, dh)
    q = L.imconv_out_extent(w, wf, sw, pw, dw)
    out = torch.empty((n * p * q, hf * wf * c), dtype=xd.dtype, device="cuda")
    _check(L.imconv_im2col_nhwc(xd.data_ptr(), out.data_ptr(), a.itemsize, n, h, w, c, hf, wf, sh, sw, ph, pw,
                                dh, dw, 1 if channel_first else 0, _stream(torch)))
    return out.cpu().numpy()


def lru_simulate(keys, capacity):
    """_native.pyx:102-149: (hits, misses) of an element-key LRU of `capacity` entries."""
    k = np.ascontiguousarray(np.asarray(keys, dtype=np.int64))
    hits, misses = ctypes.c_int64(0), ctypes.c_int64(0)
    _check(_lib().imconv_lru_simulate(k.ctypes.data, k.size, int(capacity), ctypes.byref(hits),
                                      ctypes.byref(misses)))
    return int(hits.value), int(misses.value)
