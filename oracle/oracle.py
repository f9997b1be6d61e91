"""CPU ORACLE -- TEST INFRASTRUCTURE ONLY.

Restatement of the reference's CPU convolution path
(/root/reference/pkg/src/sasim/_kernels/) used as the checker for the
sm_100a kernels and as the timed CPU baseline.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py`` (cpu_baseline leg and
``--impl reference``) may import this module.  The product package
``paper_2110_03901_b200`` never imports it and has no CPU fallback.

Pinning: every function here is checked against vectors produced by the
reference itself (``tests/golden/make_golden.py``) in
``tests/test_oracle_golden.py``.

Two arithmetic paths, mirroring the reference's routing at
``_kernels/__init__.py:37-46``:

* floats -> :func:`conv2d_nhwc_taps`, a numpy restatement of
  ``_fallback.conv2d_nhwc`` (``_fallback.py:17-42``): one strided slice per
  filter tap times ``w[r, s]`` through BLAS matmul, accumulated in
  row-major tap order.
* integers -> :func:`conv2d_nhwc_i64`, the C restatement of
  ``_native.conv2d_nhwc`` (``_native.pyx:20-47``) in ``conv_oracle.c``.
  :func:`conv2d_nhwc_exact_f64` evaluates the same integer sum through
  float64 BLAS, exact while every partial sum stays below 2**53 (int8
  operands: |acc| <= R*S*C*128**2), which makes full-size int8 checks
  tractable; it is itself pinned against the int64 path in the tests.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_BUILD = os.path.join(_HERE, "_build")
_LIB_PATH = os.path.join(_BUILD, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile conv_oracle.c -> oracle/_build/liboracle.so (gcc -O3 -fopenmp)."""
    src = os.path.join(_HERE, "conv_oracle.c")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        os.makedirs(_BUILD, exist_ok=True)
        subprocess.check_call(["gcc", "-O3", "-fPIC", "-shared", "-fopenmp", "-std=c11",
                               src, "-o", _LIB_PATH])
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        i64 = ctypes.c_int64
        vp = ctypes.c_void_p
        L.oracle_conv2d_nhwc_i64.argtypes = [vp, vp, vp] + [i64] * 13 + [ctypes.c_int]
        L.oracle_conv2d_nhwc_i64.restype = None
        L.oracle_tile_gather_nhwc.argtypes = [vp, vp] + [i64] * 15
        L.oracle_tile_gather_nhwc.restype = None
        L.oracle_im2col_nhwc.argtypes = [vp, vp] + [i64] * 13 + [ctypes.c_int]
        L.oracle_im2col_nhwc.restype = None
        L.oracle_lru_simulate.argtypes = [vp, i64, i64, ctypes.POINTER(i64), ctypes.POINTER(i64)]
        L.oracle_lru_simulate.restype = ctypes.c_int
        _lib = L
    return _lib


def out_extent(size, f, stride, pad, dil):
    """core.py:89-95."""
    return (size + 2 * pad - dil * (f - 1) - 1) // stride + 1


def _ptr(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data)


def conv2d_nhwc_i64(x, w, sh, sw, ph, pw, dh, dw, threads: int = 1) -> np.ndarray:
    """Integer direct conv (int64 accumulate); _native.pyx:20-47."""
    x = np.ascontiguousarray(x, dtype=np.int64)
    w = np.ascontiguousarray(w, dtype=np.int64)
    n, hi, wi, ci = x.shape
    hf, wf, ci2, co = w.shape
    assert ci == ci2
    ho, wo = out_extent(hi, hf, sh, ph, dh), out_extent(wi, wf, sw, pw, dw)
    y = np.empty((n, ho, wo, co), dtype=np.int64)
    lib().oracle_conv2d_nhwc_i64(_ptr(x), _ptr(w), _ptr(y), n, hi, wi, ci, hf, wf, co,
                                 sh, sw, ph, pw, dh, dw, int(threads))
    return y


def conv2d_nhwc_taps(x, w, sh, sw, ph, pw, dh, dw) -> np.ndarray:
    """Float direct conv by per-tap strided slices @ w[r,s]; _fallback.py:17-42.

    The tap loop is row-major (r outer, s inner) and each tap's bounds are
    the output rows/cols whose input index lands inside the image
    (_fallback.py:29-40).
    """
    n, hi, wi, ci = x.shape
    hf, wf, _, co = w.shape
    ho, wo = out_extent(hi, hf, sh, ph, dh), out_extent(wi, wf, sw, pw, dw)
    out = np.zeros((n, ho, wo, co), dtype=np.result_type(x, w))
    for r in range(hf):
        i0 = max(0, -(-(ph - r * dh) // sh))
        i1 = min(ho, (hi - 1 - r * dh + ph) // sh + 1)
        if i0 >= i1:
            continue
        for s in range(wf):
            j0 = max(0, -(-(pw - s * dw) // sw))
            j1 = min(wo, (wi - 1 - s * dw + pw) // sw + 1)
            if j0 >= j1:
                continue
            hs = slice(i0 * sh + r * dh - ph, (i1 - 1) * sh + r * dh - ph + 1, sh)
            ws = slice(j0 * sw + s * dw - pw, (j1 - 1) * sw + s * dw - pw + 1, sw)
            out[:, i0:i1, j0:j1, :] += x[:, hs, ws, :] @ w[r, s]
    return out


def conv2d_nhwc_exact_f64(x, w, sh, sw, ph, pw, dh, dw) -> np.ndarray:
    """Integer conv evaluated exactly through float64 BLAS (|partial sums| < 2**53)."""
    xf = np.asarray(x, dtype=np.float64)
    wf_ = np.asarray(w, dtype=np.float64)
    bound = float(np.abs(xf).max(initial=0)) * float(np.abs(wf_).max(initial=0)) * \
        w.shape[0] * w.shape[1] * w.shape[2]
    if bound >= 2.0 ** 53:
        raise ValueError("float64 path would not be exact for these operands")
    return np.rint(conv2d_nhwc_taps(xf, wf_, sh, sw, ph, pw, dh, dw)).astype(np.int64)


def tile_gather_nhwc(x, r, s, sh, sw, ph, pw, dh, dw, ho, wo) -> np.ndarray:
    """_native.pyx:50-69 (any dtype; it is a copy)."""
    x = np.ascontiguousarray(x)
    n, hi, wi, ci = x.shape
    out = np.empty((n * ho * wo, ci), dtype=x.dtype)
    lib().oracle_tile_gather_nhwc(_ptr(x), _ptr(out), x.itemsize, n, hi, wi, ci,
                                  r, s, sh, sw, ph, pw, dh, dw, ho, wo)
    return out


def im2col_nhwc(x, hf, wf, sh, sw, ph, pw, dh, dw, channel_first) -> np.ndarray:
    """_native.pyx:72-99 (any dtype)."""
    x = np.ascontiguousarray(x)
    n, hi, wi, ci = x.shape
    ho, wo = out_extent(hi, hf, sh, ph, dh), out_extent(wi, wf, sw, pw, dw)
    out = np.empty((n * ho * wo, hf * wf * ci), dtype=x.dtype)
    lib().oracle_im2col_nhwc(_ptr(x), _ptr(out), x.itemsize, n, hi, wi, ci, hf, wf,
                             sh, sw, ph, pw, dh, dw, int(bool(channel_first)))
    return out


def lru_simulate(keys, capacity):
    """_native.pyx:102-149; returns (hits, misses)."""
    keys = np.ascontiguousarray(np.asarray(keys, dtype=np.int64))
    h, m = ctypes.c_int64(0), ctypes.c_int64(0)
    rc = lib().oracle_lru_simulate(_ptr(keys), keys.size, int(capacity), ctypes.byref(h), ctypes.byref(m))
    if rc != 0:
        raise MemoryError("oracle_lru_simulate allocation failed")
    return int(h.value), int(m.value)


def conv_reference(x, w, sh=1, sw=1, ph=0, pw=0, dh=1, dw=1, threads: int = 1) -> np.ndarray:
    """The reference's dtype routing (_kernels/__init__.py:29-46): ints -> int64
    scalar loop, floats -> BLAS tap accumulation (float32 stays float32)."""
    x, w = np.asarray(x), np.asarray(w)
    if np.issubdtype(x.dtype, np.integer) and np.issubdtype(w.dtype, np.integer):
        return conv2d_nhwc_i64(x, w, sh, sw, ph, pw, dh, dw, threads=threads)
    dt = np.result_type(x, w)
    if dt not in (np.float32, np.float64):
        dt = np.float64
    return conv2d_nhwc_taps(x.astype(dt), w.astype(dt), sh, sw, ph, pw, dh, dw)


def reference_conv_loops(x, f, n, h_i, w_i, c_i, c_o, h_f, w_f, sh, sw, ph, pw, dh, dw):
    """Independent brute-force loop nest (tests/conftest.py:7-31 restated);
    pure Python, small cases only."""
    ho, wo = out_extent(h_i, h_f, sh, ph, dh), out_extent(w_i, w_f, sw, pw, dw)
    out = np.zeros((n, ho, wo, c_o), dtype=np.result_type(x, f))
    for b in range(n):
        for i in range(ho):
            for j in range(wo):
                for k in range(c_o):
                    acc = 0
                    for r in range(h_f):
                        hh = i * sh + r * dh - ph
                        if hh < 0 or hh >= h_i:
                            continue
                        for s in range(w_f):
                            ww = j * sw + s * dw - pw
                            if ww < 0 or ww >= w_i:
                                continue
                            for c in range(c_i):
                                acc += x[b, hh, ww, c] * f[r, s, c, k]
                    out[b, i, j, k] = acc
    return out


if __name__ == "__main__":  # pragma: no cover
    build(force=True)
    print(_LIB_PATH)
