"""The reference's own CPU kernels, compiled from its sources by
oracle/build_ref.py into oracle/_ref/ -- TEST INFRASTRUCTURE ONLY.

Used by ``tests/`` (pinning the restatement in oracle.py against the real
thing) and by ``bench.py``'s CPU legs (``--impl reference`` and the
``cpu_baseline`` sample), where it is the timed reference implementation
("kind": "reference").  The product package never imports it.

:func:`conv2d_nhwc` applies the reference's routing
(/root/reference/pkg/src/sasim/_kernels/__init__.py:29-46): operands coerced
to {int64, float32, float64} (``_norm``), int64 to the compiled scalar loop
(``_native.conv2d_nhwc``, _native.pyx:20-47), floats to the numpy tap
accumulation (``_fallback.conv2d_nhwc``, _fallback.py:17-42).
"""

from __future__ import annotations

import importlib.util
import os

import numpy as np

from . import build_ref

_MODS = None
_KERNEL_DTYPES = (np.int64, np.float32, np.float64)


def available() -> bool:
    return len(build_ref.built()) == len(build_ref.MODULES)


def modules():
    """(_native, _fallback) extension modules from oracle/_ref (ImportError if not built)."""
    global _MODS
    if _MODS is None:
        paths = build_ref.built()
        if len(paths) != len(build_ref.MODULES):
            raise ImportError("oracle/_ref is not built (python oracle/build_ref.py, needs /root/reference)")
        mods = {}
        for name, path in paths.items():
            spec = importlib.util.spec_from_file_location(name, path)
            m = importlib.util.module_from_spec(spec)
            spec.loader.exec_module(m)
            mods[name] = m
        _MODS = (mods["_native"], mods["_fallback"])
    return _MODS


def shared_objects() -> list:
    return sorted(build_ref.built().values())


def _norm(a):
    """__init__.py:29-34."""
    a = np.asarray(a)
    if a.dtype not in _KERNEL_DTYPES:
        a = a.astype(np.int64 if np.issubdtype(a.dtype, np.integer) else np.float64)
    return np.ascontiguousarray(a)


def conv2d_nhwc(x, w, sh, sw, ph, pw, dh, dw):
    """__init__.py:37-46, executed by the compiled reference modules."""
    native, fallback = modules()
    x, w = _norm(x), _norm(w)
    if x.dtype != w.dtype:
        dt = np.result_type(x, w)
        x, w = x.astype(dt), w.astype(dt)
    impl = native if x.dtype == np.int64 else fallback
    return impl.conv2d_nhwc(x, w, sh, sw, ph, pw, dh, dw)
