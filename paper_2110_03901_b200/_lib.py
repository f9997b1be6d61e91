"""ctypes binding of the C ABI in include/imconv.h (libimconv.so, in-tree).

The shared object is mapped on first use of ``_lib.lib`` (PEP 562 module
``__getattr__``), not at import: importing the package for its host-side
pieces (ConvSpec, the layer tables) loads no native code.  There is no
fallback: if the shared object is missing the first call fails loudly, and
every compute call raises when no CUDA device is present.
"""

from __future__ import annotations

import ctypes
import os

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libimconv.so")
# the same sources built with per-role wait counters (-DIMCONV_INSTRUMENT=1): loaded only
# by diagnostic tools that ask for it explicitly (use_instrumented), never by the package
LIB_INSTR_PATH = os.path.join(_PKG, "libimconv_instr.so")
# the same sources with the device / planner invariant checks on (-DIMCONV_DEBUG=1): loaded
# only by tests/debug_check.py (use_debug), never by the package
LIB_DEBUG_PATH = os.path.join(_PKG, "libimconv_debug.so")
_loaded = None

# element-type codes, include/imconv.h
BF16, F16, I8, F32, I32 = 0, 1, 2, 3, 4
ORDER_REUSE_AWARE, ORDER_FILTER_MAJOR = 0, 1
FLAG_SINGLE_CTA, FLAG_CTA_PAIR, FLAG_KSUB1, FLAG_MT1, FLAG_GATHER16, FLAG_NO_HALO = 1, 2, 4, 8, 16, 32
FLAG_CHANNEL_LAST = 64
FLAG_STATIC_FILTER = 128  # filter not written by kernels in flight: loads start before the PDL wait
FLAG_INDEPENDENT = 256  # nothing in flight touches this launch's buffers: no PDL wait at all (implies STATIC_FILTER)
FLAG_BARRIER = 512  # waits for every preceding grid before later launches may start (head of a batch)

# every symbol include/imconv.h declares (checked by tests/test_abi.py)
EXPORTED = (
    "imconv_conv2d_nhwc", "imconv_out_extent", "imconv_gemm", "imconv_tile_gather_nhwc",
    "imconv_im2col_nhwc", "imconv_pad_copy", "imconv_lru_simulate", "imconv_abi_version",
    "imconv_device_sm_count", "imconv_strerror", "imconv_launch_count", "imconv_reset_launch_count",
    "imconv_debug_set_buffer", "imconv_debug_set_flags", "imconv_predict_traffic", "imconv_plan",
)


class ImconvArgs(ctypes.Structure):
    """Mirror of imconv_conv_args (include/imconv.h)."""

    _fields_ = [
        ("x", ctypes.c_void_p), ("w", ctypes.c_void_p), ("y", ctypes.c_void_p),
        ("in_dtype", ctypes.c_int32), ("out_dtype", ctypes.c_int32),
        ("n", ctypes.c_int64), ("h", ctypes.c_int64), ("w_", ctypes.c_int64), ("c", ctypes.c_int64),
        ("k", ctypes.c_int64), ("r", ctypes.c_int64), ("s", ctypes.c_int64),
        ("stride_h", ctypes.c_int32), ("stride_w", ctypes.c_int32),
        ("pad_h", ctypes.c_int32), ("pad_w", ctypes.c_int32),
        ("dil_h", ctypes.c_int32), ("dil_w", ctypes.c_int32),
        ("tile_n", ctypes.c_int32), ("num_ctas", ctypes.c_int32),
        ("order", ctypes.c_int32), ("flags", ctypes.c_int32),
    ]


class ImconvTraffic(ctypes.Structure):
    """Mirror of imconv_traffic (include/imconv.h)."""

    _fields_ = [
        ("dram_read_bytes", ctypes.c_int64), ("dram_write_bytes", ctypes.c_int64),
        ("resident_dirty_bytes", ctypes.c_int64), ("line_requests", ctypes.c_int64),
        ("compulsory_read_bytes", ctypes.c_int64), ("tiles", ctypes.c_int64),
        ("bn", ctypes.c_int32), ("mt", ctypes.c_int32), ("grid", ctypes.c_int32), ("k_subtiles", ctypes.c_int32),
        ("kernel", ctypes.c_int32),
    ]


class ImconvPlanInfo(ctypes.Structure):
    """Mirror of imconv_plan_info (include/imconv.h)."""

    _fields_ = [
        ("kernel", ctypes.c_int32), ("grid", ctypes.c_int32), ("bn", ctypes.c_int32), ("mt", ctypes.c_int32),
        ("ksub", ctypes.c_int32), ("cta_pair", ctypes.c_int32), ("b_resident", ctypes.c_int32),
        ("sk_split", ctypes.c_int32), ("tiles", ctypes.c_int64), ("sk_tail", ctypes.c_int64),
        ("sk_mode", ctypes.c_int32),
    ]


class ImconvError(RuntimeError):
    def __init__(self, code: int, what: str):
        self.code = code
        super().__init__(f"{what}: {strerror(code)} (code {code})")


def _load(path: str):
    if not os.path.exists(path):
        raise ImportError(
            f"{path} is not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback)")
    L = ctypes.CDLL(path)
    vp, i32, i64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
    L.imconv_conv2d_nhwc.argtypes = [ctypes.POINTER(ImconvArgs), vp]
    L.imconv_conv2d_nhwc.restype = ctypes.c_int
    L.imconv_out_extent.argtypes = [i64] * 5
    L.imconv_out_extent.restype = i64
    L.imconv_gemm.argtypes = [vp, vp, vp, i32, i32, i64, i64, i64, vp]
    L.imconv_gemm.restype = ctypes.c_int
    L.imconv_tile_gather_nhwc.argtypes = [vp, vp, i32, i64, i64, i64, i64] + [i32] * 8 + [i64, i64, vp]
    L.imconv_tile_gather_nhwc.restype = ctypes.c_int
    L.imconv_im2col_nhwc.argtypes = [vp, vp, i32, i64, i64, i64, i64] + [i32] * 9 + [vp]
    L.imconv_im2col_nhwc.restype = ctypes.c_int
    L.imconv_pad_copy.argtypes = [vp, vp, i32, i64, i64, i64, i64, i64, vp]
    L.imconv_pad_copy.restype = ctypes.c_int
    L.imconv_lru_simulate.argtypes = [vp, i64, i64, ctypes.POINTER(i64), ctypes.POINTER(i64)]
    L.imconv_lru_simulate.restype = ctypes.c_int
    L.imconv_abi_version.argtypes = []
    L.imconv_abi_version.restype = ctypes.c_int
    L.imconv_device_sm_count.argtypes = [ctypes.POINTER(i32)]
    L.imconv_device_sm_count.restype = ctypes.c_int
    L.imconv_strerror.argtypes = [ctypes.c_int]
    L.imconv_strerror.restype = ctypes.c_char_p
    L.imconv_launch_count.argtypes = []
    L.imconv_launch_count.restype = i64
    L.imconv_reset_launch_count.argtypes = []
    L.imconv_reset_launch_count.restype = None
    L.imconv_debug_set_buffer.argtypes = [vp]
    L.imconv_debug_set_buffer.restype = None
    L.imconv_debug_set_flags.argtypes = [ctypes.c_int]
    L.imconv_debug_set_flags.restype = None
    L.imconv_predict_traffic.argtypes = [ctypes.POINTER(ImconvArgs), i64, i32, ctypes.POINTER(ImconvTraffic)]
    L.imconv_predict_traffic.restype = ctypes.c_int
    L.imconv_plan.argtypes = [ctypes.POINTER(ImconvArgs), i32, ctypes.POINTER(ImconvPlanInfo)]
    L.imconv_plan.restype = ctypes.c_int
    return L


def _use(path: str) -> None:
    global _loaded
    if _loaded is not None and _loaded[0] != path:
        raise RuntimeError(f"{_loaded[0]} is already loaded in this process")
    _loaded = (path, _load(path))
    globals()["lib"] = _loaded[1]


def use_instrumented() -> None:
    """Diagnostics only (tools/run_layer.py --waits, tools/timeline_probe.py): bind the
    instrumented build instead of the product library.  Must precede any other use."""
    _use(LIB_INSTR_PATH)


def use_debug() -> None:
    """Checks only (tests/debug_check.py): bind the debug-invariant build (device asserts on
    mbarrier phases, TMEM allocation, split-K tickets, work units, staged/stored chunk counts;
    host asserts on the planner's schedule).  Must precede any other use."""
    _use(LIB_DEBUG_PATH)


def __getattr__(name):
    global _loaded
    if name == "lib":
        if _loaded is None:
            _loaded = (LIB_PATH, _load(LIB_PATH))
        globals()["lib"] = _loaded[1]
        return _loaded[1]
    raise AttributeError(name)


def strerror(code: int) -> str:
    return lib.imconv_strerror(int(code)).decode()


def check(code: int, what: str) -> None:
    if code != 0:
        raise ImconvError(code, what)
