"""ctypes binding of the C ABI in include/imconv.h (libimconv.so, in-tree).

There is no fallback: if the shared object is missing the import fails
loudly, and every compute call raises when no CUDA device is present.
"""

from __future__ import annotations

import ctypes
import os

_PKG = os.path.dirname(os.path.abspath(__file__))
# IMCONV_INSTRUMENTED=1 (tools/run_layer.py --waits) loads the same sources built
# with per-role wait counters; it is not a different backend.
LIB_PATH = os.path.join(_PKG, "libimconv_instr.so" if os.environ.get("IMCONV_INSTRUMENTED") == "1"
                        else "libimconv.so")

# element-type codes, include/imconv.h
BF16, F16, I8, F32, I32 = 0, 1, 2, 3, 4
ORDER_REUSE_AWARE, ORDER_FILTER_MAJOR = 0, 1
FLAG_SINGLE_CTA, FLAG_CTA_PAIR, FLAG_KSUB1, FLAG_MT1, FLAG_GATHER16, FLAG_NO_HALO = 1, 2, 4, 8, 16, 32
FLAG_CHANNEL_LAST = 64
FLAG_STATIC_FILTER = 128  # filter not written by kernels in flight: loads start before the PDL wait

# every symbol include/imconv.h declares (checked by tests/test_abi.py)
EXPORTED = (
    "imconv_conv2d_nhwc", "imconv_out_extent", "imconv_gemm", "imconv_tile_gather_nhwc",
    "imconv_im2col_nhwc", "imconv_pad_copy", "imconv_lru_simulate", "imconv_abi_version",
    "imconv_device_sm_count", "imconv_strerror", "imconv_launch_count", "imconv_reset_launch_count",
    "imconv_debug_set_buffer", "imconv_debug_set_flags", "imconv_predict_traffic",
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


class ImconvError(RuntimeError):
    def __init__(self, code: int, what: str):
        self.code = code
        super().__init__(f"{what}: {strerror(code)} (code {code})")


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
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
    return L


lib = _load()
# experiment switches (A/B measurements only): host-side debug flags of the C ABI
if os.environ.get("IMCONV_DEBUG_FLAGS"):
    lib.imconv_debug_set_flags(int(os.environ["IMCONV_DEBUG_FLAGS"], 0))


def strerror(code: int) -> str:
    return lib.imconv_strerror(int(code)).decode()


def check(code: int, what: str) -> None:
    if code != 0:
        raise ImconvError(code, what)
