"""C-ABI boundary checks that need no GPU: the library loads, exports every
symbol include/imconv.h declares, and its host-only entry points behave."""

import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "imconv.h")


def _declared():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"IMCONV_API\s+[\w\s\*]*?\b(imconv_\w+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_2110_03901_b200 import _lib
    declared = _declared()
    assert len(declared) >= 12
    lib = ctypes.CDLL(_lib.LIB_PATH)
    for name in declared:
        assert hasattr(lib, name), name
    assert sorted(_lib.EXPORTED) == declared


def test_instrumented_build_exports_the_same_symbols():
    path = os.path.join(ROOT, "paper_2110_03901_b200", "libimconv_instr.so")
    if not os.path.exists(path):
        pytest.skip("instrumented library not built")
    lib = ctypes.CDLL(path)
    for name in _declared():
        assert hasattr(lib, name), name


def test_abi_version_and_strerror():
    import re
    from paper_2110_03901_b200 import _lib
    header = open(os.path.join(ROOT, "include", "imconv.h")).read()
    assert _lib.lib.imconv_abi_version() == int(re.search(r"#define IMCONV_ABI_VERSION (\d+)", header).group(1))
    assert "16 bytes" in _lib.strerror(-4)
    assert _lib.strerror(0) == "ok"
    assert _lib.strerror(-99) == "unknown error"


def test_out_extent_matches_reference_formula():
    # core.py:89-95 (h_o = (h + 2p - d(f-1) - 1)//s + 1); 224/7/s2/p3 -> 112
    from paper_2110_03901_b200 import _lib
    f = _lib.lib.imconv_out_extent
    assert f(224, 7, 2, 3, 1) == 112
    assert f(5, 3, 2, 0, 1) == 2
    assert f(64, 3, 1, 2, 2) == 64
    assert f(2, 3, 1, 0, 1) == 0          # effective filter larger than the padded input
    assert f(4, 1, 0, 0, 1) == 0          # invalid stride


def test_conv_argument_validation_without_gpu():
    from paper_2110_03901_b200 import _lib
    a = _lib.ImconvArgs()
    assert _lib.lib.imconv_conv2d_nhwc(None, None) == -1
    assert _lib.lib.imconv_conv2d_nhwc(ctypes.byref(a), None) == -1  # null pointers
    buf = (ctypes.c_uint8 * 64)()
    a.x = a.w = a.y = ctypes.addressof(buf)
    a.n = a.h = a.w_ = 1
    a.c, a.k, a.r, a.s = 8, 8, 1, 1
    a.stride_h = a.stride_w = a.dil_h = a.dil_w = 1
    a.in_dtype, a.out_dtype = _lib.BF16, _lib.I32
    assert _lib.lib.imconv_conv2d_nhwc(ctypes.byref(a), None) == -2  # dtype combination
    a.out_dtype = _lib.BF16
    a.c = 3
    assert _lib.lib.imconv_conv2d_nhwc(ctypes.byref(a), None) == -4  # channel alignment
    a.c = 8
    a.stride_h = 9
    assert _lib.lib.imconv_conv2d_nhwc(ctypes.byref(a), None) == -7  # TMA traversal stride limit


def test_lru_simulate_matches_reference_golden(golden):
    from paper_2110_03901_b200._kernels import lru_simulate
    for i in range(int(golden["n_lru"])):
        got = lru_simulate(golden[f"lru{i}_keys"], int(golden[f"lru{i}_cap"]))
        assert list(got) == golden[f"lru{i}_hm"].tolist(), i


def test_lru_basics():
    # reference tests/test_kernels.py:62-68
    from paper_2110_03901_b200._kernels import lru_simulate
    keys = np.array([1, 2, 3, 1, 2, 3], dtype=np.int64)
    assert lru_simulate(keys, 3) == (3, 3)
    assert lru_simulate(keys, 2) == (0, 6)
    assert lru_simulate(keys, 0) == (0, 6)
    assert lru_simulate(np.empty(0, np.int64), 4) == (0, 0)


def test_compute_entry_points_fail_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2110_03901_b200._kernels import conv2d_nhwc
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        conv2d_nhwc(np.ones((1, 4, 4, 8)), np.ones((1, 1, 8, 8)), 1, 1, 0, 0, 1, 1)
