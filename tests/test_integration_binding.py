"""The reference-side plug-in (integration/sasim_b200.py, what a maintainer adds as
sasim/_kernels/_b200.py) exercised with the reference's own kernel-level test patterns:

  * /root/reference/pkg/tests/test_kernels.py:20-60 -- conv2d / tile_gather / im2col / lru
    parity (there: _native vs _fallback; here: the plug-in vs the pinned oracle), with the
    same shapes, argument tuples and value ranges;
  * /root/reference/pkg/tests/test_core.py:28-67 -- direct_conv known answers (single MAC
    3*2 = 6, an all-ones 3x3 window sums to 9, the brute-force loop nest of conftest.py:7-31,
    a 1x1 conv equals the GEMM);
  * the reference's integer goldens (tests/golden, generated from the reference itself).

The plug-in imports nothing from the package (ctypes over include/imconv.h only).
"""

import importlib.util
import os

import numpy as np
import pytest

from conftest import conv_args, spec_from_vec

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def b200():
    spec = importlib.util.spec_from_file_location("sasim_b200", os.path.join(ROOT, "integration", "sasim_b200.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def _loop_nest(x, f, sh, sw, ph, pw, dh, dw):
    """Brute-force convolution restated from the reference's independent test oracle
    (tests/conftest.py:7-31): explicit bounds checks, no shared code with any kernel."""
    n, h, w, c = x.shape
    r, s, _, k = f.shape
    p = (h + 2 * ph - dh * (r - 1) - 1) // sh + 1
    q = (w + 2 * pw - dw * (s - 1) - 1) // sw + 1
    out = np.zeros((n, p, q, k), dtype=np.result_type(x, f))
    for b in range(n):
        for ho in range(p):
            for wo in range(q):
                for hf in range(r):
                    hi = ho * sh + hf * dh - ph
                    if not 0 <= hi < h:
                        continue
                    for wf in range(s):
                        wi = wo * sw + wf * dw - pw
                        if 0 <= wi < w:
                            out[b, ho, wo] += x[b, hi, wi] @ f[hf, wf]
    return out


def test_plugin_lru_host_code(b200):
    """test_kernels.py:57-66 pattern (host code, no GPU): the LRU replay behind reuse_traffic."""
    keys = np.array([1, 2, 3, 1, 2, 3], dtype=np.int64)
    assert b200.lru_simulate(keys, 3) == (3, 3)
    assert b200.lru_simulate(keys, 2) == (0, 6)
    assert b200.lru_simulate(keys, 0) == (0, 6)
    from oracle import oracle as O
    rng = np.random.default_rng(7)
    k = rng.integers(0, 64, size=5000).astype(np.int64)
    for cap in (0, 1, 7, 64, 200):
        assert b200.lru_simulate(k, cap) == O.lru_simulate(k, cap)


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", [np.int64, np.float32, np.float64])
def test_plugin_conv2d_parity(b200, dtype):
    """test_kernels.py:20-30: x (2,9,8,3) and w (3,3,3,5) integers in [-4, 4] of each kernel
    dtype, (sh, sw, ph, pw, dh, dw) = (2, 1, 1, 2, 1, 2); exact for every dtype (integer values
    are exact in int8 / bf16 and their fp32 sums are exact)."""
    rng = np.random.default_rng(20)
    x = rng.integers(-4, 5, size=(2, 9, 8, 3)).astype(dtype)
    w = rng.integers(-4, 5, size=(3, 3, 3, 5)).astype(dtype)
    got = b200.conv2d_nhwc(x, w, 2, 1, 1, 2, 1, 2)
    want = _loop_nest(x.astype(np.int64), w.astype(np.int64), 2, 1, 1, 2, 1, 2)
    assert got.dtype == (np.int64 if dtype is np.int64 else dtype)
    assert got.shape == want.shape
    assert np.array_equal(got.astype(np.int64), want)


@pytest.mark.gpu
def test_plugin_tile_gather_parity(b200):
    """test_kernels.py:33-41: every tap of a 3x3 stride-2 gather of a (2,7,7,4) int64 tensor."""
    from oracle import oracle as O
    rng = np.random.default_rng(33)
    x = rng.integers(-9, 9, size=(2, 7, 7, 4)).astype(np.int64)
    for r in range(3):
        for s in range(3):
            assert np.array_equal(b200.tile_gather_nhwc(x, r, s, 2, 2, 1, 1, 1, 1, 4, 4),
                                  O.tile_gather_nhwc(x, r, s, 2, 2, 1, 1, 1, 1, 4, 4))


@pytest.mark.gpu
@pytest.mark.parametrize("channel_first", [True, False])
def test_plugin_im2col_parity(b200, channel_first):
    """test_kernels.py:44-50: (2,8,6,3) int64, 3x2 filter, (1,2,1,0,2,1), both column orders."""
    from oracle import oracle as O
    rng = np.random.default_rng(44)
    x = rng.integers(-9, 9, size=(2, 8, 6, 3)).astype(np.int64)
    assert np.array_equal(b200.im2col_nhwc(x, 3, 2, 1, 2, 1, 0, 2, 1, channel_first),
                          O.im2col_nhwc(x, 3, 2, 1, 2, 1, 0, 2, 1, channel_first))


@pytest.mark.gpu
def test_plugin_known_answers(b200):
    """test_core.py:28-40 / :61-67: a single MAC, an all-ones window, 1x1 conv == GEMM."""
    assert b200.conv2d_nhwc(np.array([[[[3.0]]]]), np.array([[[[2.0]]]]), 1, 1, 0, 0, 1, 1).tolist() == [[[[6.0]]]]
    ones = b200.conv2d_nhwc(np.ones((1, 3, 3, 1)), np.ones((3, 3, 1, 1)), 1, 1, 0, 0, 1, 1)
    assert ones.shape == (1, 1, 1, 1) and ones.item() == 9.0
    rng = np.random.default_rng(61)
    x = rng.integers(-4, 5, size=(1, 5, 5, 6)).astype(np.int64)
    f = rng.integers(-4, 5, size=(1, 1, 6, 4)).astype(np.int64)
    conv = b200.conv2d_nhwc(x, f, 1, 1, 0, 0, 1, 1).reshape(25, 4)
    assert np.array_equal(conv, x.reshape(25, 6) @ f.reshape(6, 4))


@pytest.mark.gpu
def test_plugin_loop_nest_and_goldens(b200, golden):
    """test_core.py:43-58 (strided padded spec vs the loop nest) and the reference's own
    integer goldens (generated by importing the reference, tests/golden/make_golden.py)."""
    rng = np.random.default_rng(43)
    x = rng.integers(-4, 5, size=(2, 7, 7, 3)).astype(np.int64)
    f = rng.integers(-4, 5, size=(3, 3, 3, 4)).astype(np.int64)
    assert np.array_equal(b200.conv2d_nhwc(x, f, 2, 2, 1, 1, 1, 1), _loop_nest(x, f, 2, 2, 1, 1, 1, 1))
    for i in range(int(golden["n_int"])):
        spec = spec_from_vec(golden[f"int{i}_spec"])
        xi, wi = golden[f"int{i}_x"].astype(np.int64), golden[f"int{i}_w"].astype(np.int64)
        assert np.array_equal(b200.conv2d_nhwc(xi, wi, *conv_args(spec)), golden[f"int{i}_y"]), i


@pytest.mark.gpu
def test_plugin_rejects_out_of_range_integers(b200):
    """No CPU path: int64 values outside int8 are refused (the reference keeps _native for them)."""
    with pytest.raises(ValueError):
        b200.conv2d_nhwc(np.full((1, 3, 3, 1), 1000), np.ones((1, 1, 1, 1), dtype=np.int64), 1, 1, 0, 0, 1, 1)
