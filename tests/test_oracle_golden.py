"""Pin the CPU oracle (oracle/) to vectors produced by the reference itself
(tests/golden/make_golden.py).  CPU only."""

import numpy as np
import pytest

from oracle import oracle as O
from conftest import conv_args, spec_from_vec


def test_oracle_int_conv_matches_reference_golden(golden):
    for i in range(int(golden["n_int"])):
        spec = spec_from_vec(golden[f"int{i}_spec"])
        x = golden[f"int{i}_x"].astype(np.int64)
        w = golden[f"int{i}_w"].astype(np.int64)
        y = O.conv2d_nhwc_i64(x, w, *conv_args(spec), threads=2)
        assert y.shape == (spec.n, spec.h_o, spec.w_o, spec.c_o)
        assert np.array_equal(y, golden[f"int{i}_y"].astype(np.int64)), i


def test_oracle_exact_f64_path_matches_int64(golden):
    for i in range(int(golden["n_int"])):
        spec = spec_from_vec(golden[f"int{i}_spec"])
        x = golden[f"int{i}_x"]
        w = golden[f"int{i}_w"]
        y = O.conv2d_nhwc_exact_f64(x, w, *conv_args(spec))
        assert np.array_equal(y, golden[f"int{i}_y"].astype(np.int64)), i


def test_oracle_float_conv_matches_reference_golden(golden):
    for i in range(int(golden["n_flt"])):
        spec = spec_from_vec(golden[f"flt{i}_spec"])
        y = O.conv2d_nhwc_taps(golden[f"flt{i}_x"], golden[f"flt{i}_w"], *conv_args(spec))
        assert y.dtype == np.float32
        np.testing.assert_allclose(y, golden[f"flt{i}_y"], rtol=1e-5, atol=1e-5)


def test_oracle_reference_routing(golden):
    spec = spec_from_vec(golden["int0_spec"])
    y = O.conv_reference(golden["int0_x"], golden["int0_w"], *conv_args(spec))
    assert y.dtype == np.int64
    assert np.array_equal(y, golden["int0_y"])


def test_oracle_gathers_and_im2col_match_reference(golden):
    for i in range(int(golden["n_gat"])):
        spec = spec_from_vec(golden[f"gat{i}_spec"])
        x = golden[f"gat{i}_x"]
        r, s = (int(v) for v in golden[f"gat{i}_rs"])
        g = O.tile_gather_nhwc(x, r, s, *conv_args(spec), spec.h_o, spec.w_o)
        assert np.array_equal(g, golden[f"gat{i}_g"])
        cf = O.im2col_nhwc(x, spec.h_f, spec.w_f, *conv_args(spec), True)
        cl = O.im2col_nhwc(x, spec.h_f, spec.w_f, *conv_args(spec), False)
        assert np.array_equal(cf, golden[f"gat{i}_cf"])
        assert np.array_equal(cl, golden[f"gat{i}_cl"])


def test_oracle_lru_matches_reference(golden):
    for i in range(int(golden["n_lru"])):
        got = O.lru_simulate(golden[f"lru{i}_keys"], int(golden[f"lru{i}_cap"]))
        assert list(got) == golden[f"lru{i}_hm"].tolist()


def test_oracle_cf_implicit_simulation_golden(golden):
    # simulate(..., CHANNEL_FIRST_IMPLICIT).ofmap == direct conv (simulator.py:286-293)
    for i in range(int(golden["n_sim"])):
        spec = spec_from_vec(golden[f"sim{i}_spec"])
        y = O.conv2d_nhwc_i64(golden[f"sim{i}_x"], golden[f"sim{i}_w"], *conv_args(spec))
        assert np.array_equal(y, golden[f"sim{i}_y"])


def test_oracle_vs_independent_loop_nest(rng):
    # the reference suite's brute-force oracle (tests/conftest.py:7-31)
    x = rng.integers(-4, 5, size=(2, 7, 7, 3)).astype(np.int64)
    f = rng.integers(-4, 5, size=(3, 3, 3, 4)).astype(np.int64)
    want = O.reference_conv_loops(x, f, 2, 7, 7, 3, 4, 3, 3, 2, 2, 1, 1, 1, 1)
    assert np.array_equal(O.conv2d_nhwc_i64(x, f, 2, 2, 1, 1, 1, 1), want)


@pytest.mark.parametrize("threads", [1, 3])
def test_oracle_threading_is_deterministic(rng, threads):
    x = rng.integers(-128, 128, size=(5, 9, 9, 16)).astype(np.int64)
    f = rng.integers(-128, 128, size=(3, 3, 16, 8)).astype(np.int64)
    a = O.conv2d_nhwc_i64(x, f, 1, 1, 1, 1, 1, 1, threads=threads)
    b = O.conv2d_nhwc_i64(x, f, 1, 1, 1, 1, 1, 1, threads=1)
    assert np.array_equal(a, b)


def test_paper_known_answers():
    # single MAC 3*2 = 6 (reference tests/test_core.py:28-31)
    assert O.conv2d_nhwc_i64(np.array([[[[3]]]]), np.array([[[[2]]]]), 1, 1, 0, 0, 1, 1).tolist() == [[[[6]]]]
    # all-ones 3x3 window = 9 (tests/test_core.py:34-40)
    y = O.conv2d_nhwc_i64(np.ones((1, 3, 3, 1), np.int64), np.ones((3, 3, 1, 1), np.int64), 1, 1, 0, 0, 1, 1)
    assert y.tolist() == [[[[9]]]]


# ---- the reference's own kernels compiled from its sources (oracle/_ref, oracle/build_ref.py) ----

def _ref_or_skip():
    from oracle import ref as R
    if not R.available():
        pytest.skip("oracle/_ref not built (python oracle/build_ref.py; needs /root/reference)")
    return R


def test_compiled_reference_matches_golden(golden):
    """The compiled reference reproduces its own recorded outputs: ints bit-exact through
    _native (int64), floats through _fallback."""
    R = _ref_or_skip()
    for i in range(int(golden["n_int"])):
        spec = spec_from_vec(golden[f"int{i}_spec"])
        y = R.conv2d_nhwc(golden[f"int{i}_x"], golden[f"int{i}_w"], *conv_args(spec))
        assert y.dtype == np.int64 and np.array_equal(y, golden[f"int{i}_y"].astype(np.int64)), i
    for i in range(int(golden["n_flt"])):
        spec = spec_from_vec(golden[f"flt{i}_spec"])
        y = R.conv2d_nhwc(golden[f"flt{i}_x"], golden[f"flt{i}_w"], *conv_args(spec))
        assert np.array_equal(y, golden[f"flt{i}_y"]), i


def test_restatement_matches_compiled_reference(rng):
    """oracle.conv2d_nhwc_taps (the numpy restatement) against the compiled _fallback on the
    bench's kind of operands (strided, padded, dilated, fp32): identical tap order, so equal
    up to BLAS blocking differences."""
    R = _ref_or_skip()
    for args, xs, ws in [((2, 2, 3, 3, 1, 1), (2, 30, 30, 8), (7, 7, 8, 16)),
                         ((1, 1, 2, 2, 2, 2), (2, 12, 12, 32), (3, 3, 32, 24)),
                         ((2, 1, 0, 1, 1, 2), (3, 9, 11, 16), (1, 3, 16, 8))]:
        x = rng.standard_normal(xs).astype(np.float32)
        w = rng.standard_normal(ws).astype(np.float32)
        np.testing.assert_allclose(O.conv2d_nhwc_taps(x, w, *args), R.conv2d_nhwc(x, w, *args),
                                   rtol=1e-5, atol=1e-5)
        xi = rng.integers(-128, 128, size=xs).astype(np.int64)
        wi = rng.integers(-128, 128, size=ws).astype(np.int64)
        assert np.array_equal(O.conv2d_nhwc_i64(xi, wi, *args), R.conv2d_nhwc(xi, wi, *args))
