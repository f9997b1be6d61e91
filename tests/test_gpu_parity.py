"""GPU parity: the sm_100a kernels (through the C ABI) vs the pinned oracle.

Bars (BASELINE.json north_star):
  * int8 -> int32: bit-exact;
  * bf16 integer-valued data with fp32 output: bit-exact (values in [-4, 4]
    are exact in bf16 and fp32 accumulation of the sums is exact);
  * bf16 N(0,1) data: max|y - ref| / max|ref| <= 1e-2 against the fp32
    oracle evaluated on the same bf16-rounded operands (REL_TOL below).
"""

import numpy as np
import pytest
import torch

from conftest import conv_args, spec_from_vec

pytestmark = pytest.mark.gpu

REL_TOL = 1e-2        # north_star bf16 tolerance (normalised max error)
REL_TOL_F32OUT = 1e-4  # fp32 output: only accumulation-order differences remain


def _P():
    import paper_2110_03901_b200 as P
    return P


def _norm_err(got, ref):
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    return float(np.abs(got - ref).max() / max(np.abs(ref).max(), 1e-30))


def test_int_golden_bit_exact(golden):
    P = _P()
    for i in range(int(golden["n_int"])):
        spec = spec_from_vec(golden[f"int{i}_spec"])
        x = golden[f"int{i}_x"].astype(np.int64)
        w = golden[f"int{i}_w"].astype(np.int64)
        y = P._kernels.conv2d_nhwc(x, w, *conv_args(spec))
        assert y.dtype == np.int64
        assert np.array_equal(y, golden[f"int{i}_y"].astype(np.int64)), (i, spec)


def test_int8_device_tensors_bit_exact(golden):
    P = _P()
    for i in range(int(golden["n_int"]) - 8, int(golden["n_int"])):
        spec = spec_from_vec(golden[f"int{i}_spec"])
        x = torch.from_numpy(golden[f"int{i}_x"]).cuda()
        w = torch.from_numpy(golden[f"int{i}_w"]).cuda()
        y = P._kernels.conv2d_nhwc(x, w, *conv_args(spec))
        assert y.dtype == torch.int32 and y.is_cuda
        assert np.array_equal(y.cpu().numpy(), golden[f"int{i}_y"]), i


def test_bf16_integer_valued_exact(golden):
    P = _P()
    for i in range(0, int(golden["n_int"]) - 8):
        spec = spec_from_vec(golden[f"int{i}_spec"])
        x = torch.from_numpy(golden[f"int{i}_x"].astype(np.float32)).cuda().to(torch.bfloat16)
        w = torch.from_numpy(golden[f"int{i}_w"].astype(np.float32)).cuda().to(torch.bfloat16)
        y = P._kernels.conv2d_nhwc(x, w, *conv_args(spec), out_dtype=torch.float32)
        assert np.array_equal(y.cpu().numpy(), golden[f"int{i}_y"].astype(np.float32)), (i, spec)


def test_float_golden_tolerance(golden):
    P = _P()
    from oracle import oracle as O
    for i in range(int(golden["n_flt"])):
        spec = spec_from_vec(golden[f"flt{i}_spec"])
        x, w = golden[f"flt{i}_x"], golden[f"flt{i}_w"]
        # reference output on the exact inputs vs kernel on bf16-rounded inputs
        y = P._kernels.conv2d_nhwc(x, w, *conv_args(spec))
        assert y.dtype == np.float32
        xb = torch.from_numpy(x).to(torch.bfloat16).float().numpy()
        wb = torch.from_numpy(w).to(torch.bfloat16).float().numpy()
        ref_b = O.conv2d_nhwc_taps(xb, wb, *conv_args(spec))
        assert _norm_err(y, ref_b) <= REL_TOL_F32OUT, i
        assert _norm_err(y, golden[f"flt{i}_y"]) <= 2 * REL_TOL, i


@pytest.mark.parametrize("tile_n", [64, 128, 256])
@pytest.mark.parametrize("flags", [0, 4, 8])  # 0: 2 m-tiles per CTA (N<=128), 4: KSUB=1, 8: MT=1 KSUB=2
def test_block_shape_and_grid_invariance(rng, tile_n, flags):
    P = _P()
    from oracle import oracle as O
    for c in (64, 192):  # 9 / 27 k-subtiles: odd counts leave a half-filled last stage
        x = rng.integers(-4, 5, size=(3, 13, 11, c)).astype(np.int64)
        w = rng.integers(-4, 5, size=(3, 3, c, 200)).astype(np.int64)
        want = O.conv2d_nhwc_i64(x, w, 1, 2, 1, 1, 2, 1)
        xb = torch.from_numpy(x).float().cuda().bfloat16()
        wb = torch.from_numpy(w).float().cuda().bfloat16()
        for ctas in (0, 1, 5):
            y = P._kernels.conv2d_nhwc(xb, wb, 1, 2, 1, 1, 2, 1, out_dtype=torch.float32, tile_n=tile_n,
                                       num_ctas=ctas, flags=flags)
            assert np.array_equal(y.cpu().numpy(), want.astype(np.float32)), (c, ctas)


# (N, H, W, R, S, K, pad_h, pad_w, dil_h, dil_w): halo-tile kernel shapes (stride 1,
# 128-byte pixels) -- partial last row tile, dilation, non-square filters, wide K,
# rows wider than half a tile (TPR = 1), and the ResNet stage-2 geometry.
HALO_SHAPES = [
    (2, 13, 11, 3, 3, 64, 1, 1, 1, 1),
    (3, 9, 17, 3, 3, 128, 2, 2, 2, 2),
    (2, 12, 10, 5, 5, 64, 2, 2, 1, 1),
    (2, 7, 21, 1, 3, 256, 0, 1, 1, 1),
    (1, 6, 100, 3, 3, 64, 1, 1, 1, 1),
    (2, 56, 56, 3, 3, 64, 1, 1, 1, 1),
    (2, 10, 9, 3, 3, 64, 0, 0, 1, 1),
]


@pytest.mark.parametrize("shape", HALO_SHAPES)
def test_halo_tiles_exact(rng, shape):
    """bf16 C = 64 (and int8 C = 128) stride-1 layers run on conv_halo_kernel:
    bit-exact against the oracle and identical to the per-tap generic kernel."""
    P = _P()
    from oracle import oracle as O
    n, h, w_, r, s, k, ph, pw, dh, dw = shape
    args = (1, 1, ph, pw, dh, dw)
    x = rng.integers(-4, 5, size=(n, h, w_, 64)).astype(np.int64)
    w = rng.integers(-4, 5, size=(r, s, 64, k)).astype(np.int64)
    want = O.conv2d_nhwc_i64(x, w, *args)
    xb = torch.from_numpy(x).float().cuda().bfloat16()
    wb = torch.from_numpy(w).float().cuda().bfloat16()
    launches0 = P._lib.lib.imconv_launch_count()
    y = P._kernels.conv2d_nhwc(xb, wb, *args, out_dtype=torch.float32)
    assert P._lib.lib.imconv_launch_count() == launches0 + 1
    assert np.array_equal(y.cpu().numpy(), want.astype(np.float32)), shape
    y_generic = P._kernels.conv2d_nhwc(xb, wb, *args, out_dtype=torch.float32, flags=P._lib.FLAG_NO_HALO)
    assert torch.equal(y, y_generic)
    # bf16 output (16-bit staging layout) vs the fp32 result rounded once
    yb = P._kernels.conv2d_nhwc(xb, wb, *args)
    assert torch.equal(yb, y.bfloat16())
    if k >= 128:  # int8 needs C = 128 for a 128-byte pixel
        xi = rng.integers(-128, 128, size=(n, h, w_, 128)).astype(np.int8)
        wi = rng.integers(-128, 128, size=(r, s, 128, k)).astype(np.int8)
        yi = P._kernels.conv2d_nhwc(torch.from_numpy(xi).cuda(), torch.from_numpy(wi).cuda(), *args)
        assert np.array_equal(yi.cpu().numpy(), O.conv2d_nhwc_exact_f64(xi, wi, *args)), shape


@pytest.mark.parametrize("shape", [(1, 7, 7, 512, 512), (3, 9, 5, 512, 320), (2, 14, 14, 512, 256)])
def test_split_k_tail_exact(rng, shape):
    """Long k-loops with a short last wave run split-K (S k-ranges per tail tile, partials
    summed by the last arriving split): exact, repeatable across launches (generation-tagged
    counters), and equal to the unsplit kernel."""
    P = _P()
    from oracle import oracle as O
    n, h, w_, c, k = shape
    args = (1, 1, 1, 1, 1, 1)
    x = rng.integers(-2, 3, size=(n, h, w_, c)).astype(np.int64)
    w = rng.integers(-2, 3, size=(3, 3, c, k)).astype(np.int64)
    want = O.conv2d_nhwc_exact_f64(x, w, *args).astype(np.int64)
    xb = torch.from_numpy(x).float().cuda().bfloat16()
    wb = torch.from_numpy(w).float().cuda().bfloat16()
    ys = [P._kernels.conv2d_nhwc(xb, wb, *args, out_dtype=torch.float32) for _ in range(3)]
    for y in ys:
        assert np.array_equal(y.cpu().numpy(), want.astype(np.float32)), shape
    P._lib.lib.imconv_debug_set_flags(1 << 19)  # split-K off
    try:
        y_ref = P._kernels.conv2d_nhwc(xb, wb, *args, out_dtype=torch.float32)
    finally:
        P._lib.lib.imconv_debug_set_flags(0)
    assert torch.equal(ys[0], y_ref)
    xi = torch.from_numpy(x).to(torch.int8).cuda()
    wi = torch.from_numpy(w).to(torch.int8).cuda()
    yi = P._kernels.conv2d_nhwc(xi, wi, *args)
    assert np.array_equal(yi.cpu().numpy(), want), shape


@pytest.mark.parametrize("shape", [
    # (N, H, W, C, K, R, stride): blocks below one wave, long k-loops -> every tile split
    (4, 7, 7, 2048, 512, 1, 1),     # ResNet s5 1x1a at a small shard: BN = 256, S = 5
    (2, 14, 14, 1024, 128, 1, 1),   # BN = 128, two m-tiles per CTA (4 output blocks per tile)
    (3, 14, 14, 1024, 320, 1, 2),   # strided 1x1, ragged n-tile (K = 320: clipped blocks)
    (2, 7, 7, 512, 512, 3, 1),      # 3x3 s5 shape at N = 2
    (1, 9, 9, 256, 64, 3, 1),       # BN = 64
])
def test_split_k_sub_wave_exact(rng, shape):
    """Split-K below one wave: each split writes its partials, waits for its peers and
    reduces the output blocks it owns.  Exact on integer-valued bf16 (fp32 and bf16 out:
    the bf16 result is the fp32 sum rounded once), on int8, and equal to the unsplit
    kernel."""
    P = _P()
    from oracle import oracle as O
    n, h, w_, c, k, r, st = shape
    pad = r // 2
    args = (st, st, pad, pad, 1, 1)
    x = rng.integers(-2, 3, size=(n, h, w_, c)).astype(np.int64)
    w = rng.integers(-2, 3, size=(r, r, c, k)).astype(np.int64)
    want = O.conv2d_nhwc_exact_f64(x, w, *args).astype(np.int64)
    xb = torch.from_numpy(x).float().cuda().bfloat16()
    wb = torch.from_numpy(w).float().cuda().bfloat16()
    y = P._kernels.conv2d_nhwc(xb, wb, *args, out_dtype=torch.float32)
    assert np.array_equal(y.cpu().numpy(), want.astype(np.float32)), shape
    yb = P._kernels.conv2d_nhwc(xb, wb, *args)
    assert torch.equal(yb, y.bfloat16()), shape
    P._lib.lib.imconv_debug_set_flags(1 << 19)  # split-K off
    try:
        y_ref = P._kernels.conv2d_nhwc(xb, wb, *args, out_dtype=torch.float32)
    finally:
        P._lib.lib.imconv_debug_set_flags(0)
    assert torch.equal(y, y_ref)
    if c % 128 == 0 and k % 128 == 0:
        xi = torch.from_numpy(x).to(torch.int8).cuda()
        wi = torch.from_numpy(w).to(torch.int8).cuda()
        yi = P._kernels.conv2d_nhwc(xi, wi, *args)
        assert np.array_equal(yi.cpu().numpy(), want), shape
    # N(0,1) operands: fp32 oracle within the stated tolerance
    xf = rng.standard_normal((n, h, w_, c)).astype(np.float32)
    wf = (rng.standard_normal((r, r, c, k)) * (2.0 / (c * r * r)) ** 0.5).astype(np.float32)
    xq = torch.from_numpy(xf).bfloat16()
    wq = torch.from_numpy(wf).bfloat16()
    yq = P._kernels.conv2d_nhwc(xq.cuda(), wq.cuda(), *args, out_dtype=torch.float32).cpu().numpy()
    ref = O.conv2d_nhwc_taps(xq.float().numpy(), wq.float().numpy(), *args)
    assert np.abs(yq - ref).max() / max(np.abs(ref).max(), 1e-6) <= 1e-2


@pytest.mark.parametrize("case", [
    # (N, H, W, C, K, R, S, sh, sw, ph, pw, dh, dw)
    (2, 13, 11, 16, 24, 3, 3, 1, 1, 1, 1, 1, 1),
    (1, 17, 15, 64, 64, 3, 3, 2, 3, 1, 1, 1, 1),
    (2, 12, 10, 24, 200, 3, 2, 1, 2, 2, 1, 2, 1),
    (1, 9, 9, 40, 128, 5, 5, 4, 4, 2, 2, 1, 1),   # 1000-element reduction: partial last k-subtile
    (3, 7, 6, 128, 256, 1, 1, 1, 1, 0, 0, 1, 1),
])
def test_channel_last_baseline_exact(rng, case):
    """The channel-last baseline kernel (k = (c, r, s), thread-gathered A) is exact and
    agrees with the channel-first kernel (and with Method.CHANNEL_LAST_IMPLICIT)."""
    P = _P()
    from oracle import oracle as O
    n, h, w_, c, k, r, s_, sh, sw, ph, pw, dh, dw = case
    args = (sh, sw, ph, pw, dh, dw)
    x = rng.integers(-4, 5, size=(n, h, w_, c)).astype(np.int64)
    w = rng.integers(-4, 5, size=(r, s_, c, k)).astype(np.int64)
    want = O.conv2d_nhwc_i64(x, w, *args)
    xb = torch.from_numpy(x).float().cuda().bfloat16()
    wb = torch.from_numpy(w).float().cuda().bfloat16()
    y_cl = P._kernels.conv2d_nhwc(xb, wb, *args, out_dtype=torch.float32, flags=P._lib.FLAG_CHANNEL_LAST)
    assert np.array_equal(y_cl.cpu().numpy(), want.astype(np.float32)), case
    y_cf = P._kernels.conv2d_nhwc(xb, wb, *args, out_dtype=torch.float32)
    assert torch.equal(y_cl, y_cf)
    from paper_2110_03901_b200 import ConvSpec, Layout, Method, Tensor, functional_ofmap
    spec = ConvSpec(n=n, c_i=c, h_i=h, w_i=w_, c_o=k, h_f=r, w_f=s_, stride_h=sh, stride_w=sw, pad_h=ph, pad_w=pw,
                    dilation_h=dh, dilation_w=dw)
    yf = functional_ofmap(spec, Method.CHANNEL_LAST_IMPLICIT, Tensor.from_array(x.astype(np.float32), Layout.NHWC),
                          Tensor.from_array(w.astype(np.float32), Layout.HWCN))
    assert np.array_equal(np.asarray(yf.view()), want.astype(np.float32))


def test_host_tensor_path_pipelined(rng):
    """CPU torch tensors in -> pipelined upload / conv / download (chunked over N):
    identical to the device path, exact for integers, and ordered on the caller's stream."""
    P = _P()
    from oracle import oracle as O
    x = rng.integers(-4, 5, size=(7, 40, 36, 64)).astype(np.int64)  # 7 images -> uneven chunks
    w = rng.integers(-4, 5, size=(3, 3, 64, 96)).astype(np.int64)
    args = (1, 1, 1, 1, 1, 1)
    want = O.conv2d_nhwc_i64(x, w, *args)
    hx = torch.from_numpy(x).float().bfloat16().pin_memory()
    hw = torch.from_numpy(w).float().bfloat16().pin_memory()
    y_dev = P._kernels.conv2d_nhwc(hx.cuda(), hw.cuda(), *args, out_dtype=torch.float32)
    y_host = P._kernels.conv2d_nhwc(hx, hw, *args, out_dtype=torch.float32)  # allocates + syncs
    assert not y_host.is_cuda and torch.equal(y_host, y_dev.cpu())
    assert np.array_equal(y_host.numpy(), want.astype(np.float32))
    out = torch.empty(y_host.shape, dtype=torch.bfloat16, pin_memory=True)
    r = P._kernels.conv2d_nhwc(hx, hw, *args, out=out)  # asynchronous into `out`
    assert r is out
    torch.cuda.current_stream().synchronize()
    assert torch.equal(out, y_dev.bfloat16().cpu())
    yi = P._kernels.conv2d_nhwc(torch.from_numpy(x), torch.from_numpy(w), *args)  # int64 host -> int8 path
    assert yi.dtype == torch.int32 and np.array_equal(yi.numpy(), want)
    with pytest.raises(ValueError):
        P._kernels.conv2d_nhwc(hx, hw, *args, out=torch.empty(3))


@pytest.mark.parametrize("order", ["reuse_aware", "filter_major"])
def test_subtile_orders_identical(rng, order):
    P = _P()
    x = rng.integers(-128, 128, size=(2, 20, 20, 256)).astype(np.int8)
    w = rng.integers(-128, 128, size=(3, 3, 256, 128)).astype(np.int8)
    from oracle import oracle as O
    want = O.conv2d_nhwc_exact_f64(x, w, 2, 2, 1, 1, 1, 1)
    y = P._kernels.conv2d_nhwc(torch.from_numpy(x).cuda(), torch.from_numpy(w).cuda(), 2, 2, 1, 1, 1, 1, order=order)
    assert np.array_equal(y.cpu().numpy(), want)


@pytest.mark.parametrize("case", [
    # (N, H, W, K, R, S, sh, sw, ph, pw): 16-byte pixels (C = 8), row-band kernel
    (2, 40, 38, 64, 7, 7, 2, 2, 3, 3),   # ResNet stem shape: rows paired with filter rows 2 apart
    (1, 224, 224, 64, 7, 7, 2, 2, 3, 3),  # the stem itself: compile-time issue schedule (STEM instantiation)
    (1, 21, 30, 64, 3, 3, 1, 1, 1, 1),   # stride 1: filter rows 1 apart
    (3, 17, 19, 48, 5, 3, 3, 2, 2, 1),   # stride 3 rows, ragged P (P % 4 != 0), K < 64
])
def test_rowband_row_pairs_exact(rng, case):
    """Row-band kernel: adjacent output rows share N = 128 MMAs (B = two filter rows sh apart,
    LBO-addressed) -- exact against the oracle and equal to the unpaired kernel."""
    P = _P()
    from oracle import oracle as O
    n, h, w_, k, r, s, sh, sw, ph, pw = case
    args = (sh, sw, ph, pw, 1, 1)
    x = rng.integers(-4, 5, size=(n, h, w_, 8)).astype(np.int64)
    w = rng.integers(-4, 5, size=(r, s, 8, k)).astype(np.int64)
    want = O.conv2d_nhwc_i64(x, w, *args).astype(np.float32)
    xb = torch.from_numpy(x).float().cuda().bfloat16()
    wb = torch.from_numpy(w).float().cuda().bfloat16()
    y = P._kernels.conv2d_nhwc(xb, wb, *args, out_dtype=torch.float32)
    assert np.array_equal(y.cpu().numpy(), want), case
    P._lib.lib.imconv_debug_set_flags(1 << 22)  # row pairing off
    try:
        y_ref = P._kernels.conv2d_nhwc(xb, wb, *args, out_dtype=torch.float32)
    finally:
        P._lib.lib.imconv_debug_set_flags(0)
    assert torch.equal(y, y_ref)


@pytest.mark.parametrize("flags", [0, 8, 16])  # 16-B pixels -> 0: row-band, 8: TMA taps (MT1), 16: cp.async gathers
def test_small_channel_tap_packing(rng, flags):
    """C*elem < 128 B: several taps share one pipeline stage (16/32/64 B rows)."""
    P = _P()
    from oracle import oracle as O
    for c in (3, 8, 16, 24, 32, 40):
        x = rng.integers(-4, 5, size=(2, 15, 17, c)).astype(np.int64)
        w = rng.integers(-4, 5, size=(7, 5, c, 24)).astype(np.int64)
        for args in ((2, 1, 3, 2, 1, 1), (1, 2, 2, 1, 2, 1)):
            want = O.conv2d_nhwc_i64(x, w, *args)
            xb = torch.from_numpy(x).float().cuda().bfloat16()
            wb = torch.from_numpy(w).float().cuda().bfloat16()
            y = P._kernels.conv2d_nhwc(xb, wb, *args, out_dtype=torch.float32, flags=flags)
            assert np.array_equal(y.cpu().numpy(), want.astype(np.float32)), (c, args)
            yi = P._kernels.conv2d_nhwc(x, w, *args, flags=flags)
            assert np.array_equal(yi, want), (c, args)


def test_gather_and_im2col_match_golden(golden):
    P = _P()
    for i in range(int(golden["n_gat"])):
        spec = spec_from_vec(golden[f"gat{i}_spec"])
        x = golden[f"gat{i}_x"]
        r, s = (int(v) for v in golden[f"gat{i}_rs"])
        g = P._kernels.tile_gather_nhwc(x, r, s, *conv_args(spec), spec.h_o, spec.w_o)
        assert np.array_equal(g, golden[f"gat{i}_g"])
        cf = P._kernels.im2col_nhwc(x, spec.h_f, spec.w_f, *conv_args(spec), True)
        cl = P._kernels.im2col_nhwc(x, spec.h_f, spec.w_f, *conv_args(spec), False)
        assert np.array_equal(cf, golden[f"gat{i}_cf"]), i
        assert np.array_equal(cl, golden[f"gat{i}_cl"]), i


def test_im2col_vector_path_bf16(rng):
    P = _P()
    from oracle import oracle as O
    x = torch.randn(3, 14, 14, 64).bfloat16()
    got = P._kernels.im2col_nhwc(x.cuda(), 3, 3, 2, 2, 1, 1, 1, 1, True).cpu()
    want = O.im2col_nhwc(x.view(torch.int16).numpy(), 3, 3, 2, 2, 1, 1, 1, 1, True)
    assert np.array_equal(got.view(torch.int16).numpy(), want)
    # 1x1 filters (single tap, full lowering) and a 1xS filter through the vector path
    for hf, wf, st, pd in ((1, 1, 1, 0), (1, 1, 2, 0), (1, 3, 1, 1), (7, 7, 2, 3)):
        got = P._kernels.im2col_nhwc(x.cuda(), hf, wf, st, st, pd, pd, 1, 1, True).cpu()
        want = O.im2col_nhwc(x.view(torch.int16).numpy(), hf, wf, st, st, pd, pd, 1, 1, True)
        assert np.array_equal(got.view(torch.int16).numpy(), want), (hf, wf, st, pd)
    assert torch.equal(P._kernels.im2col_nhwc(x.cuda(), 1, 1, 1, 1, 0, 0, 1, 1, True).cpu(), x.reshape(-1, 64))


def test_explicit_path_equals_implicit(golden):
    P = _P()
    from paper_2110_03901_b200 import Layout, Method, Tensor
    for i in range(int(golden["n_sim"])):
        spec = spec_from_vec(golden[f"sim{i}_spec"])
        x = Tensor.from_array(golden[f"sim{i}_x"].astype(np.int64), Layout.NHWC)
        w = Tensor.from_array(golden[f"sim{i}_w"].astype(np.int64), Layout.HWCN)
        for m in P.ALL_METHODS:
            y = P.functional_ofmap(spec, m, x, w)
            assert np.array_equal(y.view(), golden[f"sim{i}_y"].astype(np.int64)), (i, m)


def test_gemm_matches_oracle(rng):
    P = _P()
    from paper_2110_03901_b200 import Layout, Tensor
    a = rng.integers(-6, 7, size=(300, 96)).astype(np.int64)
    b = rng.integers(-6, 7, size=(96, 40)).astype(np.int64)
    got = P.gemm(Tensor.from_array(a, Layout.ROW_MAJOR), Tensor.from_array(b, Layout.ROW_MAJOR))
    assert np.array_equal(got.view(), a @ b)


def test_direct_conv_api_and_shape_errors(rng):
    P = _P()
    from paper_2110_03901_b200 import ConvSpec, Layout, ShapeError, Tensor
    spec = ConvSpec.square(1, 1, 1, 1, 1)
    out = P.direct_conv(Tensor.from_array(np.array([[[[3.0]]]]), Layout.NHWC),
                        Tensor.from_array(np.array([[[[2.0]]]]), Layout.HWCN), spec)
    assert out.data.tolist() == [6.0]
    spec = ConvSpec.square(1, 1, 3, 1, 3)
    out = P.direct_conv(Tensor.from_array(np.ones((1, 3, 3, 1)), Layout.NHWC),
                        Tensor.from_array(np.ones((3, 3, 1, 1)), Layout.HWCN), spec)
    assert out.dims == (1, 1, 1, 1) and out.data.tolist() == [9.0]
    with pytest.raises(ShapeError):
        P.direct_conv(Tensor.from_array(np.zeros((1, 4, 4, 3)), Layout.NHWC),
                      Tensor.from_array(np.zeros((1, 1, 2, 1)), Layout.HWCN), ConvSpec.square(1, 2, 4, 1, 1))
    with pytest.raises(ValueError):
        P._kernels.conv2d_nhwc(np.full((1, 4, 4, 16), 300), np.ones((1, 1, 16, 8), np.int64), 1, 1, 0, 0, 1, 1)
    with pytest.raises(ValueError):
        P._kernels.conv2d_nhwc(np.ones((1, 4, 4, 3)), np.ones((1, 1, 2, 8)), 1, 1, 0, 0, 1, 1)


def test_nchw_input_relayout(rng):
    P = _P()
    from paper_2110_03901_b200 import ConvSpec, Layout, Tensor
    from oracle import oracle as O
    spec = ConvSpec.square(2, 8, 9, 16, 3, stride=2, pad=1)
    x = rng.integers(-4, 5, size=(2, 9, 9, 8)).astype(np.int64)
    w = rng.integers(-4, 5, size=(3, 3, 8, 16)).astype(np.int64)
    got = P.direct_conv(Tensor.from_array(x.transpose(0, 3, 1, 2), Layout.NCHW),
                        Tensor.from_array(w, Layout.HWCN), spec)
    assert np.array_equal(got.view(), O.conv2d_nhwc_i64(x, w, 2, 2, 1, 1, 1, 1))


def test_evaluate_plan_orders(rng):
    P = _P()
    from paper_2110_03901_b200 import ConvSpec, Layout, Tensor
    from paper_2110_03901_b200.blocksched import SubtileOrder, evaluate_plan, order_subtiles, partition
    from oracle import oracle as O
    spec = ConvSpec.square(2, 3, 8, 4, 3, stride=2, pad=1)
    x = rng.integers(-4, 5, size=(2, 8, 8, 3)).astype(np.int64)
    w = rng.integers(-4, 5, size=(3, 3, 3, 4)).astype(np.int64)
    want = O.conv2d_nhwc_i64(x, w, 2, 2, 1, 1, 1, 1)
    plan = partition(spec, 5, 3, 2)
    fm = order_subtiles(plan, SubtileOrder.FILTER_MAJOR)
    ra = order_subtiles(plan, SubtileOrder.REUSE_AWARE)
    sh = list(fm)
    rng.shuffle(sh)
    for order in (fm, ra, sh):
        out = evaluate_plan(plan, order, Tensor.from_array(x, Layout.NHWC), Tensor.from_array(w, Layout.HWCN))
        assert np.array_equal(out.view(), want)
    with pytest.raises(ValueError):
        evaluate_plan(plan, fm[:-1], Tensor.from_array(x, Layout.NHWC), Tensor.from_array(w, Layout.HWCN))


# ------------------------------------------------------------------ BASELINE configs

def _layer_check(layer, n=None, seed=0):
    P = _P()
    from oracle import oracle as O
    sp = layer.spec if n is None else layer.spec.with_batch(n)
    x, w = P.workloads.synthetic_operands(layer, seed=seed, n=n)
    xd, wd = x.cuda(), w.cuda()
    if layer.dtype == "int8":
        y = P._kernels.conv2d_nhwc(xd, wd, *conv_args(sp))
        want = O.conv2d_nhwc_exact_f64(x.numpy(), w.numpy(), *conv_args(sp))
        assert np.array_equal(y.cpu().numpy().astype(np.int64), want), layer.name
        return 0.0
    y = P._kernels.conv2d_nhwc(xd, wd, *conv_args(sp))  # bf16 out
    assert y.dtype == torch.bfloat16
    ref = O.conv2d_nhwc_taps(x.float().numpy(), w.float().numpy(), *conv_args(sp))
    err = _norm_err(y.float().cpu().numpy(), ref)
    assert err <= REL_TOL, (layer.name, err)
    y32 = P._kernels.conv2d_nhwc(xd, wd, *conv_args(sp), out_dtype=torch.float32)
    err32 = _norm_err(y32.cpu().numpy(), ref)
    assert err32 <= REL_TOL_F32OUT, (layer.name, err32)
    return err


@pytest.mark.parametrize("cfg", ["cfg1", "cfg2", "cfg3"])
def test_baseline_config_full_size(cfg):
    P = _P()
    for layer in P.workloads.baseline_configs()[cfg]:
        _layer_check(layer)


def test_baseline_cfg5_int8_full_size_bit_exact():
    P = _P()
    for layer in P.workloads.baseline_configs()["cfg5"]:
        _layer_check(layer)


def test_resnet50_layers_reduced_batch():
    P = _P()
    seen = set()
    for layer in P.workloads.resnet50_layers(2):
        key = layer.spec
        if key in seen:
            continue
        seen.add(key)
        _layer_check(layer)


@pytest.mark.parametrize("flags", [1, 2])
def test_cta_pair_parity(rng, flags):
    """CTA pairs (cta_group::2, B split across the pair) vs single CTAs:
    identical integer results, ragged 256-row blocks, odd grids."""
    P = _P()
    from oracle import oracle as O
    cases = [((3, 13, 11, 64), (3, 3, 64, 128), (1, 2, 1, 1, 2, 1)),
             ((2, 17, 9, 128), (1, 1, 128, 256), (1, 1, 0, 0, 1, 1)),
             ((1, 30, 30, 64), (3, 3, 64, 200), (2, 2, 1, 1, 1, 1)),
             ((2, 9, 9, 8), (5, 5, 8, 384), (1, 1, 2, 2, 1, 1))]
    for xs, ws, args in cases:
        x = rng.integers(-4, 5, size=xs).astype(np.int64)
        w = rng.integers(-4, 5, size=ws).astype(np.int64)
        want = O.conv2d_nhwc_i64(x, w, *args).astype(np.float32)
        xb = torch.from_numpy(x).float().cuda().bfloat16()
        wb = torch.from_numpy(w).float().cuda().bfloat16()
        for ctas in (0, 2, 6):
            y = P._kernels.conv2d_nhwc(xb, wb, *args, out_dtype=torch.float32, num_ctas=ctas, flags=flags,
                                       tile_n=256 if ws[3] > 128 else 0)
            assert np.array_equal(y.cpu().numpy(), want), (xs, ws, ctas)
    # int8 pairs (BN = 256)
    x = rng.integers(-128, 128, size=(2, 14, 14, 256)).astype(np.int8)
    w = rng.integers(-128, 128, size=(3, 3, 256, 256)).astype(np.int8)
    want = O.conv2d_nhwc_exact_f64(x, w, 1, 1, 1, 1, 1, 1)
    y = P._kernels.conv2d_nhwc(torch.from_numpy(x).cuda(), torch.from_numpy(w).cuda(), 1, 1, 1, 1, 1, 1,
                               flags=flags)
    assert np.array_equal(y.cpu().numpy(), want)


@pytest.mark.parametrize("shape", [
    # (N, H, C, K, R, stride): at least one wave of 128 x 256 blocks with a streamed filter
    # -> the planner picks CTA pairs on its own (ResNet s4 1x1a / s4 projection / s5 1x1b shapes)
    (100, 14, 1024, 256, 1, 1),
    (100, 28, 512, 1024, 1, 2),
    (60, 7, 512, 2048, 1, 1),
])
def test_auto_cta_pairs_exact(rng, shape):
    """Automatic CTA pairs: exact on integer-valued bf16 (fp32 out), equal to the single-CTA
    kernel, and within tolerance of the fp32 oracle on N(0,1) operands."""
    P = _P()
    from oracle import oracle as O
    n, h, c, k, r, st = shape
    args = (st, st, r // 2, r // 2, 1, 1)
    x = rng.integers(-2, 3, size=(n, h, h, c)).astype(np.int8)
    w = rng.integers(-2, 3, size=(r, r, c, k)).astype(np.int8)
    want = O.conv2d_nhwc_exact_f64(x, w, *args)
    xb = torch.from_numpy(x).cuda().float().bfloat16()
    wb = torch.from_numpy(w).cuda().float().bfloat16()
    y = P._kernels.conv2d_nhwc(xb, wb, *args, out_dtype=torch.float32)
    assert np.array_equal(y.cpu().numpy(), want.astype(np.float32)), shape
    y1 = P._kernels.conv2d_nhwc(xb, wb, *args, out_dtype=torch.float32, flags=P._lib.FLAG_SINGLE_CTA)
    assert torch.equal(y, y1)
    xf = torch.randn((n, h, h, c), dtype=torch.float32).bfloat16()
    wf = (torch.randn((r, r, c, k), dtype=torch.float32) * (2.0 / (c * r * r)) ** 0.5).bfloat16()
    yq = P._kernels.conv2d_nhwc(xf.cuda(), wf.cuda(), *args).float().cpu().numpy()
    ref = O.conv2d_nhwc_taps(xf.float().numpy(), wf.float().numpy(), *args)
    assert _norm_err(yq, ref) <= REL_TOL, shape


@pytest.mark.parametrize("case", [
    # (N, H, C, K, R, stride, pad): one shape per kernel path
    (2, 30, 8, 64, 7, 2, 3),        # row-band (16-byte pixels), row pairs
    (2, 20, 64, 64, 3, 1, 1),       # halo tiles (128-byte pixels, stride 1)
    (2, 21, 128, 200, 3, 2, 1),     # generic TMA-im2col kernel, ragged n-tile
    (2, 7, 512, 512, 3, 1, 1),      # split-K below one wave
    (100, 14, 1024, 256, 1, 1, 0),  # automatic CTA pairs
])
def test_fp16_paths_exact(rng, case):
    """fp16 inputs on every kernel path: integer-valued data is exact with fp32 output, and
    fp16 output equals the fp32 result rounded once."""
    P = _P()
    from oracle import oracle as O
    n, h, c, k, r, st, pad = case
    args = (st, st, pad, pad, 1, 1)
    x = rng.integers(-2, 3, size=(n, h, h, c)).astype(np.int8)
    w = rng.integers(-2, 3, size=(r, r, c, k)).astype(np.int8)
    want = O.conv2d_nhwc_exact_f64(x, w, *args).astype(np.float32)
    xh = torch.from_numpy(x).cuda().half()
    wh = torch.from_numpy(w).cuda().half()
    y = P._kernels.conv2d_nhwc(xh, wh, *args, out_dtype=torch.float32)
    assert np.array_equal(y.cpu().numpy(), want), case
    yh = P._kernels.conv2d_nhwc(xh, wh, *args)
    assert yh.dtype == torch.float16 and torch.equal(yh, y.half()), case


@pytest.mark.parametrize("case", [
    # (N, H, W, C, K, R, S, pad, dil): stride-1 layers with 16-bit pixels of several 128-byte
    # chunks and K <= 128 -> halo tiles with a streamed filter
    (2, 28, 28, 128, 128, 3, 3, 1, 1),   # ResNet s3 3x3
    (3, 17, 13, 256, 64, 3, 3, 1, 1),    # ragged last block, K = 64
    (2, 9, 11, 192, 128, 5, 3, 2, 1),    # 3 chunks, non-square filter
    (2, 12, 12, 128, 128, 3, 3, 2, 2),   # dilation
])
def test_halo_stream_exact(rng, case):
    """Streamed-filter halo kernel: exact against the oracle, equal to the generic kernel, and
    its bf16 output is the fp32 result rounded once."""
    P = _P()
    from oracle import oracle as O
    n, h, w_, c, k, r, s, pad, dil = case
    args = (1, 1, pad, (s // 2) * dil, dil, dil)
    x = rng.integers(-2, 3, size=(n, h, w_, c)).astype(np.int8)
    w = rng.integers(-2, 3, size=(r, s, c, k)).astype(np.int8)
    want = O.conv2d_nhwc_exact_f64(x, w, *args).astype(np.float32)
    xb = torch.from_numpy(x).cuda().float().bfloat16()
    wb = torch.from_numpy(w).cuda().float().bfloat16()
    y = P._kernels.conv2d_nhwc(xb, wb, *args, out_dtype=torch.float32)
    assert np.array_equal(y.cpu().numpy(), want), case
    y_generic = P._kernels.conv2d_nhwc(xb, wb, *args, out_dtype=torch.float32, flags=P._lib.FLAG_NO_HALO)
    assert torch.equal(y, y_generic)
    assert torch.equal(P._kernels.conv2d_nhwc(xb, wb, *args), y.bfloat16())


@pytest.mark.parametrize("case", [
    # (N, H, C, K, pad, dil): at least one wave of blocks (>= 148), so CTA pairs run two blocks each
    (64, 28, 128, 128, 1, 1),    # ResNet s3 3x3 shard shape: 256 blocks
    (151, 14, 256, 128, 1, 1),   # 151 blocks: the last pair's second CTA has no block of its own
    (75, 20, 128, 128, 2, 2),    # dilation, 2 blocks per image
])
def test_halo_stream_pairs_exact(rng, case):
    """Streamed-filter halo tiles on CTA pairs (K = 128, >= one wave of blocks; an explicit
    148-CTA grid keeps the halo-stream kernel where the planner's wave rule would pick the generic
    one): exact against the oracle on the first / middle / last images, equal to the single-CTA
    kernel (planner switch) and to the generic kernel."""
    P = _P()
    import ctypes
    from oracle import oracle as O
    from paper_2110_03901_b200._kernels import conv_device
    from paper_2110_03901_b200.core import ConvSpec
    from paper_2110_03901_b200.traffic import _args
    n, h, c, k, pad, dil = case
    sp = ConvSpec.square(n, c, h, k, 3, stride=1, pad=pad, dilation=dil)
    a = _args(sp, "bf16", "f32", "reuse_aware", 0)
    a.num_ctas = 148
    info = P._lib.ImconvPlanInfo()
    assert P._lib.lib.imconv_plan(ctypes.byref(a), 148, ctypes.byref(info)) == 0 and info.kernel == 3, case
    args = sp.conv_args()
    x = rng.integers(-2, 3, size=(n, h, h, c)).astype(np.int8)
    w = rng.integers(-2, 3, size=(3, 3, c, k)).astype(np.int8)
    xb = torch.from_numpy(x).cuda().float().bfloat16()
    wb = torch.from_numpy(w).cuda().float().bfloat16()
    y = conv_device(xb, wb, *args, out_dtype=torch.float32, num_ctas=148)
    imgs = sorted({0, n // 2, n - 2, n - 1})
    want = O.conv2d_nhwc_exact_f64(x[imgs], w, *args).astype(np.float32)
    assert np.array_equal(y[imgs].cpu().numpy(), want), case
    P._lib.lib.imconv_debug_set_flags(1 << 30)  # kDbgHaloStreamSingle
    try:
        y_single = conv_device(xb, wb, *args, out_dtype=torch.float32, num_ctas=148)
    finally:
        P._lib.lib.imconv_debug_set_flags(0)
    assert torch.equal(y, y_single)
    y_generic = conv_device(xb, wb, *args, out_dtype=torch.float32, flags=P._lib.FLAG_NO_HALO)
    assert torch.equal(y, y_generic)
    assert torch.equal(conv_device(xb, wb, *args, num_ctas=148), y.bfloat16())


@pytest.mark.parametrize("case", [
    # (N, H, pad, dil): C = K = 64 stacked halo blocks with >= one wave of blocks -> CTA pairs
    (64, 56, 1, 1),    # ResNet s2 3x3 shard: shared taps (dr = 2) and single taps
    (151, 14, 1, 1),   # one block per image (no shared taps), odd block count: a dead second CTA
    (40, 30, 2, 2),    # dilation
])
def test_halo_pairs_exact(rng, case):
    """Stacked halo tiles on CTA pairs (M = 256; each CTA holds one sub-block's shared-tap filter
    atoms and 32 of the 64 columns of every tap): exact against the oracle, equal to the single-CTA
    kernel (planner switch) and to the generic kernel."""
    P = _P()
    from oracle import oracle as O
    from paper_2110_03901_b200._kernels import conv_device
    from paper_2110_03901_b200.core import ConvSpec
    n, h, pad, dil = case
    sp = ConvSpec.square(n, 64, h, 64, 3, stride=1, pad=pad, dilation=dil)
    args = sp.conv_args()
    x = rng.integers(-2, 3, size=(n, h, h, 64)).astype(np.int8)
    w = rng.integers(-2, 3, size=(3, 3, 64, 64)).astype(np.int8)
    xb = torch.from_numpy(x).cuda().float().bfloat16()
    wb = torch.from_numpy(w).cuda().float().bfloat16()
    y = conv_device(xb, wb, *args, out_dtype=torch.float32, num_ctas=148)
    imgs = sorted({0, n // 2, n - 2, n - 1})
    want = O.conv2d_nhwc_exact_f64(x[imgs], w, *args).astype(np.float32)
    assert np.array_equal(y[imgs].cpu().numpy(), want), case
    P._lib.lib.imconv_debug_set_flags(1 << 30)  # kDbgHaloStreamSingle: halo kernels on single CTAs
    try:
        y_single = conv_device(xb, wb, *args, out_dtype=torch.float32, num_ctas=148)
    finally:
        P._lib.lib.imconv_debug_set_flags(0)
    assert torch.equal(y, y_single)
    assert torch.equal(y, conv_device(xb, wb, *args, out_dtype=torch.float32, flags=P._lib.FLAG_NO_HALO))
    assert torch.equal(conv_device(xb, wb, *args, num_ctas=148), y.bfloat16())


def test_static_filter_dependent_chain():
    """IMCONV_FLAG_STATIC_FILTER: the filter loads start before the programmatic-launch wait.
    A chain of dependent convs through every kernel family (row-band stem, stacked halo, generic
    1x1, streamed-filter halo, generic strided 3x3), queued back to back into NaN-filled output
    buffers, must give each layer exactly what a separate flag-free launch on the same input gives:
    an input read before the previous grid finished would show up as NaN or stale values."""
    P = _P()
    from paper_2110_03901_b200._kernels import conv_device
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev).manual_seed(7)
    # (C, K, R, stride, pad): input 64x64 with C = 8 (stem-like, 3 live channels)
    chain = [(8, 64, 7, 2, 3), (64, 64, 3, 1, 1), (64, 128, 1, 1, 0), (128, 128, 3, 1, 1), (128, 256, 3, 2, 1)]
    x0 = torch.randn((4, 64, 64, 8), device=dev, generator=g)
    x0[..., 3:] = 0
    x0 = x0.bfloat16()
    ws, ys, args = [], [], []
    h = 64
    for c, k, r, st, pad in chain:
        w = (torch.randn((r, r, c, k), device=dev, generator=g) * (2.0 / (r * r * c)) ** 0.5).bfloat16()
        ho = (h + 2 * pad - r) // st + 1
        ws.append(w)
        ys.append(torch.full((4, ho, ho, k), float("nan"), device=dev, dtype=torch.bfloat16))
        args.append((st, st, pad, pad, 1, 1))
        h = ho
    torch.cuda.synchronize()
    for rep in range(3):
        for y in ys:
            y.fill_(float("nan"))
        torch.cuda.synchronize()
        inp = x0
        for w, y, a in zip(ws, ys, args):
            conv_device(inp, w, *a, y=y, flags=P._lib.FLAG_STATIC_FILTER)
            inp = y
        torch.cuda.synchronize()
        inp = x0
        for i, (w, y, a) in enumerate(zip(ws, ys, args)):
            ref = conv_device(inp, w, *a)
            torch.cuda.synchronize()
            assert not torch.isnan(y).any(), (rep, i)
            assert torch.equal(y, ref), (rep, i)
            inp = y


def test_independent_launches_overlap_exact():
    """IMCONV_FLAG_INDEPENDENT: a sweep of independent convolutions over their own buffers (every
    kernel family, split-K tails included) queued back to back in one CUDA graph with no
    programmatic-launch wait, so each layer's CTAs start while the previous layer still runs.
    Replayed several times into NaN-refilled outputs, every layer must equal a separate
    serialised launch; and a flag-free launch queued after the sweep still waits for it."""
    P = _P()
    from paper_2110_03901_b200._kernels import conv_device
    from paper_2110_03901_b200.core import ConvSpec
    from paper_2110_03901_b200.traffic import plan
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev).manual_seed(11)
    sq = ConvSpec.square
    sweep = [sq(16, 8, 224, 64, 7, stride=2, pad=3), sq(32, 64, 56, 64, 3, stride=1, pad=1),
             sq(32, 64, 56, 256, 1), sq(64, 128, 28, 128, 3, stride=1, pad=1),
             sq(256, 512, 7, 512, 3, stride=1, pad=1), sq(64, 256, 14, 1024, 1), sq(32, 512, 7, 512, 3, stride=1, pad=1)]
    assert any(plan(sp).sk_split > 1 for sp in sweep)
    xs, ws, ys, refs = [], [], [], []
    for sp in sweep:
        x = torch.randint(-2, 3, (sp.n, sp.h_i, sp.w_i, sp.c_i), device=dev, generator=g).bfloat16()
        w = torch.randint(-2, 3, (sp.h_f, sp.w_f, sp.c_i, sp.c_o), device=dev, generator=g).bfloat16()
        xs.append(x)
        ws.append(w)
        ys.append(torch.empty((sp.n, sp.h_o, sp.w_o, sp.c_o), device=dev, dtype=torch.float32))
        refs.append(conv_device(x, w, *sp.conv_args(), out_dtype=torch.float32))
    torch.cuda.synchronize()
    flags = P._lib.FLAG_STATIC_FILTER | P._lib.FLAG_INDEPENDENT
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for sp, x, w, y in zip(sweep, xs, ws, ys):
            conv_device(x, w, *sp.conv_args(), y=y, out_dtype=torch.float32, flags=flags)
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=s):
        for sp, x, w, y in zip(sweep, xs, ws, ys):
            conv_device(x, w, *sp.conv_args(), y=y, out_dtype=torch.float32, flags=flags)
    total = torch.zeros((), device=dev, dtype=torch.float64)
    for rep in range(20):
        for y in ys:
            y.fill_(float("nan"))
        graph.replay()
        # a flag-free consumer queued after the sweep: must see the last layer's finished output
        total += ys[-1].double().sum()
        torch.cuda.synchronize()
        for i, (y, ref) in enumerate(zip(ys, refs)):
            assert torch.equal(y, ref), (rep, i)
    assert total.item() == 20 * refs[-1].double().sum().item()


def test_conv_sweep_concurrent_exact():
    """paper_2110_03901_b200.sweep.conv_sweep: independent convolutions in flight together
    (IMCONV_FLAG_INDEPENDENT on sms // jobs CTAs each, the first launch IMCONV_FLAG_BARRIER).
    A conv queued just BEFORE the sweep writes the input of the sweep's third member -- the
    barrier head must keep that member from running ahead of it -- and every output must equal
    a serialised launch, for several values of jobs."""
    P = _P()
    from paper_2110_03901_b200._kernels import conv_device
    from paper_2110_03901_b200.core import ConvSpec
    from paper_2110_03901_b200.sweep import conv_sweep
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev).manual_seed(21)
    sq = ConvSpec.square
    specs = [sq(32, 8, 224, 64, 7, stride=2, pad=3), sq(64, 64, 56, 64, 3, stride=1, pad=1),
             sq(64, 256, 56, 64, 1), sq(64, 128, 28, 128, 3, stride=1, pad=1), sq(128, 512, 7, 512, 3, stride=1, pad=1),
             sq(64, 256, 14, 1024, 1), sq(16, 1024, 14, 512, 1)]
    xs = [torch.randint(-2, 3, (sp.n, sp.h_i, sp.w_i, sp.c_i), device=dev, generator=g).bfloat16() for sp in specs]
    ws = [torch.randint(-2, 3, (sp.h_f, sp.w_f, sp.c_i, sp.c_o), device=dev, generator=g).bfloat16() for sp in specs]
    # producer of sweep member 2's input (a 1x1 conv from another tensor, queued before the sweep)
    src = torch.randint(-1, 2, (64, 56, 56, 64), device=dev, generator=g).bfloat16()
    wsrc = torch.randint(-1, 2, (1, 1, 64, 256), device=dev, generator=g).bfloat16()
    xs[2] = torch.empty((64, 56, 56, 256), device=dev, dtype=torch.bfloat16)
    ref_x2 = conv_device(src, wsrc, 1, 1, 0, 0, 1, 1)
    refs = [conv_device(x if i != 2 else ref_x2, w, *sp.conv_args(), out_dtype=torch.float32)
            for i, (sp, x, w) in enumerate(zip(specs, xs, ws))]
    torch.cuda.synchronize()
    ys = [torch.empty_like(r) for r in refs]
    for jobs in (2, 4, 8):
        for rep in range(3):
            xs[2].fill_(float("nan"))
            for y in ys:
                y.fill_(float("nan"))
            conv_device(src, wsrc, 1, 1, 0, 0, 1, 1, y=xs[2])
            # (the barrier head is the first LAUNCH whatever the order puts there)
            conv_sweep([(x, w, sp.conv_args(), y) for sp, x, w, y in zip(specs, xs, ws, ys)], jobs=jobs,
                       order=("given", "mix", "lpt")[rep])
            torch.cuda.synchronize()
            for i, (y, ref) in enumerate(zip(ys, refs)):
                assert torch.equal(y, ref), (jobs, rep, i)
