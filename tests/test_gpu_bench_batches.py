"""GPU parity of what bench.py runs: the ResNet-50 layer shapes at the batch sizes the
benchmark and the scaling run use per GPU (256 / 128 / 64 / 32 images), and split-K
under CUDA-graph replay (bench.py times the step as a replayed graph).

The batch size selects the planner branch (imconv_plan): CTA pairs once a wave of
128 x 256 blocks exists, split-K tails (3-way at 256 images, 5-way at 32), 128 x 128
blocks below one wave, halo-stream vs generic by wave count.  Images are independent,
so every layer runs on the full shard (same launch as the benchmark) and sampled
images are checked against the CPU oracle (reference semantics: ``direct_conv`` is the
ground truth, /root/reference/pkg/src/sasim/core.py:194-208).

Tolerances (BASELINE.json north_star): bf16 N(0,1) data, bf16 output: normalised max
error <= 1e-2 against the fp32 oracle on the same bf16-rounded operands; integer-valued
data: bit-exact.
"""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

REL_TOL = 1e-2


def _norm_err(got, ref):
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    return float(np.abs(got - ref).max() / max(np.abs(ref).max(), 1e-30))


def _operands(layer, sp, seed, dev):
    """bench.py's synthetic operands (N(0,1), post-ReLU clamp, Kaiming weights, stem C=3 of 8)."""
    g = torch.Generator(device=dev).manual_seed(seed)
    x = torch.randn((sp.n, sp.h_i, sp.w_i, sp.c_i), generator=g, device=dev)
    if layer.relu_input:
        x.clamp_(min=0)
    w = torch.randn((sp.h_f, sp.w_f, sp.c_i, sp.c_o), generator=g, device=dev) * (2.0 / (sp.c_i * sp.h_f * sp.w_f)) ** 0.5
    if layer.name == "stem":
        x[..., 3:] = 0
        w[:, :, 3:, :] = 0
    return x.bfloat16(), w.bfloat16()


# branches each shard size must exercise (imconv_plan labels; see the module docstring)
EXPECTED_BRANCHES = {
    256: {"row-band", "halo", "halo-stream", "generic 256x256 pair", "generic 256x256 pair split3",

          "generic 128x256 b-stationary", "generic 256x64 b-stationary"},
    128: {"row-band", "halo", "generic 256x128", "generic 256x256 pair", "generic 256x256 pair split3", "generic 128x256"},
    64: {"halo-stream", "generic 128x256", "generic 128x128 ksub2", "generic 256x256 pair"},
    32: {"halo-stream", "generic 128x256 split5", "generic 128x128 ksub2", "generic 256x256 pair"},
}


@pytest.mark.parametrize("n", [256, 128, 64, 32])
def test_resnet50_shapes_at_shard_batch(n):
    _check_shapes_at_shard_batch(n, independent=False)


@pytest.mark.parametrize("n", [64, 32])
def test_resnet50_shapes_throughput_mode(n):
    """bench.py launches the sweep with IMCONV_FLAG_INDEPENDENT: sub-wave layers then take the
    throughput-mode plans (CTA pairs, no split-K) -- checked against the oracle the same way."""
    _check_shapes_at_shard_batch(n, independent=True)


def _check_shapes_at_shard_batch(n, independent):
    import paper_2110_03901_b200 as P
    from oracle import oracle as O
    from paper_2110_03901_b200._kernels import conv_device
    from paper_2110_03901_b200.traffic import plan
    dev = torch.device("cuda", 0)
    branches = set()
    seen = set()
    for li, layer in enumerate(P.workloads.resnet50_layers(n)):
        if layer.spec in seen:
            continue
        seen.add(layer.spec)
        sp = layer.spec
        flags = P._lib.FLAG_STATIC_FILTER | (P._lib.FLAG_INDEPENDENT if independent else 0)
        branches.add(plan(sp, flags=flags).branch)
        x, w = _operands(layer, sp, 100 + li, dev)
        y = conv_device(x, w, *sp.conv_args(), flags=flags)  # bench.py's call
        torch.cuda.synchronize()
        wf = w.float().cpu().numpy()
        for i in sorted({0, n // 2, n - 1}):
            ref = O.conv2d_nhwc_taps(x[i:i + 1].float().cpu().numpy(), wf, *sp.conv_args())
            err = _norm_err(y[i:i + 1].float().cpu().numpy(), ref)
            assert err <= REL_TOL, (n, layer.name, i, err)
        del x, w, y
    if independent:
        assert not any("split" in b for b in branches if "x" in b and n <= 64), branches
        assert "generic 256x256 pair" in branches
        return
    missing = EXPECTED_BRANCHES[n] - branches
    assert not missing, (n, missing, branches)


def _tail_first_image(pl, sp):
    """First image whose output rows belong to a split-K tail block."""
    first_tile = pl.tiles - pl.sk_tail
    rows_per_block = 128 * pl.mt * (2 if pl.cta_pair else 1)
    n_tiles = -(-sp.c_o // pl.bn)
    return int((first_tile // n_tiles) * rows_per_block // (sp.h_o * sp.w_o))


def test_split_k_graph_replay_bit_exact():
    """Split-K tails captured in ONE CUDA graph and replayed 300 times, the inputs rewritten
    before every replay: every replay's output is bit-exact.  Cases: s5 3x3 at 256 images
    (CTA pairs, 3-way split, bf16 out), s5 3x3 at 32 images (5-way, fp32 out), an int8 5-way
    split (C = K = 1024 at 16 images) and an int8 CTA-pair 2-way split (128 images).
    Integer-valued operands scaled by a per-replay factor c: y(c x) = c y(x) exactly, so a
    split that reads a peer's stale partial (an earlier replay's) or skips the wait fails."""
    import paper_2110_03901_b200 as P
    from oracle import oracle as O
    from paper_2110_03901_b200.core import ConvSpec
    from paper_2110_03901_b200._kernels import conv_device
    from paper_2110_03901_b200.traffic import plan
    dev = torch.device("cuda", 0)
    rng = np.random.default_rng(11)
    cases = [  # (spec, compute dtype, out dtype, expected split, expected sk_mode)
        (ConvSpec.square(256, 512, 7, 512, 3, stride=1, pad=1), torch.bfloat16, torch.bfloat16, 3, 1),
        (ConvSpec.square(32, 512, 7, 512, 3, stride=1, pad=1), torch.bfloat16, torch.float32, 5, 1),
        # int8: s5 3x3 at 32 images plans 128 x 128 blocks with no split; C = K = 1024 at 16 splits 5 ways
        (ConvSpec.square(16, 1024, 7, 1024, 3, stride=1, pad=1), torch.int8, torch.int32, 5, 1),
        # CTA pairs with a split tail (pair tiles over 74 clusters), int8
        (ConvSpec.square(128, 1024, 7, 1024, 3, stride=1, pad=1), torch.int8, torch.int32, 2, 1),
        # stream-K over the last two waves (opt-in planner switch, set during capture below):
        # s4 3x3 at 256 images (CTA pairs), s3 3x3 at 128 (single CTAs)
        (ConvSpec.square(256, 256, 14, 256, 3, stride=1, pad=1), torch.bfloat16, torch.bfloat16, 1, 2),
        (ConvSpec.square(128, 128, 28, 128, 3, stride=1, pad=1), torch.bfloat16, torch.float32, 1, 2),
    ]
    STREAM_K = 1 << 29  # imconv_api.cu kDbgStreamK
    P._lib.lib.imconv_debug_set_flags(STREAM_K)
    work = []
    for sp, cdt, odt, want_split, want_mode in cases:
        pl = plan(sp, dtype="int8" if cdt == torch.int8 else "bf16", flags=P._lib.FLAG_STATIC_FILTER)
        assert pl.kernel == "generic" and pl.sk_split == want_split and pl.sk_mode == want_mode, (sp, pl)
        lim = 42 if cdt == torch.int8 else 2  # |c * x| <= 126 (int8, |c| <= 3) / 6 (exact in bf16)
        bases = [rng.integers(-lim, lim + 1, size=(sp.n, sp.h_i, sp.w_i, sp.c_i)) for _ in range(2)]
        w = rng.integers(-lim, lim + 1, size=(sp.h_f, sp.w_f, sp.c_i, sp.c_o))
        t0 = _tail_first_image(pl, sp)
        imgs = sorted(set([0, 1]) | set(range(max(t0 - 1, 0), sp.n)))
        want = [O.conv2d_nhwc_exact_f64(b[imgs], w, *sp.conv_args()) for b in bases]
        xs = [torch.from_numpy(b).to(dev).to(cdt) for b in bases]
        x = torch.empty_like(xs[0])
        wd = torch.from_numpy(w).to(dev).to(cdt)
        y = torch.empty((sp.n, sp.h_o, sp.w_o, sp.c_o), dtype=odt, device=dev)
        idx = torch.tensor(imgs, device=dev)
        exp = [torch.from_numpy(v).to(dev).to(torch.float64) for v in want]
        work.append((sp, x, xs, wd, y, idx, exp, cdt, odt))
    # warm up outside capture (kernel attributes, counters), then capture all three launches
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for sp, x, xs, wd, y, *_ in work:
            x.copy_(xs[0])
            conv_device(x, wd, *sp.conv_args(), y=y, out_dtype=y.dtype)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for sp, x, xs, wd, y, *_ in work:
            conv_device(x, wd, *sp.conv_args(), y=y, out_dtype=y.dtype, flags=P._lib.FLAG_STATIC_FILTER)
    P._lib.lib.imconv_debug_set_flags(0)
    factors = [1, -2, 3, -1, 2, -3]
    for it in range(300):
        c = factors[it % len(factors)]
        b = (it // len(factors)) % 2
        for sp, x, xs, wd, y, *_ in work:
            x.copy_(xs[b] * c)
            y.fill_(0)
        g.replay()
        for sp, x, xs, wd, y, idx, exp, cdt, odt in work:
            got = y.index_select(0, idx).to(torch.float64)
            ref = exp[b] * c
            if odt == torch.bfloat16:  # exact fp32 sums, rounded once to bf16
                ref = ref.float().bfloat16().to(torch.float64)
            assert torch.equal(got, ref), (it, tuple(sp.conv_args()), sp.n, odt)
    # eager calls after the replays still see consistent counters
    for sp, x, xs, wd, y, idx, exp, cdt, odt in work:
        x.copy_(xs[1])
        yy = conv_device(x, wd, *sp.conv_args(), out_dtype=odt)
        ref = exp[1] if odt != torch.bfloat16 else exp[1].float().bfloat16().to(torch.float64)
        assert torch.equal(yy.index_select(0, idx).to(torch.float64), ref)


def test_debug_invariant_build():
    """Every kernel path through the debug-invariant build (libimconv_debug.so): device checks
    on mbarrier phases, TMEM allocation, split-K / stream-K tickets, work units and epilogue
    chunk counts, host checks on the planner's schedule; outputs bit-exact on integer data.
    Runs in its own process (the debug library is bound explicitly, never by the package)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, os.path.join(root, "tests", "debug_check.py")], capture_output=True,
                       text=True, timeout=900, cwd=root)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "all cases clean and exact" in r.stdout
