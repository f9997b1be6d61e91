"""DRAM-traffic predictor (host C++ replay of the kernel raster).

CPU tests: the replay runs on the host and needs no GPU.  Measured-vs-predicted
agreement on B200 is in profiles/r1/traffic_predictor.md (tools/traffic_validate.py).
"""

import ctypes

import pytest

from paper_2110_03901_b200 import ConvSpec, _lib
from paper_2110_03901_b200.traffic import predict


def _lines(nbytes):
    return (nbytes + 127) // 128 * 128


def test_large_cache_reads_are_compulsory():
    # 1x1 stride 1: every input and filter byte exactly once; output stays resident
    sp = ConvSpec.square(4, 64, 28, 128, 1)
    p = predict(sp, l2_bytes=1 << 30)
    assert p.dram_read_bytes == p.compulsory_read_bytes
    assert p.dram_read_bytes == _lines(4 * 28 * 28 * 64 * 2) + _lines(64 * 128 * 2)
    assert p.dram_write_bytes == 0 and p.resident_dirty_bytes == 4 * 28 * 28 * 128 * 2


def test_padding_taps_touch_no_memory():
    # 3x3 pad 1 on a 1x1 image: only the centre tap reads the single pixel
    sp = ConvSpec.square(2, 64, 1, 64, 3, stride=1, pad=1)
    p = predict(sp, l2_bytes=1 << 30)
    assert p.compulsory_read_bytes == _lines(2 * 64 * 2) + _lines(9 * 64 * 64 * 2)


def test_no_cache_reads_every_request():
    sp = ConvSpec.square(2, 128, 14, 64, 3, stride=1, pad=1)
    p = predict(sp, l2_bytes=0)
    y_lines = 2 * 14 * 14 * 64 * 2 // 128
    assert p.dram_read_bytes == (p.line_requests - y_lines) * 128
    assert p.dram_write_bytes == 2 * 14 * 14 * 64 * 2


def test_reuse_aware_order_never_worse_and_helps_small_caches():
    """The paper's claim in the replay: channel chunk outer / tap inner re-reads the same
    input window while it is still cached."""
    sp = ConvSpec.square(8, 512, 14, 256, 3, stride=1, pad=1)
    for cap in (1 << 20, 4 << 20, 64 << 20):
        ra = predict(sp, order="reuse_aware", l2_bytes=cap).dram_read_bytes
        fm = predict(sp, order="filter_major", l2_bytes=cap).dram_read_bytes
        assert ra <= fm
    assert predict(sp, order="reuse_aware", l2_bytes=2 << 20).dram_read_bytes < \
        predict(sp, order="filter_major", l2_bytes=2 << 20).dram_read_bytes


def test_plan_matches_launcher_geometry():
    sp = ConvSpec.square(256, 256, 14, 1024, 1)  # s4 1x1b: BN 256, 4 channel blocks, B-stationary grid
    p = predict(sp)
    assert (p.bn, p.mt, p.kernel) == (256, 1, "generic")
    assert p.tiles == (256 * 14 * 14 + 127) // 128 * 4
    assert p.grid % 4 == 0
    stem = predict(ConvSpec.square(256, 8, 224, 64, 7, stride=2, pad=3))
    assert stem.kernel == "row-band"


def test_planner_choices_on_resnet50():
    """The planner's kernel / block-shape decisions for the ResNet-50 layers, as
    reported by the host-side replay: a regression guard for the measured choices."""
    from paper_2110_03901_b200.workloads import resnet50_layers
    layers = {l.name: l.spec for l in resnet50_layers(256)}
    expect = {
        "stem": ("row-band", None),
        "s2b1_3x3": ("halo", None),          # C = 64, stride 1: stacked halo sub-blocks
        "s3b1_3x3": ("halo-stream", None),   # C = 128, stride 1, K = 128: streamed-filter halo tiles
        "s3b0_3x3": ("generic", 128),        # stride 2
        "s4b1_1x1b": ("generic", 256),       # B-stationary output layer
        "s2b1_1x1b": ("generic", 128),       # output-heavy 1x1, >= 16 waves: streamed filter, 128-wide
        "s4b1_3x3": ("generic", 256),
    }
    for name, (kernel, bn) in expect.items():
        t = predict(layers[name])
        assert t.kernel == kernel, name
        if bn is not None:
            assert t.bn == bn, name
    # 32 images per GPU (8-GPU shard): stage-4 3x3 runs 128-wide blocks (more blocks than 256-wide)
    assert predict(resnet50_layers(32)[[l.name for l in resnet50_layers(32)].index("s4b1_3x3")].spec).bn == 128
    # 128 images per GPU (2-GPU shard): s5 3x3 keeps 128 x 256 blocks (no split-K tail on 128 x 128),
    # s4 3x3 runs CTA pairs (a 3-way split of a 36-stage tail loses), s3 3x3 the generic kernel
    # (4 halo-stream waves vs 3 generic waves)
    l128 = {l.name: l.spec for l in resnet50_layers(128)}
    t = predict(l128["s5b1_3x3"])
    assert (t.bn, t.tiles, t.grid) == (256, 98, 98)
    t = predict(l128["s4b1_3x3"])
    assert (t.bn, t.tiles) == (256, 98)  # 98 CTA-pair blocks of 256 x 256
    assert predict(l128["s3b1_3x3"]).kernel == "generic"


def test_invalid_arguments():
    a = _lib.ImconvArgs()
    t = _lib.ImconvTraffic()
    assert _lib.lib.imconv_predict_traffic(None, 1 << 20, 148, ctypes.byref(t)) == -1
    assert _lib.lib.imconv_predict_traffic(ctypes.byref(a), 1 << 20, 148, ctypes.byref(t)) == -1  # zero extents
    with pytest.raises(_lib.ImconvError):
        predict(ConvSpec.square(1, 64, 8, 64, 3), sms=0)


def test_launch_plan_branches_of_the_benchmarked_batches():
    """imconv_plan (host code): the planner branches bench.py's shards select, which the GPU
    tests in test_gpu_bench_batches.py then check against the oracle."""
    from paper_2110_03901_b200.traffic import plan
    from paper_2110_03901_b200.workloads import resnet50_layers
    by_name = {n: {l.name: plan(l.spec) for l in resnet50_layers(n)} for n in (256, 32)}
    assert by_name[256]["stem"].kernel == "row-band"
    assert by_name[256]["s2b0_3x3"].kernel == "halo"
    assert by_name[256]["s3b1_3x3"].kernel == "halo-stream"
    s5 = by_name[256]["s5b0_3x3"]
    # CTA pairs: 98 pair blocks on 74 clusters, the last 24 split 3 ways
    assert s5.kernel == "generic" and s5.cta_pair and s5.sk_mode == 1 and s5.sk_split == 3
    assert s5.sk_tail == 98 % 74
    assert by_name[256]["s4b0_3x3"].cta_pair and by_name[256]["s4b0_3x3"].sk_mode == 0  # stream-K is opt-in
    assert by_name[32]["s5b0_3x3"].sk_split == 5
    # a caller grid above one CTA per SM turns split-K off (splits must be co-resident)
    from paper_2110_03901_b200 import _lib
    from paper_2110_03901_b200.traffic import _args
    import ctypes
    sp = resnet50_layers(32)[-2].spec
    a = _args(sp, "bf16", None, "reuse_aware", 0)
    a.num_ctas = 300
    t = _lib.ImconvPlanInfo()
    assert _lib.lib.imconv_plan(ctypes.byref(a), 148, ctypes.byref(t)) == 0
    assert t.sk_split == 1
