"""Host-side logic of the drop-in (no GPU): layer descriptor, layouts, the
lowering index maths, block planning and the traffic model, checked against
the reference's known-answer tests and golden vectors."""

import numpy as np
import pytest

from conftest import SPEC_FIELDS, spec_from_vec


def P():
    import paper_2110_03901_b200 as p
    return p


# ------------------------------------------------------------------ ConvSpec (core.py:50-125)

def test_conv_spec_derived_dims():
    ConvSpec = P().ConvSpec
    spec = ConvSpec.square(1, 3, 224, 64, 7, stride=2, pad=3)
    assert (spec.h_o, spec.w_o) == (112, 112)
    assert (ConvSpec.square(1, 1, 5, 1, 3, stride=2).h_o,) == (2,)
    assert spec.gemm_m == 112 * 112 and spec.gemm_k == 7 * 7 * 3 and spec.gemm_n == 64
    assert spec.flops == 2 * spec.macs


def test_conv_spec_rejects_bad_shapes():
    p = P()
    with pytest.raises(p.ShapeError):
        p.ConvSpec.square(1, 1, 2, 1, 3)
    with pytest.raises(p.ShapeError):
        p.ConvSpec.square(0, 1, 4, 1, 1)
    with pytest.raises(p.ShapeError):
        p.ConvSpec(n=1, c_i=1, h_i=4, w_i=4, c_o=1, h_f=1, w_f=1, pad_h=-1)
    assert issubclass(p.ShapeError, ValueError)


def test_random_spec_reproduces_reference_sequence(golden):
    # the golden file was produced with the reference's random_spec on this seed
    # (make_golden.py); our sampler must yield the same layers from the same
    # rng stream (operands are drawn between specs exactly as there).
    from paper_2110_03901_b200.workloads import random_spec
    rng = np.random.default_rng(20261020)
    for i in range(64):
        spec = random_spec(rng, max_hw=12, max_n=4, max_co=16)
        rng.integers(-4, 5, size=(spec.n, spec.h_i, spec.w_i, spec.c_i))
        rng.integers(-4, 5, size=(spec.h_f, spec.w_f, spec.c_i, spec.c_o))
        assert spec == spec_from_vec(golden[f"int{i}_spec"]), i


# ------------------------------------------------------------------ Tensor / relayout (core.py:128-175)

def test_relayout_known_answers_and_round_trips(rng):
    p = P()
    t = p.Tensor((1, 2, 1, 2), p.Layout.NCHW, np.array([1, 2, 3, 4]))
    assert p.relayout(t, p.Layout.NHWC).data.tolist() == [1, 3, 2, 4]
    arr = rng.integers(0, 100, size=(2, 3, 4, 5))
    t = p.Tensor.from_array(arr, p.Layout.NCHW)
    for mid in (p.Layout.NHWC, p.Layout.HWCN):
        back = p.relayout(p.relayout(t, mid), p.Layout.NCHW)
        assert np.array_equal(back.view(), arr)
    with pytest.raises(p.ShapeError):
        p.relayout(p.Tensor((2, 2), p.Layout.ROW_MAJOR, np.arange(4)), p.Layout.NCHW)
    with pytest.raises(p.ShapeError):
        p.Tensor((2, 2, 2), p.Layout.NCHW, np.arange(8))


def test_relayout_torch_cpu_tensor():
    import torch
    p = P()
    x = torch.arange(24).reshape(1, 2, 3, 4)
    t = p.Tensor.from_array(x, p.Layout.NCHW)
    got = p.relayout(t, p.Layout.NHWC).view()
    assert torch.equal(got, x.permute(0, 2, 3, 1))


# ------------------------------------------------------------------ lowering.py

def test_column_orderings_are_inverse_bijections():
    p = P()
    spec = p.ConvSpec.square(1, 3, 6, 2, 3)
    for ordr in p.ColumnOrdering:
        seen = set()
        for r in range(3):
            for s in range(3):
                for c in range(3):
                    k = ordr.index(r, s, c, spec)
                    assert ordr.unindex(k, spec) == (r, s, c)
                    seen.add(k)
        assert seen == set(range(27))


def test_column_permutation_known_answers():
    # reference tests/test_lowering.py:100-119
    p = P()
    assert np.array_equal(p.column_permutation(p.ConvSpec.square(1, 1, 6, 1, 3)), np.arange(9))
    assert np.array_equal(p.column_permutation(p.ConvSpec.square(1, 7, 6, 1, 1)), np.arange(7))
    assert p.column_permutation(p.ConvSpec.square(1, 2, 4, 1, 2)).tolist() == [0, 4, 1, 5, 2, 6, 3, 7]


def test_lower_filter_orderings_are_row_permutations(rng):
    p = P()
    spec = p.ConvSpec.square(1, 3, 6, 4, 3, pad=1)
    f = rng.integers(-4, 5, size=(3, 3, 3, 4))
    cf = p.lower_filter(p.Tensor.from_array(f, p.Layout.HWCN), spec, p.ColumnOrdering.CHANNEL_FIRST).view()
    cl = p.lower_filter(p.Tensor.from_array(f, p.Layout.HWCN), spec, p.ColumnOrdering.CHANNEL_LAST).view()
    assert np.array_equal(cf, f.reshape(27, 4))  # HWCN reshaped IS the channel-first B matrix
    assert np.array_equal(cl[p.column_permutation(spec)], cf)


def test_tile_descriptor_known_answers():
    # reference tests/test_lowering.py:133-146, :182-202
    p = P()
    spec = p.ConvSpec.square(1, 3, 6, 2, 1, stride=2)
    tiles = p.decompose_tiles(spec)
    assert len(tiles) == 1
    assert [tiles[0].gather(i, j) for i in range(2) for j in range(2)] == [(0, 0), (0, 2), (2, 0), (2, 2)]
    spec = p.ConvSpec.square(1, 1, 5, 1, 3, stride=2)
    by = {(t.r, t.s): t for t in p.decompose_tiles(spec)}
    assert by[0, 0].coords() == {(0, 0), (0, 2), (2, 0), (2, 2)}
    assert by[0, 1].coords() == {(0, 1), (0, 3), (2, 1), (2, 3)}
    assert p.tile_overlap(by[1, 1], by[1, 1], spec) == 1.0
    assert p.tile_overlap(by[0, 0], by[0, 2], spec) == 2 / 6
    big = p.ConvSpec.square(1, 1, 99, 1, 3, stride=2)
    bb = {(t.r, t.s): t for t in p.decompose_tiles(big)}
    assert p.tile_overlap(bb[0, 0], bb[0, 2], big) == 0.96


def test_footprint_known_answers():
    p = P()
    assert p.lowered_memory_footprint(p.ConvSpec.square(4, 16, 14, 16, 3, pad=1))["ratio"] == 9.0
    fp = p.lowered_memory_footprint(p.ConvSpec.square(1, 3, 224, 64, 3, stride=2, pad=1))
    assert fp["ratio"] == 9 * (112 * 112) / (224 * 224) and fp["original_bytes"] == 3 * 224 * 224 * 2
    assert p.lowered_memory_footprint(p.ConvSpec.square(1, 8, 10, 4, 1, stride=2))["ratio"] <= 1.0


def test_touched_pixels_T():
    # T = H*W except the 1x1 stride-2 layers (T = H*W/4)
    from paper_2110_03901_b200.lowering import touched_pixels
    p = P()
    assert touched_pixels(p.ConvSpec.square(32, 256, 56, 512, 1, stride=2)) == 28 * 28
    assert touched_pixels(p.ConvSpec.square(8, 64, 56, 64, 3, pad=1)) == 56 * 56
    assert touched_pixels(p.ConvSpec.square(16, 512, 64, 512, 3, pad=2, dilation=2)) == 64 * 64


# ------------------------------------------------------------------ blocksched.py

def test_partition_and_orders():
    p = P()
    from paper_2110_03901_b200.blocksched import SubtileOrder, order_subtiles, partition
    spec = p.ConvSpec.square(2, 3, 7, 5, 3)
    plan = partition(spec, block_m=7, block_n=2, block_k=2)
    assert plan.m_ranges[0][0] == 0 and plan.m_ranges[-1][1] == spec.gemm_m
    assert plan.k_chunks == [(0, 2), (2, 3)]
    with pytest.raises(p.ShapeError):
        partition(spec, 0, 1, 1)
    spec = p.ConvSpec.square(1, 4, 9, 3, 3, stride=2)
    plan = partition(spec, block_m=5, block_n=3, block_k=2)
    fm = order_subtiles(plan, SubtileOrder.FILTER_MAJOR)
    ra = order_subtiles(plan, SubtileOrder.REUSE_AWARE)
    key = lambda s: (s.m_block, s.n_block, s.tile.r, s.tile.s, s.chunk)
    assert sorted(map(key, fm)) == sorted(map(key, ra))
    assert [s.m_block for s in fm[:len(plan.m_ranges)]] == list(range(len(plan.m_ranges)))
    assert all(s.m_block == 0 for s in ra[:plan.subtiles_per_block])


def test_reuse_traffic_matches_reference_golden(golden):
    from paper_2110_03901_b200.blocksched import SubtileOrder, order_subtiles, partition, reuse_traffic, \
        working_set_bytes
    for i in range(int(golden["n_trf"])):
        spec = spec_from_vec(golden[f"trf{i}_spec"])
        bm, bn, bk, budget, pol = (int(v) for v in golden[f"trf{i}_blk"])
        plan = partition(spec, block_m=bm, block_n=bn, block_k=bk)
        order = order_subtiles(plan, SubtileOrder.REUSE_AWARE if pol else SubtileOrder.FILTER_MAJOR)
        res = reuse_traffic(plan, order, budget, spec)
        want = golden[f"trf{i}_res"].tolist()
        assert [res.dram_bytes, res.hits, res.misses, working_set_bytes(plan)] == want, i


def test_reuse_aware_beats_filter_major_on_strided_case():
    # reference tests/test_blocksched.py:108-121
    p = P()
    from paper_2110_03901_b200.blocksched import SubtileOrder, order_subtiles, partition, reuse_traffic, \
        working_set_bytes
    spec = p.ConvSpec.square(1, 4, 99, 4, 3, stride=2)
    plan = partition(spec, block_m=-(-spec.gemm_m // 4), block_n=spec.c_o, block_k=spec.c_i)
    budget = 2 * working_set_bytes(plan)
    fm = reuse_traffic(plan, order_subtiles(plan, SubtileOrder.FILTER_MAJOR), budget, spec)
    ra = reuse_traffic(plan, order_subtiles(plan, SubtileOrder.REUSE_AWARE), budget, spec)
    assert ra.dram_bytes < fm.dram_bytes and ra.hit_fraction > max(fm.hit_fraction, 0.3)


def test_traffic_csv(tmp_path):
    from paper_2110_03901_b200.blocksched import write_traffic_csv
    rows = [{"policy": "reuse_aware", "block_m": 4, "block_n": 2, "block_k": 2, "dram_bytes": 10,
             "hit_fraction": 0.5}]
    path = tmp_path / "traffic.csv"
    write_traffic_csv(path, rows)
    text = path.read_text().splitlines()
    assert text[0].startswith("policy,") and text[1] == "reuse_aware,4,2,2,10,0.5"


# ------------------------------------------------------------------ workloads

def test_resnet50_layer_table():
    from paper_2110_03901_b200.workloads import baseline_configs, resnet50_layers
    layers = resnet50_layers(256)
    assert len(layers) == 53
    assert abs(sum(l.spec.flops for l in layers) / 1e9 - 2193.3) < 0.1
    assert len({l.spec for l in layers}) == 23
    cfg = baseline_configs()
    assert abs(cfg["cfg1"][0].spec.flops / 1e9 - 1.850) < 1e-3
    assert abs(cfg["cfg3"][0].spec.flops / 1e9 - 309.24) < 1e-2
    assert abs(cfg["cfg5"][0].spec.flops / 1e9 - 59.19) < 1e-2


def test_synthetic_operands_distributions():
    import torch
    from paper_2110_03901_b200.workloads import baseline_configs, resnet50_layers
    stem = resnet50_layers(2)[0]
    x, w = __import__("paper_2110_03901_b200.workloads", fromlist=["x"]).synthetic_operands(stem, n=2)
    assert x.dtype == torch.bfloat16 and x.shape == (2, 224, 224, 8)
    assert torch.count_nonzero(x[..., 3:]) == 0 and torch.count_nonzero(w[:, :, 3:]) == 0
    l5 = baseline_configs()["cfg5"][0]
    xi, wi = __import__("paper_2110_03901_b200.workloads", fromlist=["x"]).synthetic_operands(l5, n=1)
    assert xi.dtype == torch.int8 and int(xi.min()) >= -128


def test_sweep_mixed_order_balances_memory_and_tensor_work():
    """sweep.mixed_order (host code): a permutation of the sweep in which memory-bound and
    compute-bound convolutions alternate (bounded running surplus of memory time), and the
    long-pole stem is launched early."""
    import torch
    from paper_2110_03901_b200 import sweep as SW
    from paper_2110_03901_b200.workloads import baseline_configs
    layers = baseline_configs()["cfg4"]
    convs = []
    for l in layers:
        sp = l.spec
        convs.append((torch.empty((sp.n, sp.h_i, sp.w_i, sp.c_i), dtype=torch.bfloat16, device="meta"),
                      torch.empty((sp.h_f, sp.w_f, sp.c_i, sp.c_o), dtype=torch.bfloat16, device="meta"),
                      sp.conv_args(),
                      torch.empty((sp.n, sp.h_o, sp.w_o, sp.c_o), dtype=torch.bfloat16, device="meta")))
    order = SW.mixed_order(convs)
    assert sorted(order) == list(range(len(convs)))
    est = [SW._est_us2(x, w, y) for x, w, _a, y in convs]
    goal = sum(m for _t, m in est) / sum(t + m for t, m in est)
    # the running surplus of memory time over the sweep's mix never exceeds one layer's worth,
    # where the ResNet order accumulates several stage-2 layers' worth
    surplus = [est[i][1] - goal * sum(est[i]) for i in range(len(convs))]
    bound = max(abs(v) for v in surplus) + 1e-9

    def worst(seq):
        run, w = 0.0, 0.0
        for i in seq:
            run += surplus[i]
            w = max(w, abs(run))
        return w

    assert worst(order) <= bound
    assert worst(range(len(convs))) > 3 * bound
    assert [layers[i].name for i in order].index("stem") < 4
    # one-sided sweeps keep their order
    assert SW.mixed_order(convs[1:2] * 3) == [0, 1, 2]


def test_sweep_rejects_overlapping_buffers():
    """sweep._check_disjoint (host code): a sweep output may not overlap any operand or output of
    another member -- the IMCONV_FLAG_INDEPENDENT contract."""
    import pytest
    import torch
    from paper_2110_03901_b200.sweep import _check_disjoint, default_jobs
    buf = torch.zeros(4096)
    a, b, c = buf[:1024], buf[1024:2048], buf[2048:3072]
    w = torch.zeros(64)
    _check_disjoint([(a, w, None, b), (a, w, None, c)])          # shared inputs are fine
    with pytest.raises(ValueError):
        _check_disjoint([(a, w, None, b), (b, w, None, c)])      # output 0 is input 1
    with pytest.raises(ValueError):
        _check_disjoint([(a, w, None, buf[1000:1100]), (c, w, None, b)])  # outputs overlap
    with pytest.raises(ValueError):
        _check_disjoint([(buf.view(64, 64).t(), w, None, b)])          # non-contiguous operand
    assert default_jobs(2.2e12, 53) < default_jobs(2.7e11, 53)
    assert default_jobs(2 * 309e9, 2) == 1.0 and default_jobs(76e9, 41) == 8.0 and default_jobs(266e9, 6) == 2.0
