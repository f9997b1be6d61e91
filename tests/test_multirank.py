"""N>1 path on CPU: world_size-2 gloo ranks shard the batch, convolve their
slabs (the CPU oracle stands in for the GPU kernel here) and all-gather the
NHWC output; the result must equal the single-rank convolution bit for bit."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2110_03901_b200.sharding import shard_range


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n_total, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle as O
        from paper_2110_03901_b200.sharding import gather_shards
        rng = np.random.default_rng(7)  # identical operands on every rank (replicated filters)
        x = rng.integers(-4, 5, size=(n_total, 9, 8, 16)).astype(np.int64)
        w = rng.integers(-4, 5, size=(3, 3, 16, 8)).astype(np.int64)
        lo, hi = shard_range(n_total, world, rank)
        y_local = torch.from_numpy(O.conv2d_nhwc_i64(x[lo:hi], w, 2, 1, 1, 1, 1, 2))
        y = gather_shards(y_local, n_total)
        if rank == 0:
            want = O.conv2d_nhwc_i64(x, w, 2, 1, 1, 1, 1, 2)
            out_q.put(bool(np.array_equal(y.numpy(), want)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n_total", [5, 8])
def test_two_rank_sharded_conv_gathers_to_full_result(n_total):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n_total, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert q.get(timeout=10) is True


def test_shard_ranges_cover_batch_exactly():
    for n in (1, 7, 8, 256):
        for world in (1, 2, 4, 8):
            ranges = [shard_range(n, world, r) for r in range(world)]
            assert ranges[0][0] == 0 and ranges[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(ranges, ranges[1:]))
            sizes = [hi - lo for lo, hi in ranges]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_range(8, 2, 2)


def _verify_worker(rank, world, port, corrupt, out_q):
    """bench.verify_outputs over gloo: each rank's shard output (the CPU oracle stands in for
    the kernel), all-gathered; rank 0 checks the first and last image of every shard."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import bench
        from oracle import oracle as O
        from paper_2110_03901_b200.core import ConvSpec
        from paper_2110_03901_b200.workloads import Layer
        dev = torch.device("cpu")
        layers_full = [Layer("a", ConvSpec.square(5, 16, 9, 24, 3, stride=2, pad=1), relu_input=True),
                       Layer("b", ConvSpec.square(5, 8, 12, 16, 7, stride=2, pad=3)),
                       Layer("stem", ConvSpec.square(5, 8, 10, 16, 3, stride=1, pad=1))]
        work = []
        for li, layer in enumerate(layers_full):
            lo, hi = shard_range(layer.spec.n, world, rank)
            sp = layer.spec.with_batch(hi - lo)
            x, w = bench.make_operands(layer, sp, li, lo, dev)
            y = torch.from_numpy(O.conv2d_nhwc_taps(x.float().numpy(), w.float().numpy(),
                                                    *sp.conv_args())).bfloat16()
            if corrupt and rank == 1 and li == 1:
                y[-1, 0, 0, 0] += 1.0
            work.append((layer, sp, x, w, y))
        res = bench.verify_outputs(work, layers_full, world, rank, dev,
                                   lambda n, r: shard_range(n, world, r),
                                   lambda layer, sp, li, lo: bench.make_operands(layer, sp, li, lo, dev)[0],
                                   O.conv2d_nhwc_taps)
        if rank == 0:
            out_q.put((res["ok"], res["checked_images"], res["failures"]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("corrupt", [False, True])
def test_bench_parity_gather_two_ranks(corrupt):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_verify_worker, args=(r, 2, port, corrupt, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=180)
        assert p.exitcode == 0
    ok, checked, failures = q.get(timeout=10)
    assert checked == 3 * 4  # 3 layers x (first, last image) x 2 shards
    if corrupt:
        assert not ok and failures == ["b[4]"]
    else:
        assert ok and not failures
