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
