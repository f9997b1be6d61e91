"""Batch (N) sharding across ranks -- the only parallelism the path needs
(SURVEY.md §8(e)): every image is independent, so rank r convolves the
contiguous image range ``shard_range(N, world, r)`` with replicated filters
and there is no collective on the hot path.  ``gather_shards`` reassembles
the NHWC output (N is outermost, so shards are contiguous slabs) for
verification only -- NCCL over NVLink on GPUs, gloo on CPU.
"""

from __future__ import annotations

import torch
import torch.distributed as dist


def shard_range(n_total: int, world: int, rank: int) -> tuple:
    """Contiguous, balanced image range [lo, hi) of ``rank`` (sizes differ by <= 1)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError(f"bad rank {rank} for world {world}")
    base, extra = divmod(n_total, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def gather_shards(y_local: torch.Tensor, n_total: int, group=None) -> torch.Tensor:
    """All-gather per-rank (n_r, P, Q, K) slabs into the full (N, P, Q, K) tensor.

    Shards may differ in size by one image; each is padded to the largest
    shard for the collective and trimmed afterwards.  Verification only --
    never inside a timed region.
    """
    world = dist.get_world_size(group)
    sizes = [shard_range(n_total, world, r) for r in range(world)]
    cap = max(hi - lo for lo, hi in sizes)
    pad = torch.zeros((cap,) + tuple(y_local.shape[1:]), dtype=y_local.dtype, device=y_local.device)
    pad[: y_local.shape[0]] = y_local
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad, group=group)
    return torch.cat([parts[r][: hi - lo] for r, (lo, hi) in enumerate(sizes)], dim=0)


__all__ = ["gather_shards", "shard_range"]
