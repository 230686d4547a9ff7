"""Multi-GPU partitioning of the HieraSparse hot path.

One process per GPU (torch.distributed, NCCL over NVLink/NVSwitch).  Two
partitions, both taken from the reference's own arithmetic:

* Unit sharding (configs 2-4): a unit is one (request, KV head) pair; units are
  independent (attention.hpp:360-409 runs per query group against one KV head,
  pipeline.hpp:247-263), so each rank owns a contiguous range of units — whole
  KV heads with all their GQA query heads — and no collective touches the data
  path.

* Sequence split (config 5, 1M tokens): rank r owns the contiguous block range
  [nb*r/W, nb*(r+1)/W) of every KV head — the same partition decode_attention
  uses for its splits (attention.hpp:380-381) — compresses and stores only that
  shard, and produces the unnormalised SplitPartial (O, m, l) of attend_range
  over it (attention.hpp:249-304, :65-69).  One all-gather of the packed
  partials (units x gqa x (d+2) fp32, 16.6 KB at 8 heads x GQA 4) and the
  reference's LSE combine (attention.hpp:387-407) finish the step; only the
  last rank carries the dense tail (attention.hpp:383).

The data path runs on the device kernels behind the C ABI; this module only
decides who owns what and moves the partials.
"""
from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class Shard:
    """A contiguous [begin, end) range of units or blocks owned by one rank."""

    begin: int
    end: int

    @property
    def size(self) -> int:
        return self.end - self.begin


def contiguous_shard(n: int, world: int, rank: int) -> Shard:
    """[n*rank/world, n*(rank+1)/world) — the split rule of attention.hpp:380-381."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of world {world}")
    return Shard(n * rank // world, n * (rank + 1) // world)


def unit_shard(n_requests: int, n_kv_heads: int, world: int, rank: int) -> Shard:
    """Units (request-major: unit = request * n_kv_heads + head) owned by `rank`.
    When the KV heads divide evenly across ranks every rank serves all requests
    for its heads (config 4); otherwise units are split contiguously."""
    n_units = n_requests * n_kv_heads
    return contiguous_shard(n_units, world, rank)


def heads_of_rank(n_kv_heads: int, world: int, rank: int) -> Shard:
    """KV heads owned by `rank` when sharding by head (config 4: 8/N heads per GPU,
    every request)."""
    if n_kv_heads % world:
        raise ValueError(f"{n_kv_heads} KV heads do not split over {world} ranks")
    return contiguous_shard(n_kv_heads, world, rank)


def sequence_shard(n_blocks: int, world: int, rank: int) -> Shard:
    """Blocks of every KV head owned by `rank` in the sequence split (config 5)."""
    return contiguous_shard(n_blocks, world, rank)


def gather_partials(partial, group=None):
    """All-gather one packed SplitPartial per rank: partial [units, gqa, d+2] ->
    [world, units, gqa, d+2] in rank order (= block order of the shards)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group) if dist.is_available() and dist.is_initialized() else 1
    if world == 1:
        return partial.unsqueeze(0)
    partial = partial.contiguous()
    if dist.get_backend(group) == "nccl":
        out = torch.empty((world, *partial.shape), dtype=partial.dtype, device=partial.device)
        dist.all_gather_into_tensor(out, partial, group=group)
        return out
    parts = [torch.empty_like(partial) for _ in range(world)]  # gloo (CPU tests)
    dist.all_gather(parts, partial, group=group)
    return torch.stack(parts)


def sequence_split_decode(q, k_shard, v_shard, *, is_last: bool, k_tail=None, v_tail=None,
                          scale: float | None = None, group=None):
    """decode_attention (attention.hpp:360-409) over a sequence split across ranks.

    k_shard / v_shard: this rank's DeviceCompressedCache of its own block range
    (every unit), q: [units, gqa, d].  Returns the normalised output
    [units, gqa, d] fp32 on every rank."""
    from . import hierasparse as hs
    partial = hs.decode_partial(q, k_shard, v_shard, 0, k_shard.logical_blocks,
                                k_tail if is_last else None, v_tail if is_last else None,
                                include_tail=is_last, scale=scale)
    return hs.decode_combine(gather_partials(partial, group))
