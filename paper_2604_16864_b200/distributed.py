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
  uses for its splits (attention.hpp:380-381) — stores only that shard, and
  produces the unnormalised SplitPartial (O, m, l) of attend_range over it
  (attention.hpp:249-304, :65-69).  One all-gather of the packed partials
  (units x gqa x (d+2) fp32, 16.6 KB at 8 heads x GQA 4) and the reference's
  LSE combine (attention.hpp:387-407) finish the step; only the last rank
  carries the dense tail (attention.hpp:383).

  Compressing a shard is not compressing the whole sequence: select_blocks
  ranks losses across the whole cache (pruner.hpp:94-117) and the sink /
  window protection sits at its two ends (:127-131).  prune_cache_sharded
  therefore computes the block losses of its own shard on the device, gathers
  every rank's losses (nb doubles per unit, one all-gather), runs the global
  selection on the device and compresses its blocks under its slice of the
  global BlockMask — the same pools, index maps and flags as prune_cache of the
  whole sequence, sliced by block range.  (Compressing each shard on its own
  with prune_cache matches this only at S = 0 or 1 without protection.)

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


def gather_block_losses(local_losses, n_blocks: int, group=None):
    """All-gather every rank's block losses [units, shard blocks] (float64) into the
    whole sequence's [units, n_blocks] in block order (shards of
    sequence_shard(n_blocks, world, r) may differ by one block: padded)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group) if dist.is_available() and dist.is_initialized() else 1
    if world == 1:
        return local_losses
    U = local_losses.shape[0]
    width = max(contiguous_shard(n_blocks, world, r).size for r in range(world))
    padded = torch.zeros((U, width), dtype=local_losses.dtype, device=local_losses.device)
    padded[:, :local_losses.shape[1]] = local_losses
    if dist.get_backend(group) == "nccl":
        out = torch.empty((world, U, width), dtype=padded.dtype, device=padded.device)
        dist.all_gather_into_tensor(out, padded, group=group)
        parts = list(out)
    else:
        parts = [torch.empty_like(padded) for _ in range(world)]  # gloo (CPU tests)
        dist.all_gather(parts, padded, group=group)
    return torch.cat([parts[r][:, :contiguous_shard(n_blocks, world, r).size] for r in range(world)], dim=1)


def prune_cache_sharded(key_shard, value_shard, cfg, n_blocks: int, group=None):
    """prune_cache (pruner.hpp:165-176) + fused_magnitude_compress of the whole
    sequence, for this rank's shard only (see the module docstring).

    key_shard / value_shard: [units, shard rows, d] on this rank's GPU, the
    blocks of sequence_shard(n_blocks, world, rank).  Returns (k_cache,
    v_cache, k_flags, v_flags): the shard's compressed caches (pools sized per
    unit for decode) and the global BlockMasks [units, n_blocks]."""
    import torch.distributed as dist
    from . import capi
    from . import hierasparse as hs
    world = dist.get_world_size(group) if dist.is_available() and dist.is_initialized() else 1
    rank = dist.get_rank(group) if world > 1 else 0
    sh = sequence_shard(n_blocks, world, rank)
    if key_shard.shape[1] != sh.size * cfg.block_size:
        raise hs.ConfigError(f"prune_cache_sharded: rank {rank} holds {key_shard.shape[1]} rows, its shard is "
                             f"{sh.size} blocks of {cfg.block_size}")
    out = []
    for x, s, axis in ((key_shard, cfg.s_key, capi.AXIS_CHANNEL), (value_shard, cfg.s_value, capi.AXIS_SEQUENCE)):
        losses = gather_block_losses(hs.block_losses(x, cfg, axis), n_blocks, group)
        flags = hs.select_blocks(losses, cfg, s)
        cache = hs.fused_magnitude_compress(x, flags[:, sh.begin:sh.end], cfg, axis, capacity=True)
        out.append((cache, flags))
    return out[0][0], out[1][0], out[0][1], out[1][1]
