"""The `.hsc` cache container (container.hpp:16-270) for device-resident pools.

`serialize` / `parse` / `save_cache` / `load_cache` keep the reference's format
byte for byte: magic "HSPARSE\\0", version 1, a 38-byte little-endian header
(container.hpp:42), then four u64-length-prefixed sections — index map, dense
pool, nnz pool, metadata — with pool scalars as IEEE binary16 (elem_width_tag 1)
and the same validation order and DataError conditions on parse
(container.hpp:150-250).  One container holds one unit (one CompressedCache).

fp16 device pools are written as their own bits.  bf16 pools are converted value
by value to binary16 with round-to-nearest-even, exactly as the reference's
float_to_half_bits (fp16.hpp:14) converts the same values.  Passing
`native_bf16=True` instead writes elem_width_tag 2 with the raw bf16 bits, a
lossless extension that the reference's parser rejects (tag != 1).
"""
from __future__ import annotations

import struct
from dataclasses import dataclass

import numpy as np

from .errors import ConfigError, DataError, IoError

MAGIC = b"HSPARSE\0"
VERSION = 1
ELEM_HALF, ELEM_BF16 = 1, 2
HEADER_BYTES = 8 + 2 + 5 * 4 + 4 * 2  # kContainerHeaderBytes, container.hpp:42
MAX_POOL_BLOCKS = 32767                # compressed_cache.hpp:116


@dataclass
class HostCache:
    """One unit of a compressed cache on the host, pools as raw 16-bit storage."""

    axis: int              # 0 channel (key), 1 sequence (value)
    head_dim: int
    block_size: int
    logical_blocks: int
    dense_count: int
    sparse_count: int
    index_map: np.ndarray  # int16 [nb]
    dense_pool: np.ndarray  # uint16 [dense * B * d] (bits of elem_tag's type)
    nnz_pool: np.ndarray    # uint16 [sparse * B * d / 2]
    meta_pool: np.ndarray   # uint16 [sparse * B * d / 16]
    elem_tag: int = ELEM_HALF


def _bf16_to_f16_bits(b: np.ndarray) -> np.ndarray:
    """bf16 bits -> binary16 bits, RNE (fp16.hpp:14-62 on the same values)."""
    f = (b.astype(np.uint32) << 16).view(np.float32)
    return f.astype(np.float16).view(np.uint16)  # numpy's float32->float16 cast is IEEE RNE


def serialize(c: HostCache) -> bytes:
    """serialize (container.hpp:119-148)."""
    out = bytearray(MAGIC)
    out += struct.pack("<H5I4H", VERSION, c.block_size, c.head_dim, c.logical_blocks, c.dense_count,
                       c.sparse_count, 2, 4, c.elem_tag, c.axis)
    for arr in (c.index_map.astype(np.int16).view(np.uint16), c.dense_pool, c.nnz_pool, c.meta_pool):
        a = np.ascontiguousarray(arr, dtype="<u2")
        out += struct.pack("<Q", a.size * 2)
        out += a.tobytes()
    return bytes(out)


def parse(data: bytes, allow_bf16: bool = True) -> HostCache:
    """parse (container.hpp:150-250): the same checks, in the same order."""
    pos = 0

    def need(n, what):
        if len(data) - pos < n:
            raise DataError(f"container truncated at offset {pos} while reading {what}")

    need(8, "magic")
    if data[:8] != MAGIC:
        raise DataError("container magic mismatch: not a cache container")
    pos = 8
    fields = []
    for name, fmt in (("version", "<H"), ("block_size", "<I"), ("head_dim", "<I"), ("logical_blocks", "<I"),
                      ("dense_count", "<I"), ("sparse_count", "<I"), ("n_keep", "<H"), ("m_group", "<H"),
                      ("elem_width_tag", "<H"), ("axis_tag", "<H")):
        n = struct.calcsize(fmt)
        need(n, name)
        fields.append(struct.unpack_from(fmt, data, pos)[0])
        pos += n
        if name == "version" and fields[0] != VERSION:
            raise DataError(f"unsupported container version {fields[0]}")
    _, B, d, nb, dense, sparse, n_keep, m_group, tag, axis = fields
    if tag != ELEM_HALF and not (allow_bf16 and tag == ELEM_BF16):
        raise DataError(f"unsupported element width tag {tag}")
    if axis > 1:
        raise DataError(f"unsupported axis tag {axis}")
    if not (n_keep == 2 and m_group == 4):
        raise DataError(f"container: unsupported N:M pattern {n_keep}:{m_group}")
    if B == 0 or d == 0:
        raise DataError("container: zero block_size or head_dim")
    if B % m_group:
        raise DataError("container: block_size not divisible by m_group")
    if axis == 0 and d % m_group:
        raise DataError("container: channel-grouped head_dim not divisible by m_group")
    if dense + sparse != nb:
        raise DataError("container: pool counts do not sum to logical blocks")
    if dense > MAX_POOL_BLOCKS or sparse > MAX_POOL_BLOCKS:
        raise DataError("container: pool count exceeds int16 index capacity")
    be = B * d
    sections = []
    for name, items in (("index_map", nb), ("dense_pool", dense * be), ("nnz_pool", sparse * be // 2),
                        ("meta_pool", sparse * ((be // 4 * 2 + 7) // 8))):
        at = pos
        need(8, name)
        ln = struct.unpack_from("<Q", data, pos)[0]
        pos += 8
        if ln != items * 2:
            raise DataError(f"container section '{name}' at offset {at} declares {ln} bytes, expected {items * 2}")
        need(items * 2, name)
        sections.append(np.frombuffer(data, dtype="<u2", count=items, offset=pos).copy())
        pos += items * 2
    if pos != len(data):
        raise DataError(f"container holds {len(data) - pos} trailing bytes after the last section")
    index_map = sections[0].view(np.int16)
    dense_seen = np.zeros(dense, bool)
    sparse_seen = np.zeros(sparse, bool)
    for b, e in enumerate(index_map.tolist()):
        if e == 0:
            raise DataError(f"container: index map entry {b} is zero")
        slot = abs(e) - 1
        seen = dense_seen if e > 0 else sparse_seen
        if slot >= seen.size:
            raise DataError(f"container: index map entry {b} points past its pool")
        if seen[slot]:
            raise DataError(f"container: pool slot referenced twice by entry {b}")
        seen[slot] = True
    return HostCache(axis, d, B, nb, dense, sparse, index_map, sections[1], sections[2], sections[3], tag)


def host_cache(axis: int, head_dim: int, block_size: int, index_map, dense_bits, nnz_bits, meta, bf16: bool,
               native_bf16: bool = False) -> HostCache:
    """A HostCache from 16-bit storage arrays (bf16 pools converted to binary16
    unless native_bf16)."""
    im = np.asarray(index_map, np.int16)
    dense, nnz = np.asarray(dense_bits, np.uint16), np.asarray(nnz_bits, np.uint16)
    tag = ELEM_HALF
    if bf16 and not native_bf16:
        dense, nnz = _bf16_to_f16_bits(dense), _bf16_to_f16_bits(nnz)
    elif bf16:
        tag = ELEM_BF16
    dc = int((im > 0).sum())
    return HostCache(axis, head_dim, block_size, im.size, dc, im.size - dc, im, dense, nnz,
                     np.asarray(meta, np.uint16), tag)


def from_device(cache, unit: int = 0, native_bf16: bool = False) -> HostCache:
    """One unit of a DeviceCompressedCache as a HostCache in container storage."""
    import torch
    u16 = lambda t: t[unit].contiguous().view(torch.int16).cpu().numpy().view(np.uint16).reshape(-1)  # noqa: E731
    dense = u16(cache.dense_pool) if cache.dense_count else np.zeros(0, np.uint16)
    nnz = u16(cache.nnz_pool) if cache.sparse_count else np.zeros(0, np.uint16)
    meta = u16(cache.meta_pool) if cache.sparse_count else np.zeros(0, np.uint16)
    return host_cache(cache.axis, cache.head_dim, cache.block_size, cache.index_map[unit].cpu().numpy(), dense, nnz,
                      meta, cache.dtype == torch.bfloat16, native_bf16)


def to_device(hc: HostCache, device=None):
    """A one-unit DeviceCompressedCache from a HostCache (fp16 for tag 1, bf16 for tag 2).
    slot_block and the BlockMask flags are rebuilt from the index map."""
    import torch
    from .hierasparse import DeviceCompressedCache
    if hc.head_dim != 128 or hc.block_size != 64:
        raise ConfigError("device kernels take head_dim 128 and block_size 64")
    dt = torch.float16 if hc.elem_tag == ELEM_HALF else torch.bfloat16
    c = DeviceCompressedCache(dt, hc.axis, 1, hc.logical_blocks, hc.dense_count, hc.sparse_count, device)
    t16 = lambda a: torch.from_numpy(a.astype(np.uint16).view(np.int16).copy())  # noqa: E731
    c.index_map.copy_(torch.from_numpy(hc.index_map.astype(np.int16)).reshape(1, -1))
    if hc.dense_count:
        c.dense_pool.view(torch.int16).copy_(t16(hc.dense_pool).reshape(c.dense_pool.shape))
    if hc.sparse_count:
        c.nnz_pool.view(torch.int16).copy_(t16(hc.nnz_pool).reshape(c.nnz_pool.shape))
        c.meta_pool.copy_(t16(hc.meta_pool).reshape(c.meta_pool.shape))
    im = hc.index_map.astype(np.int64)
    slot_block = np.empty(hc.logical_blocks, np.int32)
    dense_b, sparse_b = np.nonzero(im > 0)[0], np.nonzero(im < 0)[0]
    slot_block[im[dense_b] - 1] = dense_b
    slot_block[hc.dense_count + (-im[sparse_b] - 1)] = sparse_b
    c.slot_block.copy_(torch.from_numpy(slot_block).reshape(1, -1))
    c.flags.copy_(torch.from_numpy((im > 0).astype(np.uint8)).reshape(1, -1))
    c.losses.fill_(float("nan"))
    return c


def save_cache(path: str, cache, unit: int = 0, native_bf16: bool = False) -> None:
    """save_cache (container.hpp:252-259)."""
    data = serialize(from_device(cache, unit, native_bf16))
    try:
        with open(path, "wb") as f:
            f.write(data)
    except OSError as e:
        raise IoError(f"cannot open '{path}' for writing: {e}") from e


def load_cache(path: str, device=None):
    """load_cache (container.hpp:261-270) -> one-unit DeviceCompressedCache."""
    try:
        with open(path, "rb") as f:
            data = f.read()
    except OSError as e:
        raise IoError(f"cannot open '{path}' for reading: {e}") from e
    return to_device(parse(data), device)
