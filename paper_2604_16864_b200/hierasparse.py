"""Host-side mirror of the reference's hot-path API over device-resident caches.

Same names and argument meaning as /root/reference/proj/include/hierasparse
(prune_cache, fused_magnitude_compress, decompress, decode_attention,
prefill_attention, measure_size, flop_and_byte_count), batched over "units"
(request, KV-head pairs).  PyTorch only provides device memory and the current
stream; every computation runs in the sm_100a kernels behind the C ABI
(include/hierasparse_b200.h) — there is no CPU or eager fallback.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

import torch

from . import capi
from .errors import ConfigError, DataError  # noqa: F401  (re-exported for callers)

BLOCK = 64
HEAD_DIM = 128
HEADER_BYTES = 8 + 2 + 5 * 4 + 4 * 2  # container.hpp:42 kContainerHeaderBytes


def _dtype_code(dt: torch.dtype) -> int:
    if dt == torch.bfloat16:
        return capi.DTYPE_BF16
    if dt == torch.float16:
        return capi.DTYPE_F16
    raise ConfigError(f"unsupported dtype {dt}: device kernels take bfloat16 or float16")


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def _LIB():
    return capi._lib if capi._lib is not None else capi.load()


def _ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None or t.numel() == 0 else t.data_ptr()


@dataclass
class SparsityConfig:
    """masks.hpp:73-99 (2:4 pattern)."""

    s_key: float = 0.0
    s_value: float = 0.0
    block_size: int = BLOCK
    sink_tokens: int = 0
    local_window: int = 0

    def c(self) -> capi.SparsityConfigC:
        return capi.SparsityConfigC(self.s_key, self.s_value, self.block_size, 0, self.sink_tokens,
                                    self.local_window)

    def protected_prefix_blocks(self) -> int:
        return (self.sink_tokens + self.block_size - 1) // self.block_size

    def protected_suffix_blocks(self) -> int:
        return (self.local_window + self.block_size - 1) // self.block_size


def pool_counts(rows: int, cfg: SparsityConfig, sparsity: float):
    """(logical_blocks, dense_count, sparse_count, prefix, suffix) before any data is seen
    (pruner.hpp:106-108, :127-131)."""
    lib = capi.load()
    out = [C.c_uint32() for _ in range(5)]
    c = cfg.c()
    capi.check(lib.hs_pool_counts(rows, C.byref(c), sparsity, *[C.byref(o) for o in out]))
    return tuple(o.value for o in out)


class DeviceCompressedCache:
    """CompressedCache (compressed_cache.hpp:37-110) for n_units units on one GPU,
    in the reference's canonical layout (see include/hierasparse_b200.h)."""

    def __init__(self, dtype: torch.dtype, axis: int, n_units: int, logical_blocks: int,
                 dense_count: int, sparse_count: int, device=None, head_dim: int = HEAD_DIM,
                 block_size: int = BLOCK, cfg: SparsityConfig | None = None):
        dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.dtype, self.axis, self.n_units = dtype, axis, n_units
        self.head_dim, self.block_size = head_dim, block_size
        self.logical_blocks, self.dense_count, self.sparse_count = logical_blocks, dense_count, sparse_count
        self.cfg = cfg
        be = block_size * head_dim
        U = n_units
        self.index_map = torch.empty((U, logical_blocks), dtype=torch.int16, device=dev)
        self.dense_pool = torch.empty((U, dense_count, be), dtype=dtype, device=dev)
        self.nnz_pool = torch.empty((U, sparse_count, be // 2), dtype=dtype, device=dev)
        self.meta_pool = torch.empty((U, sparse_count, be // 16), dtype=torch.int16, device=dev)
        self.slot_block = torch.empty((U, logical_blocks), dtype=torch.int32, device=dev)
        self.flags = torch.empty((U, logical_blocks), dtype=torch.uint8, device=dev)
        # block losses of the last selection that computed them (NaN: not computed --
        # a static selection needs none unless asked for, with_losses=True)
        self.losses = torch.full((U, logical_blocks), float("nan"), dtype=torch.float64, device=dev)

    @property
    def sequence_length(self) -> int:
        return self.logical_blocks * self.block_size

    def c(self) -> capi.DeviceCacheC:
        """The C-ABI descriptor (built once; the pool tensors never move)."""
        cs = getattr(self, "_c_struct", None)
        if cs is None:
            cs = capi.DeviceCacheC(_dtype_code(self.dtype), self.axis, self.head_dim, self.block_size,
                                   self.n_units, self.logical_blocks, self.dense_count, self.sparse_count,
                                   _ptr(self.index_map), _ptr(self.dense_pool), _ptr(self.nnz_pool),
                                   _ptr(self.meta_pool), _ptr(self.slot_block))
            self._c_struct = cs
            self._c_ref = C.byref(cs)
        return cs

    def cref(self):
        self.c()
        return self._c_ref

    def measure_size(self) -> dict:
        """measure_size (compressed_cache.hpp:303-310), per unit."""
        be = self.block_size * self.head_dim
        return dict(size_idx=self.logical_blocks * 2, size_den=self.dense_count * be * 2,
                    size_nnz=self.sparse_count * (be // 2) * 2, size_e=self.sparse_count * (be // 16) * 2)

    def nbytes(self) -> int:
        """Bytes a full traversal of every unit reads (pools + index map): the sum of
        measure_size over units (per-unit counts when units differ)."""
        counts = getattr(self, "unit_dense_counts", None)
        if counts is None:
            return self.n_units * sum(self.measure_size().values())
        be = self.block_size * self.head_dim
        return sum(self.logical_blocks * 2 + c * be * 2 + (self.logical_blocks - c) * (be // 2 + be // 8)
                   for c in counts)


class StatusWord:
    """A device status word (hierasparse_b200.h "status words"): the kernels that
    validate data record the first DataError in the reference's order into it
    without a host synchronisation.  check() synchronises and raises it."""

    def __init__(self, device):
        self.word = torch.zeros(1, dtype=torch.int64, device=device)

    def ptr(self) -> int:
        return self.word.data_ptr()

    def check(self) -> None:
        capi.check_status_word(int(self.word.item()))


def _status(status: StatusWord | None, device) -> StatusWord:
    return status if status is not None else StatusWord(device)


def _check_src(x: torch.Tensor) -> torch.Tensor:
    if not x.is_cuda:
        raise ConfigError("source must be a CUDA tensor (use the host-buffer entry points for host data)")
    if x.dim() == 2:
        x = x.unsqueeze(0)
    if x.dim() != 3:
        raise ConfigError("source must be [units, rows, head_dim]")
    if x.stride(2) != 1 or x.stride(1) != x.shape[2] or (x.shape[0] > 1 and x.stride(0) < x.shape[1] * x.shape[2]):
        x = x.contiguous()
    return x


def _unit_stride(x: torch.Tensor) -> int:
    return x.stride(0) if x.shape[0] > 1 else x.shape[1] * x.shape[2]


def _static_selection(nb: int, sc: int, prefix: int, suffix: int) -> bool:
    """select_blocks' quota is 0 or every prunable block (pruner.hpp:106-116): the
    block mask follows from the protected regions alone, no loss is consulted."""
    return sc == 0 or sc == nb - prefix - suffix


def prune_compress(x: torch.Tensor, cfg: SparsityConfig, sparsity: float, axis: int,
                   out: DeviceCompressedCache | None = None, with_losses: bool = True) -> DeviceCompressedCache:
    """hierarchical_mask_for (pruner.hpp:121-158) + fused_magnitude_compress
    (compressed_cache.hpp:232-267) for one cache kind of every unit.  The block
    losses (pruner.hpp:81-89) land in out.losses; with_losses=False skips them when
    the selection does not need them (quota 0 or all prunable blocks)."""
    x = _check_src(x)
    U, rows, d = x.shape
    nb, dc, sc, pre, suf = pool_counts(rows, cfg, sparsity)
    if out is None:
        out = DeviceCompressedCache(x.dtype, axis, U, nb, dc, sc, x.device, d, cfg.block_size, cfg)
    elif (out.n_units, out.logical_blocks, out.dense_count, out.sparse_count, out.dtype, out.axis, out.head_dim) != \
            (U, nb, dc, sc, x.dtype, axis, d):
        raise ConfigError("prune_cache: the output cache's geometry does not match")
    lib = capi.load()
    cc = cfg.c()
    lp = out.losses.data_ptr() if with_losses or not _static_selection(nb, sc, pre, suf) else None
    capi.check(lib.hs_prune_compress(x.data_ptr(), _unit_stride(x), rows, C.byref(cc), sparsity, out.cref(),
                                     lp, out.flags.data_ptr(), _stream()))
    return out


def prune_cache(key: torch.Tensor, value: torch.Tensor, cfg: SparsityConfig, out=None, with_losses: bool = False):
    """prune_cache (pruner.hpp:165-176) followed by compression of both caches:
    key along channels at S_K, value along the sequence at S_V.  out: an earlier
    (key, value) result of the same geometry to overwrite (no allocation).  Like
    the reference's HierarchicalMask (block + element masks, no losses), block
    losses are computed only when the selection ranks them, unless with_losses."""
    if key.shape[-2] != value.shape[-2]:
        raise ConfigError("prune_cache: key/value sequence lengths differ")
    if key.shape[-1] % 4:
        raise ConfigError("prune_cache: head dimension not divisible by m_group")
    ko, vo = out if out is not None else (None, None)
    if not (key.is_cuda and value.is_cuda):
        return (prune_compress(key, cfg, cfg.s_key, capi.AXIS_CHANNEL, ko, with_losses),
                prune_compress(value, cfg, cfg.s_value, capi.AXIS_SEQUENCE, vo, with_losses))
    # The two caches are independent: the value cache runs on a side stream (forked
    # from and joined back into the caller's stream), so one cache's selection
    # kernels -- a CTA per unit -- overlap the other cache's block kernels.  Both
    # outputs are allocated on the caller's stream before the fork.
    if vo is None:
        vo = _alloc_cache(value, cfg, cfg.s_value, capi.AXIS_SEQUENCE)
    main = torch.cuda.current_stream(key.device)
    side = _side_stream(key.device)
    side.wait_stream(main)
    kc = prune_compress(key, cfg, cfg.s_key, capi.AXIS_CHANNEL, ko, with_losses)
    with torch.cuda.stream(side):
        vc = prune_compress(value, cfg, cfg.s_value, capi.AXIS_SEQUENCE, vo, with_losses)
    main.wait_stream(side)
    return kc, vc


_SIDE_STREAMS: dict = {}


def _side_stream(device) -> "torch.cuda.Stream":
    idx = device.index if device.index is not None else torch.cuda.current_device()
    if idx not in _SIDE_STREAMS:
        _SIDE_STREAMS[idx] = torch.cuda.Stream(device=idx)
    return _SIDE_STREAMS[idx]


def _alloc_cache(x: torch.Tensor, cfg: SparsityConfig, sparsity: float, axis: int) -> DeviceCompressedCache:
    U, rows, d = (x.shape if x.dim() == 3 else (1, *x.shape))
    nb, dc, sc, _, _ = pool_counts(rows, cfg, sparsity)
    return DeviceCompressedCache(x.dtype, axis, U, nb, dc, sc, x.device, d, cfg.block_size, cfg)


def block_losses(x: torch.Tensor, cfg: SparsityConfig, axis: int) -> torch.Tensor:
    """block_loss (pruner.hpp:81-89) of every block of every unit (element masks of
    element_mask, :40-77): float64 [units, blocks], bit-identical to the reference."""
    x = _check_src(x)
    U, rows, d = x.shape
    geo = DeviceCompressedCache(x.dtype, axis, U, 0, 0, 0, x.device, d, cfg.block_size)
    if rows % cfg.block_size:
        raise ConfigError("prune_cache: sequence length not divisible by block_size")
    losses = torch.empty((U, rows // cfg.block_size), dtype=torch.float64, device=x.device)
    capi.check(capi.load().hs_block_losses(x.data_ptr(), _unit_stride(x), rows, geo.cref(), losses.data_ptr(),
                                           _stream()))
    return losses


def select_blocks(losses: torch.Tensor, cfg: SparsityConfig, sparsity: float) -> torch.Tensor:
    """select_blocks (pruner.hpp:94-117) with the protected prefix / suffix of
    cfg (masks.hpp:93-98, pruner.hpp:127-131) over losses [units, blocks] on the
    device: u8 flags [units, blocks], 1 = dense."""
    if not losses.is_cuda or losses.dtype != torch.float64 or losses.dim() != 2:
        raise ConfigError("select_blocks: losses must be a CUDA float64 [units, blocks] tensor")
    losses = losses.contiguous()
    U, nb = losses.shape
    flags = torch.empty((U, nb), dtype=torch.uint8, device=losses.device)
    cc = cfg.c()
    capi.check(capi.load().hs_select_blocks(losses.data_ptr(), U, nb, C.byref(cc), sparsity, flags.data_ptr(),
                                            _stream()))
    return flags


def fused_magnitude_compress(x: torch.Tensor, flags: torch.Tensor, cfg: SparsityConfig,
                             axis: int, check: bool = True, status: StatusWord | None = None,
                             capacity: bool = False) -> DeviceCompressedCache:
    """fused_magnitude_compress (compressed_cache.hpp:262-267) under a given BlockMask
    (flags u8 [units, blocks], 1 = dense).  Every unit's dense count must equal
    unit 0's (the pooled layout); a mismatch raises ConfigError (device-checked).
    capacity=True sizes the pools for the largest unit instead (units may differ;
    the result then serves decode only, per-unit counts in .unit_dense_counts)."""
    x = _check_src(x)
    U, rows, d = x.shape
    if rows % cfg.block_size:
        raise ConfigError("compress: sequence length not divisible by block_size")
    flags = flags.to(device=x.device, dtype=torch.uint8).reshape(U, -1).contiguous()
    nb = rows // cfg.block_size
    if flags.shape[1] != nb:
        raise ConfigError("compress: block mask does not cover the sequence")
    if capacity:
        # per-unit dense counts may differ (a shard of a globally selected
        # sequence): pools sized for the largest unit, decode-only
        counts = (flags != 0).sum(dim=1).cpu() if nb else torch.zeros(U, dtype=torch.int64)
        dc, sc = int(counts.max().item()) if U else 0, int((nb - counts).max().item()) if U else 0
    else:
        dc = int((flags[0] != 0).sum().item()) if nb else 0
        sc = nb - dc
    out = DeviceCompressedCache(x.dtype, axis, U, nb, dc, sc, x.device, d, cfg.block_size, cfg)
    if capacity:
        out.unit_dense_counts = [int(c) for c in counts]
    st = _status(status, x.device)
    capi.check(capi.load().hs_compress_with_flags(x.data_ptr(), _unit_stride(x), rows, flags.data_ptr(),
                                                  out.cref(), st.ptr(), _stream()))
    out.flags.copy_(flags != 0)
    out.status = st
    if check:
        st.check()
    return out


def compress(x: torch.Tensor, element_mask: torch.Tensor, flags: torch.Tensor, cfg: SparsityConfig, axis: int,
             check: bool = True, status: StatusWord | None = None) -> DeviceCompressedCache:
    """compress (compressed_cache.hpp:196-225): pack under an explicit HierarchicalMask
    -- element_mask (bool/u8 [units, rows, d], nonzero = kept) and BlockMask flags
    (u8 [units, blocks], 1 = dense).  Dense blocks are copied verbatim; every 2:4
    group of a sparse block must keep exactly 2 elements, else DataError
    ("compress: group keeps more / fewer than n_keep elements")."""
    x = _check_src(x)
    U, rows, d = x.shape
    em = element_mask.to(device=x.device, dtype=torch.uint8).reshape(U, rows, d).contiguous()
    if em.shape != x.shape:
        raise ConfigError("compress: element mask shape mismatch")
    if rows % cfg.block_size:
        raise ConfigError("compress: sequence length not divisible by block_size")
    flags = flags.to(device=x.device, dtype=torch.uint8).reshape(U, -1).contiguous()
    nb = rows // cfg.block_size
    if flags.shape[1] != nb:
        raise ConfigError("compress: block mask does not cover the sequence")
    dc = int((flags[0] != 0).sum().item()) if nb else 0
    out = DeviceCompressedCache(x.dtype, axis, U, nb, dc, nb - dc, x.device, d, cfg.block_size, cfg)
    st = _status(status, x.device)
    capi.check(capi.load().hs_compress_with_mask(x.data_ptr(), _unit_stride(x), rows, em.data_ptr(), rows * d,
                                                 flags.data_ptr(), out.cref(), st.ptr(), _stream()))
    out.flags.copy_(flags != 0)
    out.status = st
    if check:
        st.check()
    return out


def decompress(c: DeviceCompressedCache, check: bool = True, status: StatusWord | None = None) -> torch.Tensor:
    """decompress (compressed_cache.hpp:271-298) -> [units, rows, d].  Corrupt
    index maps / metadata raise DataError (check=True: synchronises to read the
    status word; check=False: the word is left on the result as .status)."""
    out = torch.empty((c.n_units, c.sequence_length, c.head_dim), dtype=c.dtype, device=c.index_map.device)
    st = _status(status, out.device)
    capi.check(capi.load().hs_decompress(c.cref(), out.data_ptr(), st.ptr(), _stream()))
    if check:
        st.check()
    return out


def recompress(c: DeviceCompressedCache, cfg: SparsityConfig, sparsity: float, check: bool = True,
               status: StatusWord | None = None, with_losses: bool = False) -> DeviceCompressedCache:
    """The decode-phase re-prune (pipeline.hpp:227-240): decompress
    (compressed_cache.hpp:271-298) -> hierarchical_mask_for at the decode sparsity
    (pruner.hpp:121-158) -> fused_magnitude_compress, for every unit on the
    device, in one pass over the input pools (hs_recompress: blocks are expanded
    on the fly, the dense cache is never materialised).  Bit-identical to the
    reference's chain on the same pools.  A corrupt input cache raises
    decompress's DataError (check=False defers it to out.status.check(), so the
    call stays free of host synchronisation, e.g. inside a CUDA graph).  Block
    losses only when the selection ranks them, unless with_losses (as prune_cache)."""
    return _recompress_into(c, cfg, sparsity, _recompress_out(c, cfg, sparsity), check, status, with_losses)


def _recompress_out(c: DeviceCompressedCache, cfg: SparsityConfig, sparsity: float) -> DeviceCompressedCache:
    nb, dc, sc, _, _ = pool_counts(c.logical_blocks * c.block_size, cfg, sparsity)
    return DeviceCompressedCache(c.dtype, c.axis, c.n_units, nb, dc, sc, c.index_map.device, c.head_dim,
                                 cfg.block_size, cfg)


def _recompress_into(c, cfg, sparsity, out, check, status, with_losses=False):
    cc = cfg.c()
    st = _status(status, out.index_map.device)
    nb, _, sc, pre, suf = pool_counts(c.logical_blocks * c.block_size, cfg, sparsity)
    lp = out.losses.data_ptr() if with_losses or not _static_selection(nb, sc, pre, suf) else None
    capi.check(capi.load().hs_recompress(c.cref(), C.byref(cc), sparsity, out.cref(), lp,
                                         out.flags.data_ptr(), st.ptr(), _stream()))
    out.status = st
    if check:
        st.check()
    return out


def absorb_tail(c: DeviceCompressedCache, tail: torch.Tensor, cfg: SparsityConfig, sparsity: float,
                check: bool = True, status: StatusWord | None = None, with_losses: bool = False):
    """Dense-tail growth during decode: once the dense tail
    (CacheView::dense_tail, attention.hpp:19-31) holds whole blocks, re-prune the
    cache over its blocks followed by those tail blocks -- prune_cache + compress
    of [decompress(c); tail blocks] -- in one pass (hs_absorb_tail).  tail:
    [units, T, d] tokens after the cache.  Returns (cache, remaining tail of
    T % block_size tokens); with no whole block the inputs come back unchanged.
    Block losses only when the selection ranks them, unless with_losses (as prune_cache)."""
    U, d, B = c.n_units, c.head_dim, c.block_size
    tail = tail.reshape(U, -1, d)
    full = (tail.shape[1] // B) * B
    if full == 0:
        return c, tail
    if tail.dtype != c.dtype:
        raise ConfigError("absorb_tail: tail dtype differs from the cache")
    if tail.stride(2) != 1 or tail.stride(1) != d:
        tail = tail.contiguous()
    src = tail[:, :full]  # unit stride = the whole tail's; rows contiguous
    rows = c.logical_blocks * B + full
    nb, dc, sc, pre, suf = pool_counts(rows, cfg, sparsity)
    out = DeviceCompressedCache(c.dtype, c.axis, U, nb, dc, sc, c.index_map.device, d, cfg.block_size, cfg)
    cc = cfg.c()
    st = _status(status, out.index_map.device)
    lp = out.losses.data_ptr() if with_losses or not _static_selection(nb, sc, pre, suf) else None
    capi.check(capi.load().hs_absorb_tail(c.cref(), src.data_ptr(), _unit_stride(src), full, C.byref(cc),
                                          sparsity, out.cref(), lp, out.flags.data_ptr(),
                                          st.ptr(), _stream()))
    out.status = st
    if check:
        st.check()
    return out, tail[:, full:]


def absorb_tail_pair(k: DeviceCompressedCache, v: DeviceCompressedCache, k_tail: torch.Tensor,
                     v_tail: torch.Tensor, cfg: SparsityConfig, with_losses: bool = False):
    """absorb_tail for the key (S_K, channel groups) and value (S_V, sequence groups) caches."""
    k2, kt = absorb_tail(k, k_tail, cfg, cfg.s_key, with_losses=with_losses)
    v2, vt = absorb_tail(v, v_tail, cfg, cfg.s_value, with_losses=with_losses)
    return k2, v2, kt, vt


def recompress_unfused(c: DeviceCompressedCache, cfg: SparsityConfig, sparsity: float) -> DeviceCompressedCache:
    """recompress as the reference composes it: decompress to a dense device
    cache, then prune_compress (the parity check for the fused path)."""
    dense = decompress(c)
    out = prune_compress(dense, cfg, sparsity, c.axis)
    del dense
    return out


def recompress_pair(k: DeviceCompressedCache, v: DeviceCompressedCache, cfg: SparsityConfig, check: bool = True,
                    status: StatusWord | None = None, with_losses: bool = False):
    """prune_cache at the decode sparsity (cfg.s_key / cfg.s_value) of already
    compressed caches (pipeline.hpp:228-240, "further pruned").  The
    value cache runs on a side stream forked from and joined into the caller's
    stream (outputs allocated on the caller's stream first), as in prune_cache."""
    st = _status(status, k.index_map.device)
    vo = _recompress_out(v, cfg, cfg.s_value)
    main = torch.cuda.current_stream(k.index_map.device)
    side = _side_stream(k.index_map.device)
    side.wait_stream(main)
    k2 = recompress(k, cfg, cfg.s_key, check=False, status=st, with_losses=with_losses)
    with torch.cuda.stream(side):
        v2 = _recompress_into(v, cfg, cfg.s_value, vo, False, st, with_losses)
    main.wait_stream(side)
    if check:
        st.check()
    return k2, v2


def _tails(k_tail, v_tail, U, d, dtype):
    if k_tail is None or k_tail.numel() == 0:
        return None, None, 0
    for t in (k_tail, v_tail):
        if t is None or not t.is_cuda or t.dtype != dtype:
            raise ConfigError(f"attention: dense tails must be CUDA tensors of the caches' dtype {dtype}")
    k_tail = k_tail.reshape(U, -1, d).contiguous()
    v_tail = v_tail.reshape(U, -1, d).contiguous()
    if k_tail.shape != v_tail.shape:
        raise ConfigError("attention: key/value token counts differ")
    return k_tail, v_tail, k_tail.shape[1]


def _check_queries(q: torch.Tensor, k: DeviceCompressedCache, what: str, host_ok: bool = False) -> None:
    """The device kernels read q as [units, ..., head_dim] of the caches' 16-bit
    dtype: reject anything else instead of reinterpreting its bits.  host_ok: a
    contiguous pinned host tensor is accepted too (read over the host link)."""
    pinned = host_ok and isinstance(q, torch.Tensor) and not q.is_cuda and q.is_pinned() and q.is_contiguous()
    if not isinstance(q, torch.Tensor) or not (q.is_cuda or pinned):
        raise ConfigError(f"{what}: queries must be a CUDA tensor" +
                          (" or a contiguous pinned host tensor" if host_ok else ""))
    if q.dtype != k.dtype:
        raise ConfigError(f"{what}: query dtype {q.dtype} differs from the caches' {k.dtype}")
    if q.dim() < 2 or q.shape[0] != k.n_units or q.shape[-1] != k.head_dim:
        raise ConfigError(f"{what}: queries {tuple(q.shape)} do not match {k.n_units} units x head_dim "
                          f"{k.head_dim}")


def _tail_only_view(k, v, k_tail, v_tail, q, what):
    """CacheView{compressed = nullptr, dense_tail} (attention.hpp:22-31): the
    attention runs over the tail alone, through zero-block caches."""
    if k is not None and v is not None:
        return k, v
    if k is not None or v is not None:
        raise ConfigError(f"{what}: key and value caches must both be given or both be None")
    if k_tail is None or k_tail.numel() == 0:
        raise ConfigError(f"{what}: empty key/value cache")
    U = q.shape[0]
    d = k_tail.shape[-1]
    ke = DeviceCompressedCache(k_tail.dtype, capi.AXIS_CHANNEL, U, 0, 0, 0, k_tail.device, d)
    ve = DeviceCompressedCache(k_tail.dtype, capi.AXIS_SEQUENCE, U, 0, 0, 0, k_tail.device, d)
    return ke, ve


def decode_attention(q: torch.Tensor, k: DeviceCompressedCache | None, v: DeviceCompressedCache | None,
                     k_tail: torch.Tensor | None = None, v_tail: torch.Tensor | None = None,
                     scale: float | None = None, splits: int = 0,
                     out: torch.Tensor | None = None) -> torch.Tensor:
    """decode_attention (attention.hpp:360-409) for every unit: q [units, gqa, d] -> fp32.
    k = v = None attends to the dense tail alone (CacheView without a compressed cache).
    q and out may be contiguous pinned host tensors (zero-copy: the kernel reads q and
    writes out over the host link; out is complete once the stream synchronises)."""
    k, v = _tail_only_view(k, v, k_tail, v_tail, q, "decode_attention")
    _check_queries(q, k, "decode_attention", host_ok=True)
    if out is not None and not out.is_cuda and not (out.is_pinned() and out.is_contiguous()):
        raise ConfigError("decode_attention: out must be a CUDA tensor or a contiguous pinned host tensor")
    U = k.n_units
    if q.dim() != 3 or not q.is_contiguous():
        q = q.reshape(U, -1, k.head_dim).contiguous()
    gqa = q.shape[1]
    kt, vt, tail = _tails(k_tail, v_tail, U, k.head_dim, k.dtype)
    scale = 1.0 / math.sqrt(k.head_dim) if scale is None else scale
    if out is None:
        out = torch.empty((U, gqa, k.head_dim), dtype=torch.float32, device=k.index_map.device)
    capi.check(_LIB().hs_decode(q.data_ptr(), k.cref(), v.cref(), _ptr(kt), _ptr(vt), tail, gqa,
                                scale, splits, out.data_ptr(), _stream()))
    return out


class DecodePlan:
    """A decode step captured once as a CUDA graph and replayed per token:
    hs_decode's kernels with fixed caches, query and output buffers (the host
    enqueue cost disappears from the step; inputs are refreshed in place).
    The plan owns its workspace (split partials + arrival counters,
    hs_decode_ws), so replays share no state with other decode work."""

    def __init__(self, q: torch.Tensor, k: DeviceCompressedCache, v: DeviceCompressedCache,
                 scale: float | None = None, splits: int = 0, host_io: bool = False):
        """host_io: the step reads the queries from pinned host memory (self.q_host)
        and writes the output to pinned host memory (self.out_host) directly over
        the host link (zero-copy), so one replay is a whole host-to-host decode
        step: write q_host, replay, synchronise, read out_host."""
        _check_queries(q, k, "DecodePlan")
        self.q = q.contiguous().clone()
        self.k, self.v = k, v
        gqa = self.q.shape[1]
        self.out = torch.empty((k.n_units, gqa, k.head_dim), dtype=torch.float32, device=q.device)
        self.host_io = host_io
        if host_io:
            self.q_host = self.q.cpu().pin_memory()
            self.out_host = torch.empty(self.out.shape, dtype=torch.float32).pin_memory()
        lib = capi.load()
        nbytes = C.c_uint64()
        capi.check(lib.hs_decode_workspace_bytes(k.cref(), gqa, splits, C.byref(nbytes)))
        self.workspace = torch.zeros(int(nbytes.value), dtype=torch.uint8, device=q.device)
        scale = 1.0 / math.sqrt(k.head_dim) if scale is None else scale

        # host_io: zero-copy -- the kernel reads the queries from the pinned (UVA
        # mapped) q_host and the split combine writes O straight into out_host, so
        # the step needs no copy-engine transfers (two small DMAs cost ~16 us).
        qp = self.q_host.data_ptr() if host_io else self.q.data_ptr()
        op = self.out_host.data_ptr() if host_io else self.out.data_ptr()

        def step():
            capi.check(lib.hs_decode_ws(qp, k.cref(), v.cref(), None, None, 0, gqa, scale, splits, op,
                                        self.workspace.data_ptr(), self.workspace.numel(), _stream()))
        # Warm up on the capture stream so the TMA descriptors exist before
        # capture (no allocation may happen inside the graph).
        self.stream = torch.cuda.Stream()
        self.stream.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(self.stream):
            step()
        torch.cuda.synchronize()
        self.graph = torch.cuda.CUDAGraph()
        n0 = capi.kernel_launches()
        with torch.cuda.graph(self.graph, stream=self.stream):
            step()
        torch.cuda.synchronize()
        self.kernels_per_step = capi.kernel_launches() - n0  # native kernels inside the graph

    def __call__(self, q: torch.Tensor | None = None) -> torch.Tensor:
        if q is not None:
            (self.q_host if self.host_io else self.q).copy_(q, non_blocking=not self.host_io)
        self.graph.replay()
        return self.out_host if self.host_io else self.out


def decode_partial(q, k: DeviceCompressedCache, v: DeviceCompressedCache, block_begin: int, block_end: int,
                   k_tail=None, v_tail=None, include_tail: bool = True, scale: float | None = None):
    """attend_range (attention.hpp:249-304) over [block_begin, block_end) as an
    unnormalised SplitPartial per unit: float [units, gqa, d + 2] = (O, m, l)."""
    k, v = _tail_only_view(k, v, k_tail, v_tail, q, "attend_range")
    _check_queries(q, k, "attend_range")
    U = k.n_units
    q = q.reshape(U, -1, k.head_dim).contiguous()
    gqa = q.shape[1]
    kt, vt, tail = _tails(k_tail, v_tail, U, k.head_dim, k.dtype)
    scale = 1.0 / math.sqrt(k.head_dim) if scale is None else scale
    out = torch.empty((U, gqa, k.head_dim + 2), dtype=torch.float32, device=q.device)
    capi.check(capi.load().hs_decode_partial(q.data_ptr(), k.cref(), v.cref(), _ptr(kt), _ptr(vt), tail,
                                             gqa, scale, block_begin, block_end, int(include_tail),
                                             out.data_ptr(), _stream()))
    return out


def decode_combine(partials: torch.Tensor) -> torch.Tensor:
    """LSE combine (attention.hpp:387-407) of partials [parts, units, gqa, d + 2]."""
    if not partials.is_cuda or partials.dtype != torch.float32 or partials.dim() != 4:
        raise ConfigError("decode_combine: partials must be a CUDA float32 [parts, units, gqa, d + 2] tensor")
    partials = partials.contiguous()
    P, U, gqa, d2 = partials.shape
    out = torch.empty((U, gqa, d2 - 2), dtype=torch.float32, device=partials.device)
    capi.check(capi.load().hs_decode_combine(partials.data_ptr(), P, U, gqa, d2 - 2, out.data_ptr(), _stream()))
    return out


def prefill_attention(q: torch.Tensor, k: DeviceCompressedCache | None, v: DeviceCompressedCache | None,
                      k_tail=None, v_tail=None, causal: bool = True, scale: float | None = None,
                      out: torch.Tensor | None = None) -> torch.Tensor:
    """prefill_attention (attention.hpp:323-354): q [units, gqa, n_q, d] -> fp32.
    k = v = None attends to the dense tail alone (CacheView without a compressed cache)."""
    k, v = _tail_only_view(k, v, k_tail, v_tail, q, "prefill_attention")
    _check_queries(q, k, "prefill_attention")
    U = k.n_units
    if q.dim() == 3:
        q = q.unsqueeze(1)
    if q.dim() != 4:
        raise ConfigError("prefill_attention: queries must be [units, gqa, n_q, head_dim]")
    q = q.contiguous()
    _, gqa, n_q, d = q.shape
    kt, vt, tail = _tails(k_tail, v_tail, U, k.head_dim, k.dtype)
    scale = 1.0 / math.sqrt(k.head_dim) if scale is None else scale
    if out is None:
        out = torch.empty((U, gqa, n_q, d), dtype=torch.float32, device=q.device)
    elif out.shape != (U, gqa, n_q, d) or out.dtype != torch.float32 or not out.is_contiguous():
        raise ConfigError("prefill_attention: out must be a contiguous float32 [units, gqa, n_q, head_dim] tensor")
    capi.check(capi.load().hs_prefill(q.data_ptr(), n_q, gqa, k.cref(), v.cref(), _ptr(kt), _ptr(vt), tail,
                                      int(causal), scale, out.data_ptr(), _stream()))
    return out


def flop_count(k_dense, v_dense, block: int, d: int, n_q: int, tail: int = 0, causal: bool = False) -> int:
    """Counted GEMM flops of flop_and_byte_count (attention.hpp:426-456) in closed
    form: per (query row, visible key) 2*d per GEMM on a dense block, d on a
    sparse one, 4*d on the dense tail; causal at row granularity."""
    import numpy as np
    kd = np.asarray(k_dense, dtype=np.int64)
    vd = np.asarray(v_dense, dtype=np.int64)
    nb = kd.shape[0]
    w = (1 + kd) + (1 + vd)                       # per-key flop weight / d
    prefix = nb * block
    n_kv = prefix + tail
    if not causal:
        return int(n_q * (int(w.sum()) * block * d + 4 * tail * d))
    off = n_kv - n_q                              # query i sits at position off + i
    lo, hi = off, off + n_q - 1                   # query positions
    b = np.arange(nb, dtype=np.int64)
    start = b * block
    # keys seen in block b by a query at position p: clamp(p - start + 1, 0, block)
    full_from = start + block - 1                 # p >= full_from -> whole block
    n_full = np.clip(hi - np.maximum(full_from, lo) + 1, 0, None)
    a = np.maximum(start, lo)                     # partial range p in [a, e]
    e = np.minimum(full_from - 1, hi)
    cnt = np.clip(e - a + 1, 0, None)
    first = a - start + 1
    partial = np.where(cnt > 0, cnt * first + cnt * (cnt - 1) // 2, 0)
    keys = n_full * block + partial
    flops = int((keys * w).sum()) * d
    if tail:
        # tail keys seen by query p: clamp(p - prefix + 1, 0, tail)
        p = np.arange(lo, hi + 1, dtype=np.int64)
        flops += int(np.clip(p - prefix + 1, 0, tail).sum()) * 4 * d
    return flops


def flop_and_byte_count(n_q: int, k: DeviceCompressedCache, v: DeviceCompressedCache, tail: int = 0,
                        causal: bool = False, unit: int = 0) -> tuple[int, int]:
    """flop_and_byte_count (attention.hpp:426-467) for one unit, from the index maps."""
    def kinds(c):
        if c.sparse_count and c.dense_count:
            return (c.index_map[unit] > 0).cpu().numpy()
        return [1 if c.sparse_count == 0 else 0] * c.logical_blocks
    flops = flop_count(kinds(k), kinds(v), k.block_size, k.head_dim, n_q, tail, causal)
    nbytes = 0
    for c in (k, v):
        nbytes += HEADER_BYTES + sum(c.measure_size().values())
    nbytes += 2 * tail * k.head_dim * 2
    return flops, nbytes
