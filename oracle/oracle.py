"""TEST INFRASTRUCTURE ONLY — ctypes binding of the CPU oracle.

Loads either the plain-C restatement (``oracle/build/libhs_oracle.so``, symbol
prefix ``hso_``) or the reference compiled in place (``oracle/_ref/libhs_ref.so``,
prefix ``ref_``); both export the interface in ``oracle/hs_oracle.h``.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU-baseline legs may
import this module.  It is the checker, never the thing measured or shipped.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "build", "libhs_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libhs_ref.so")


class ConfigError(ValueError):
    """errors.hpp:10-13 (std::invalid_argument)."""


class DataError(RuntimeError):
    """errors.hpp:17-20 (std::runtime_error)."""


class _Cache(C.Structure):
    _fields_ = [
        ("axis", C.c_int),
        ("head_dim", C.c_size_t),
        ("block_size", C.c_size_t),
        ("logical_blocks", C.c_size_t),
        ("dense_count", C.c_size_t),
        ("sparse_count", C.c_size_t),
        ("index_map", C.POINTER(C.c_int16)),
        ("dense_pool", C.POINTER(C.c_float)),
        ("nnz_pool", C.POINTER(C.c_float)),
        ("meta_pool", C.POINTER(C.c_uint16)),
    ]


class _Config(C.Structure):
    _fields_ = [
        ("s_key", C.c_double),
        ("s_value", C.c_double),
        ("block_size", C.c_size_t),
        ("sink_tokens", C.c_size_t),
        ("local_window", C.c_size_t),
    ]


@dataclass
class SparsityConfig:
    """masks.hpp:73-99 (pattern fixed at 2:4)."""

    s_key: float = 0.0
    s_value: float = 0.0
    block_size: int = 64
    sink_tokens: int = 0
    local_window: int = 0

    def _c(self) -> _Config:
        return _Config(self.s_key, self.s_value, self.block_size, self.sink_tokens,
                       self.local_window)


@dataclass
class CompressedCache:
    """compressed_cache.hpp:37-110 as numpy arrays (float32 pools)."""

    axis: int
    head_dim: int
    block_size: int
    logical_blocks: int
    dense_count: int
    sparse_count: int
    index_map: np.ndarray
    dense_pool: np.ndarray
    nnz_pool: np.ndarray
    meta_pool: np.ndarray
    flags: np.ndarray | None = None
    losses: np.ndarray | None = None
    element_mask: np.ndarray | None = field(default=None, repr=False)

    @property
    def block_elems(self) -> int:
        return self.block_size * self.head_dim

    @property
    def meta_words(self) -> int:
        return self.block_elems // 16

    def _c(self) -> _Cache:
        self._keep = [np.ascontiguousarray(a) for a in
                      (self.index_map, self.dense_pool, self.nnz_pool, self.meta_pool)]
        im, dp, nz, mp = self._keep
        return _Cache(self.axis, self.head_dim, self.block_size, self.logical_blocks,
                      self.dense_count, self.sparse_count,
                      im.ctypes.data_as(C.POINTER(C.c_int16)),
                      dp.ctypes.data_as(C.POINTER(C.c_float)),
                      nz.ctypes.data_as(C.POINTER(C.c_float)),
                      mp.ctypes.data_as(C.POINTER(C.c_uint16)))

    def size_breakdown(self) -> dict:
        """measure_size (compressed_cache.hpp:303-310)."""
        return dict(size_idx=self.logical_blocks * 2,
                    size_den=self.dense_count * self.block_elems * 2,
                    size_nnz=self.sparse_count * self.block_elems // 2 * 2,
                    size_e=self.sparse_count * self.meta_words * 2)


def _fp(a):
    return a.ctypes.data_as(C.POINTER(C.c_float))


def build(quiet: bool = True) -> None:
    """Run oracle/Makefile (the port always; the reference when present)."""
    out = subprocess.run(["make", "-C", HERE], capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError(f"oracle build failed:\n{out.stdout}\n{out.stderr}")
    if not quiet:
        print(out.stdout)


class Oracle:
    """One oracle library.  ``kind`` is "port" (hso_) or "reference" (ref_)."""

    def __init__(self, kind: str = "port"):
        path, prefix = (PORT_SO, "hso_") if kind == "port" else (REF_SO, "ref_")
        if not os.path.exists(path):
            raise FileNotFoundError(f"oracle library missing: {path} (run make -C oracle)")
        self.kind = kind
        self.lib = C.CDLL(path)
        self.p = prefix
        L = self.lib
        f = lambda n: getattr(L, prefix + n)  # noqa: E731
        f("last_error").restype = C.c_char_p
        f("derive_seed").restype = C.c_uint64
        f("derive_seed").argtypes = [C.c_uint64, C.c_uint64]
        f("head_seed").restype = C.c_uint64
        f("head_seed").argtypes = [C.c_uint64, C.c_size_t, C.c_size_t]
        f("random_gaussian").argtypes = [C.c_size_t, C.c_size_t, C.c_uint64, C.c_float,
                                         C.POINTER(C.c_float)]
        f("random_gaussian").restype = None
        vp = C.c_void_p
        f("prune_compress").argtypes = [vp, C.c_size_t, C.c_size_t, C.POINTER(_Config), C.c_int,
                                        C.c_double, C.c_int, C.POINTER(_Cache), vp, vp, vp]
        f("compress_with_flags").argtypes = [vp, C.c_size_t, C.c_size_t, C.POINTER(_Config),
                                             C.c_int, vp, C.POINTER(_Cache)]
        f("compress_with_mask").argtypes = [vp, C.c_size_t, C.c_size_t, C.POINTER(_Config),
                                            C.c_int, vp, vp, C.POINTER(_Cache)]
        f("decompress").argtypes = [C.POINTER(_Cache), vp]
        f("attend_rows").argtypes = [vp, C.c_size_t, C.c_size_t, C.POINTER(_Cache),
                                     C.POINTER(_Cache), vp, vp, C.c_size_t, C.c_size_t,
                                     C.c_size_t, C.c_int, C.c_float, vp, vp, vp, vp]
        f("decode").argtypes = [vp, C.c_size_t, C.c_size_t, C.POINTER(_Cache), C.POINTER(_Cache),
                                vp, vp, C.c_size_t, C.c_float, C.c_size_t, C.c_size_t, vp]
        f("prefill").argtypes = [vp, C.c_size_t, C.c_size_t, C.POINTER(_Cache), C.POINTER(_Cache),
                                 vp, vp, C.c_size_t, C.c_int, C.c_float, C.c_size_t, vp]
        f("dense_attention").argtypes = [vp, C.c_size_t, vp, vp, C.c_size_t, C.c_size_t, C.c_int,
                                         C.c_float, vp]
        f("flop_and_byte_count").argtypes = [C.c_size_t, C.c_size_t, C.POINTER(_Cache),
                                             C.POINTER(_Cache), C.c_size_t, C.c_int,
                                             C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]
        if kind == "port":
            L.hso_pool_counts.argtypes = [C.c_size_t, C.c_size_t, C.c_double, C.c_size_t,
                                          C.c_size_t] + [C.POINTER(C.c_size_t)] * 3
            L.hso_round_bf16.argtypes = [vp, C.c_size_t]
            L.hso_round_f16.argtypes = [vp, C.c_size_t]

    # -- plumbing ---------------------------------------------------------
    def _fn(self, name):
        return getattr(self.lib, self.p + name)

    def _check(self, rc: int) -> None:
        if rc == 0:
            return
        msg = self._fn("last_error")().decode()
        if rc == 2:
            raise ConfigError(msg)
        raise DataError(msg)

    # -- tensor.hpp -----------------------------------------------------------
    def derive_seed(self, base: int, stream: int) -> int:
        return self._fn("derive_seed")(base, stream)

    def head_seed(self, base: int, head: int, role: int) -> int:
        return self._fn("head_seed")(base, head, role)

    def random_gaussian(self, rows: int, cols: int, seed: int, scale: float = 1.0) -> np.ndarray:
        out = np.empty((rows, cols), np.float32)
        self._fn("random_gaussian")(rows, cols, seed, scale, _fp(out))
        return out

    def round_to(self, x: np.ndarray, dtype: str) -> np.ndarray:
        """RNE rounding to bf16 / f16 values kept as float32 (port only)."""
        x = np.ascontiguousarray(x, np.float32).copy()
        lib = self.lib if self.kind == "port" else Oracle("port").lib
        (lib.hso_round_bf16 if dtype == "bf16" else lib.hso_round_f16)(x.ctypes.data, x.size)
        return x

    def pool_counts(self, rows, block_size, sparsity, sink=0, window=0):
        p, s, q = C.c_size_t(), C.c_size_t(), C.c_size_t()
        lib = self.lib if self.kind == "port" else Oracle("port").lib
        rc = lib.hso_pool_counts(rows, block_size, sparsity, sink, window, C.byref(p),
                                 C.byref(s), C.byref(q))
        if rc:
            lib.hso_last_error.restype = C.c_char_p
            raise ConfigError(lib.hso_last_error().decode())
        return p.value, s.value, q.value

    # -- pruner + compressor --------------------------------------------------
    def _empty_cache(self, rows, cols, block, axis):
        nb = rows // block if block else 0
        be = block * cols
        return CompressedCache(axis, cols, block, nb, 0, 0,
                               np.zeros(max(nb, 1), np.int16),
                               np.zeros(max(nb * be, 1), np.float32),
                               np.zeros(max(nb * be // 2, 1), np.float32),
                               np.zeros(max(nb * be // 16, 1), np.uint16))

    def _finish(self, c: CompressedCache, cs: _Cache) -> CompressedCache:
        c.logical_blocks = cs.logical_blocks
        c.dense_count, c.sparse_count = cs.dense_count, cs.sparse_count
        be = c.block_elems
        c.index_map = c.index_map[: c.logical_blocks].copy()
        c.dense_pool = c.dense_pool[: c.dense_count * be].copy()
        c.nnz_pool = c.nnz_pool[: c.sparse_count * be // 2].copy()
        c.meta_pool = c.meta_pool[: c.sparse_count * (be // 16)].copy()
        return c

    def prune_compress(self, x: np.ndarray, cfg: SparsityConfig, axis: int, sparsity: float,
                       fused: bool = True, element_mask: bool = False) -> CompressedCache:
        """hierarchical_mask_for (pruner.hpp:121) + compress / fused_magnitude_compress."""
        x = np.ascontiguousarray(x, np.float32)
        rows, cols = x.shape
        block = cfg.block_size
        c = self._empty_cache(rows, cols, block if block else 1, axis)
        nb = rows // block if block else 0
        flags = np.zeros(max(nb, 1), np.uint8)
        losses = np.zeros(max(nb, 1), np.float64)
        em = np.zeros(rows * cols, np.uint8) if element_mask else None
        cs = c._c()
        cc = cfg._c()
        rc = self._fn("prune_compress")(x.ctypes.data, rows, cols, C.byref(cc), axis, sparsity,
                                        int(fused), C.byref(cs), flags.ctypes.data,
                                        losses.ctypes.data,
                                        em.ctypes.data if em is not None else None)
        self._check(rc)
        c = self._finish(c, cs)
        c.flags = flags[:nb].copy()
        c.losses = losses[:nb].copy()
        if em is not None:
            c.element_mask = em.reshape(rows, cols)
        return c

    def compress_with_flags(self, x, cfg: SparsityConfig, axis: int, flags) -> CompressedCache:
        """fused_magnitude_compress (compressed_cache.hpp:262) under a given BlockMask."""
        x = np.ascontiguousarray(x, np.float32)
        rows, cols = x.shape
        flags = np.ascontiguousarray(flags, np.uint8)
        c = self._empty_cache(rows, cols, cfg.block_size if cfg.block_size else 1, axis)
        cs = c._c()
        cc = cfg._c()
        rc = self._fn("compress_with_flags")(x.ctypes.data, rows, cols, C.byref(cc), axis,
                                             flags.ctypes.data, C.byref(cs))
        self._check(rc)
        return self._finish(c, cs)

    def compress_with_mask(self, x, cfg: SparsityConfig, axis: int, element_mask, flags) -> CompressedCache:
        """compress (compressed_cache.hpp:196-225) under an explicit element + block mask."""
        x = np.ascontiguousarray(x, np.float32)
        rows, cols = x.shape
        em = np.ascontiguousarray(element_mask, np.uint8).reshape(rows, cols)
        flags = np.ascontiguousarray(flags, np.uint8)
        c = self._empty_cache(rows, cols, cfg.block_size if cfg.block_size else 1, axis)
        cs = c._c()
        cc = cfg._c()
        rc = self._fn("compress_with_mask")(x.ctypes.data, rows, cols, C.byref(cc), axis, em.ctypes.data,
                                            flags.ctypes.data, C.byref(cs))
        self._check(rc)
        return self._finish(c, cs)

    def decompress(self, c: CompressedCache) -> np.ndarray:
        out = np.zeros((c.logical_blocks * c.block_size, c.head_dim), np.float32)
        cs = c._c()
        self._check(self._fn("decompress")(C.byref(cs), out.ctypes.data))
        return out

    # -- attention -------------------------------------------------------------
    @staticmethod
    def _tails(d, k_tail, v_tail):
        if k_tail is None or len(k_tail) == 0:
            z = np.zeros((1, d), np.float32)
            return z, z, 0
        kt = np.ascontiguousarray(k_tail, np.float32)
        vt = np.ascontiguousarray(v_tail, np.float32)
        return kt, vt, kt.shape[0]

    def attend_rows(self, q, k, v, k_tail=None, v_tail=None, block_begin=0, block_end=None,
                    include_tail=True, scale=1.0, qpos=None):
        """attend_range (attention.hpp:249-304) -> (output_t [d][rows], m_s, l_s)."""
        q = np.ascontiguousarray(q, np.float32)
        rows, d = q.shape
        kt, vt, tail = self._tails(d, k_tail, v_tail)
        if block_end is None:
            block_end = k.logical_blocks if k is not None else 0
        out_t = np.zeros((d, rows), np.float32)
        m = np.zeros(rows, np.float32)
        l = np.zeros(rows, np.float32)
        qp = None if qpos is None else np.ascontiguousarray(qpos, np.int64)
        ks = C.byref(k._c()) if k is not None else None
        vs = C.byref(v._c()) if v is not None else None
        rc = self._fn("attend_rows")(q.ctypes.data, rows, d, ks, vs, kt.ctypes.data,
                                     vt.ctypes.data, tail, block_begin, block_end,
                                     int(include_tail), scale,
                                     qp.ctypes.data if qp is not None else None,
                                     out_t.ctypes.data, m.ctypes.data, l.ctypes.data)
        self._check(rc)
        return out_t, m, l

    def decode(self, q, k, v, k_tail=None, v_tail=None, scale=1.0, splits=1, gqa_group=None):
        """decode_attention (attention.hpp:360-409)."""
        q = np.ascontiguousarray(q, np.float32)
        n_q, d = q.shape
        kt, vt, tail = self._tails(d, k_tail, v_tail)
        out = np.zeros((n_q, d), np.float32)
        ks = C.byref(k._c()) if k is not None else None
        vs = C.byref(v._c()) if v is not None else None
        rc = self._fn("decode")(q.ctypes.data, n_q, d, ks, vs, kt.ctypes.data, vt.ctypes.data,
                                tail, scale, splits, n_q if gqa_group is None else gqa_group,
                                out.ctypes.data)
        self._check(rc)
        return out

    def prefill(self, q, k, v, k_tail=None, v_tail=None, causal=True, scale=1.0, b_r=64):
        """prefill_attention (attention.hpp:323-354)."""
        q = np.ascontiguousarray(q, np.float32)
        n_q, d = q.shape
        kt, vt, tail = self._tails(d, k_tail, v_tail)
        out = np.zeros((n_q, d), np.float32)
        ks = C.byref(k._c()) if k is not None else None
        vs = C.byref(v._c()) if v is not None else None
        rc = self._fn("prefill")(q.ctypes.data, n_q, d, ks, vs, kt.ctypes.data, vt.ctypes.data,
                                 tail, int(causal), scale, b_r, out.ctypes.data)
        self._check(rc)
        return out

    def dense_attention(self, q, k, v, causal, scale):
        """dense_attention_oracle (attention.hpp:84-115)."""
        q = np.ascontiguousarray(q, np.float32)
        k = np.ascontiguousarray(k, np.float32)
        v = np.ascontiguousarray(v, np.float32)
        out = np.zeros((q.shape[0], v.shape[1]), np.float32)
        rc = self._fn("dense_attention")(q.ctypes.data, q.shape[0], k.ctypes.data, v.ctypes.data,
                                         k.shape[0], q.shape[1], int(causal), scale,
                                         out.ctypes.data)
        self._check(rc)
        return out

    def flop_and_byte_count(self, n_q, d, k, v, tail=0, causal=False):
        """flop_and_byte_count (attention.hpp:426-467)."""
        fl, by = C.c_uint64(), C.c_uint64()
        ks = C.byref(k._c()) if k is not None else None
        vs = C.byref(v._c()) if v is not None else None
        rc = self._fn("flop_and_byte_count")(n_q, d, ks, vs, tail, int(causal), C.byref(fl),
                                             C.byref(by))
        self._check(rc)
        return fl.value, by.value


def available(kind: str) -> bool:
    return os.path.exists(PORT_SO if kind == "port" else REF_SO)


def ref_serialize(c: CompressedCache) -> bytes:
    """The reference's serialize (container.hpp:119-148) of one cache (oracle/_ref only)."""
    ref = Oracle("reference")
    ref.lib.ref_serialize.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.POINTER(C.c_size_t)]
    n = C.c_size_t()
    cs = c._c()
    ref._check(ref.lib.ref_serialize(C.byref(cs), None, 0, C.byref(n)))
    buf = (C.c_uint8 * n.value)()
    cs = c._c()
    ref._check(ref.lib.ref_serialize(C.byref(cs), buf, n.value, C.byref(n)))
    return bytes(buf)


def ref_parse(data: bytes):
    """The reference's parse (container.hpp:150-250): (rc, message, (nb, dense, sparse))."""
    ref = Oracle("reference")
    ref.lib.ref_parse.argtypes = [C.c_void_p, C.c_size_t, C.POINTER(C.c_size_t), C.POINTER(C.c_size_t),
                                  C.POINTER(C.c_size_t)]
    a, b, c = C.c_size_t(), C.c_size_t(), C.c_size_t()
    buf = (C.c_uint8 * len(data)).from_buffer_copy(data)
    rc = ref.lib.ref_parse(buf, len(data), C.byref(a), C.byref(b), C.byref(c))
    msg = ref.lib.ref_last_error().decode() if rc else ""
    return rc, msg, (a.value, b.value, c.value)
