"""Shared test helpers: seeded inputs from the reference generator and
device-cache -> oracle-cache conversion.  Test infrastructure only."""
from __future__ import annotations

import concurrent.futures as cf
import os

import numpy as np

from oracle.oracle import CompressedCache, Oracle

THREADS = max(1, min(16, os.cpu_count() or 1))


def gen_units(port: Oracle, n_units: int, rows: int, d: int, seed: int, role: int, dtype: str) -> np.ndarray:
    """random_gaussian(rows, d, head_seed(seed, unit, role)) per unit (pipeline.hpp:168-169),
    rounded once (RNE) to the kernel dtype.  float32 [units, rows, d]."""
    def one(u):
        x = port.random_gaussian(rows, d, port.head_seed(seed, u, role))
        return port.round_to(x, dtype)
    with cf.ThreadPoolExecutor(THREADS) as ex:
        return np.stack(list(ex.map(one, range(n_units))))


def to_torch(x: np.ndarray, dtype: str):
    import torch
    t = torch.from_numpy(np.ascontiguousarray(x))
    return t.to(torch.bfloat16 if dtype == "bf16" else torch.float16).cuda()


def device_to_oracle(c, u: int) -> CompressedCache:
    """Unit u of a DeviceCompressedCache as an oracle CompressedCache (float32 pools)."""
    f = lambda t: t[u].float().cpu().numpy().reshape(-1).astype(np.float32)  # noqa: E731
    return CompressedCache(
        axis=c.axis, head_dim=c.head_dim, block_size=c.block_size, logical_blocks=c.logical_blocks,
        dense_count=c.dense_count, sparse_count=c.sparse_count,
        index_map=c.index_map[u].cpu().numpy().astype(np.int16),
        dense_pool=f(c.dense_pool) if c.dense_count else np.zeros(1, np.float32),
        nnz_pool=f(c.nnz_pool) if c.sparse_count else np.zeros(1, np.float32),
        meta_pool=(c.meta_pool[u].cpu().numpy().view(np.uint16).reshape(-1) if c.sparse_count
                   else np.zeros(1, np.uint16)),
        flags=c.flags[u].cpu().numpy(), losses=c.losses[u].cpu().numpy())


def parallel(fn, items):
    with cf.ThreadPoolExecutor(THREADS) as ex:
        return list(ex.map(fn, items))


def err_stats(got: np.ndarray, want: np.ndarray) -> tuple[float, float]:
    """(max-abs, mean-rel = sum|e| / sum|ref|) — the north-star tolerance metrics."""
    e = np.abs(got.astype(np.float64) - want.astype(np.float64))
    return float(e.max()), float(e.sum() / max(np.abs(want).sum(), 1e-30))


# North-star bar for attention outputs (BASELINE.json north_star).
MAX_ABS_TOL = 2e-2
MEAN_REL_TOL = 1e-3
