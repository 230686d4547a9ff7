"""Generate tests/golden/small_shapes.npz from the UNMODIFIED reference.

The reference accepts any block size B and head dimension d that are multiples
of the 2:4 group (masks.hpp:87, pruner.hpp:172-173) and its own tests use small
ones (test_compressor.cpp, test_attention.cpp).  These fixtures run the
reference compiled in place (oracle/_ref) on seeded bf16 inputs at such shapes
-- prune_cache + fused_magnitude_compress pools, decode_attention (GQA up to
16) and causal prefill_attention with a ragged dense tail -- so the device
path's generic-shape kernels are pinned on the GPU box, where /root/reference
is absent.

    python tests/golden/make_small_shapes.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle.oracle import Oracle, SparsityConfig  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "small_shapes.npz")

# (name, L, tail, d, B, S, sink, window, gqa)
SHAPES = [
    ("b4d8", 32, 3, 8, 4, 0.5, 0, 0, 2),
    ("b16d32", 128, 9, 32, 16, 0.5, 16, 16, 4),
    ("b32d64", 320, 0, 64, 32, 1.0, 0, 0, 8),
    ("b64d64", 512, 17, 64, 64, 0.25, 64, 70, 16),
    ("b128d256", 512, 5, 256, 128, 0.75, 0, 0, 2),
    ("b8d128", 96, 0, 128, 8, 1.0, 0, 0, 4),
    ("b64d128g12", 256, 0, 128, 64, 1.0, 0, 0, 12),  # standard shape, GQA 12 > 8 rows
]


def bf16_bits(x: np.ndarray) -> np.ndarray:
    u = np.ascontiguousarray(x, np.float32).view(np.uint32)
    assert (u & 0xFFFF).max(initial=0) == 0, "values are not bf16-representable"
    return (u >> 16).astype(np.uint16)


def main() -> None:
    ref = Oracle("reference")
    port = Oracle("port")
    g = {}
    for name, L, tail, d, B, s, sink, window, gqa in SHAPES:
        seed = 100 + len(name)
        scale = np.float32(1.0 / np.sqrt(d))
        key = port.round_to(ref.random_gaussian(L + tail, d, ref.head_seed(seed, 0, 0)), "bf16")
        val = port.round_to(ref.random_gaussian(L + tail, d, ref.head_seed(seed, 0, 1)), "bf16")
        cfg = SparsityConfig(s_key=s, s_value=s, block_size=B, sink_tokens=sink, local_window=window)
        caches = {}
        for axis, x in ((0, key), (1, val)):
            c = ref.prune_compress(x[:L], cfg, axis, s)
            caches[axis] = c
            p = f"{name}_{'k' if axis == 0 else 'v'}"
            g[p + "_index_map"] = c.index_map
            g[p + "_flags"] = c.flags
            g[p + "_losses"] = c.losses
            g[p + "_dense_pool"] = bf16_bits(c.dense_pool) if c.dense_count else np.zeros(0, np.uint16)
            g[p + "_nnz_pool"] = bf16_bits(c.nnz_pool) if c.sparse_count else np.zeros(0, np.uint16)
            g[p + "_meta_pool"] = c.meta_pool if c.sparse_count else np.zeros(0, np.uint16)
        kc, vc = caches[0], caches[1]
        kt, vt = (key[L:], val[L:]) if tail else (None, None)
        qd = port.round_to(np.stack([ref.random_gaussian(1, d, ref.head_seed(seed, 0, 32 + j))[0]
                                     for j in range(gqa)]), "bf16")
        g[name + "_decode_q"] = qd
        g[name + "_decode_out"] = ref.decode(qd, kc, vc, kt, vt, scale, splits=2)
        n_q = min(L + tail, 160)
        qp = port.round_to(ref.random_gaussian(n_q, d, ref.head_seed(seed, 0, 2)), "bf16")
        g[name + "_prefill_q"] = qp
        g[name + "_prefill_out"] = ref.prefill(qp, kc, vc, kt, vt, True, scale, b_r=B)
        g[name + "_shape"] = np.array([L, tail, d, B, gqa, n_q, sink, window], np.int64)
        g[name + "_s"] = np.array([s], np.float64)
        g[name + "_key"] = bf16_bits(key)
        g[name + "_val"] = bf16_bits(val)
    g["names"] = np.array([s[0] for s in SHAPES])
    np.savez_compressed(OUT, **g)
    print(f"wrote {OUT} ({os.path.getsize(OUT)} bytes, {len(g)} arrays)")


if __name__ == "__main__":
    main()
