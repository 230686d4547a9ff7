"""Generate tests/golden/reference_vectors.npz from the UNMODIFIED reference.

Runs the reference compiled in place (oracle/_ref/libhs_ref.so, built by
oracle/Makefile from /root/reference/proj/include) on small seeded inputs and
stores its outputs.  The fixtures pin the oracle port and the GPU path on
machines where /root/reference is absent (the GPU box).

    python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle.oracle import Oracle, SparsityConfig  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "reference_vectors.npz")


def bf16_bits(x: np.ndarray) -> np.ndarray:
    u = np.ascontiguousarray(x, np.float32).view(np.uint32)
    assert (u & 0xFFFF).max(initial=0) == 0, "values are not bf16-representable"
    return (u >> 16).astype(np.uint16)


def main() -> None:
    ref = Oracle("reference")
    port = Oracle("port")
    g = {}
    # tensor.hpp:91-137 generator streams
    for i, seed in enumerate([1, 42, (1 << 63) - 1]):
        g[f"gauss_{i}_seed"] = np.uint64(seed)
        g[f"gauss_{i}"] = ref.random_gaussian(4, 8, seed)
    g["head_seed_7_3_2"] = np.uint64(ref.head_seed(7, 3, 2))

    # Pruning + compression: L=256 (4 blocks) + 17-token dense tail, d=128, bf16 inputs.
    L, tail, d, B, seed = 256, 17, 128, 64, 7
    scale = np.float32(1.0 / np.sqrt(d))
    key = port.round_to(ref.random_gaussian(L + tail, d, ref.head_seed(seed, 0, 0)), "bf16")
    val = port.round_to(ref.random_gaussian(L + tail, d, ref.head_seed(seed, 0, 1)), "bf16")
    for name, s, sink, window in [("s50", 0.5, 0, 0), ("s100w", 1.0, 64, 70), ("s25", 0.25, 0, 0)]:
        cfg = SparsityConfig(s_key=s, s_value=s, block_size=B, sink_tokens=sink,
                             local_window=window)
        caches = {}
        for axis, x in ((0, key), (1, val)):
            c = ref.prune_compress(x[:L], cfg, axis, s)
            caches[axis] = c
            p = f"{name}_{'k' if axis == 0 else 'v'}"
            g[p + "_index_map"] = c.index_map
            g[p + "_flags"] = c.flags
            g[p + "_losses"] = c.losses
            g[p + "_dense_pool"] = bf16_bits(c.dense_pool)
            g[p + "_nnz_pool"] = bf16_bits(c.nnz_pool)
            g[p + "_meta_pool"] = c.meta_pool
            g[p + "_cfg"] = np.array([s, sink, window], np.float64)
        kc, vc = caches[0], caches[1]
        qd = port.round_to(np.stack([ref.random_gaussian(1, d, ref.head_seed(seed, 0, 32 + j))[0]
                                     for j in range(4)]), "bf16")
        g[name + "_decode_q"] = qd
        g[name + "_decode_out"] = ref.decode(qd, kc, vc, key[L:], val[L:], scale, splits=3)
        qp = port.round_to(ref.random_gaussian(L + tail, d, ref.head_seed(seed, 0, 2)), "bf16")
        g[name + "_prefill_out"] = ref.prefill(qp, kc, vc, key[L:], val[L:], True, scale, b_r=64)
        f, by = ref.flop_and_byte_count(L + tail, d, kc, vc, tail, True)
        g[name + "_prefill_counts"] = np.array([f, by], np.uint64)
    g["key"] = bf16_bits(key)
    g["val"] = bf16_bits(val)
    np.savez_compressed(OUT, **g)
    print(f"wrote {OUT} ({os.path.getsize(OUT)} bytes, {len(g)} arrays)")


if __name__ == "__main__":
    main()
