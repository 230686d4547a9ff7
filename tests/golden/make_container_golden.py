"""Generate tests/golden/container_vectors.npz from the UNMODIFIED reference's
container code (serialize / parse, container.hpp:119-250) via oracle/_ref.

For small caches compressed by the reference from fp16- and bf16-rounded inputs,
stores the 16-bit storage arrays of each cache and the reference's serialized
bytes; and for corrupted byte strings, the reference's parse verdict and message.

    python tests/golden/make_container_golden.py
"""
import os
import struct
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle.oracle import Oracle, SparsityConfig, ref_parse, ref_serialize  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "container_vectors.npz")


def bits(x: np.ndarray, dtype: str) -> np.ndarray:
    x = np.ascontiguousarray(x, np.float32)
    if dtype == "f16":
        return x.astype(np.float16).view(np.uint16)
    u = x.view(np.uint32)
    assert (u & 0xFFFF).max(initial=0) == 0
    return (u >> 16).astype(np.uint16)


def main() -> None:
    ref, port = Oracle("reference"), Oracle("port")
    g = {}
    L, d = 256, 128
    cases = [("f16_s50_k", "f16", 0.5, 0), ("f16_s100_v", "f16", 1.0, 1), ("bf16_s25_k", "bf16", 0.25, 0),
             ("bf16_s0_v", "bf16", 0.0, 1)]
    for name, dt, s, axis in cases:
        x = port.round_to(ref.random_gaussian(L, d, ref.head_seed(11, 0, axis)), dt)
        c = ref.prune_compress(x, SparsityConfig(s, s, 64), axis, s)
        g[name + "_geom"] = np.array([axis, d, 64, c.logical_blocks, c.dense_count, c.sparse_count], np.int64)
        g[name + "_index_map"] = c.index_map
        g[name + "_dense_bits"] = bits(c.dense_pool[: c.dense_count * 64 * d], dt)
        g[name + "_nnz_bits"] = bits(c.nnz_pool[: c.sparse_count * 32 * d], dt)
        g[name + "_meta_pool"] = c.meta_pool[: c.sparse_count * 512]
        g[name + "_bytes"] = np.frombuffer(ref_serialize(c), np.uint8)
    good = bytes(g["f16_s50_k_bytes"])
    corrupt = {
        "magic": b"X" + good[1:],
        "version": good[:8] + struct.pack("<H", 2) + good[10:],
        "truncated_header": good[:20],
        "truncated_payload": good[:-3],
        "section_length": good[:38] + struct.pack("<Q", 6) + good[46:],
        "trailing": good + b"\0",
        "width_tag": good[:34] + struct.pack("<H", 2) + good[36:],
        "zero_index": good[:46] + b"\0\0" + good[48:],
        "dup_slot": good[:46] + good[48:50] + good[48:],
    }
    for k, v in corrupt.items():
        rc, msg, _ = ref_parse(v)
        g["bad_" + k + "_bytes"] = np.frombuffer(v, np.uint8)
        g["bad_" + k + "_rc"] = np.int64(rc)
        g["bad_" + k + "_msg"] = np.array(msg)
    np.savez_compressed(OUT, **g)
    print(f"wrote {OUT} ({os.path.getsize(OUT)} bytes)")


if __name__ == "__main__":
    main()
