"""Pins the CPU oracle (oracle/hs_oracle.c) before it is trusted as the checker.

1. Golden vectors restated from the reference's own gtest suites
   (proj/tests/test_{metadata,pruner,compressor,attention}.cpp).
2. The committed fixtures produced by the compiled reference
   (tests/golden/reference_vectors.npz, tests/golden/make_golden.py).
3. Randomised bit-for-bit cross-checks against the reference compiled in place
   (oracle/_ref), when present (it is in the build container).
"""
import os

import numpy as np
import pytest

from oracle.oracle import CompressedCache, ConfigError, DataError, SparsityConfig

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "reference_vectors.npz")


def one_block(rows, block, axis=0):
    return SparsityConfig(block_size=block)


# ---------------------------------------------------------------- metadata ----
def test_single_group_metadata_word(port):
    # test_compressor.cpp:67-80 + test_metadata.cpp:16-22: kept {1,3} -> 0x000D
    x = np.zeros((4, 4), np.float32)
    x[0] = [0.1, -3.0, 0.0, 2.5]
    c = port.compress_with_flags(x, SparsityConfig(block_size=4), 0, [0])
    assert c.nnz_pool[0] == -3.0 and c.nnz_pool[1] == 2.5
    assert c.meta_pool[0] & 0xF == 0xD


def test_all_zero_groups_keep_lowest_positions(port):
    # test_pruner.cpp:47-54 (ties keep {0,1}) and test_metadata.cpp:24-28 (0x4444)
    x = np.zeros((4, 16), np.float32)
    c = port.compress_with_flags(x, SparsityConfig(block_size=4), 0, [0])
    assert (c.meta_pool == 0x4444).all()


def test_code_order_0x00d8(port):
    # test_metadata.cpp:37-44: groups {0,2},{1,3} -> 0x00D8
    x = np.zeros((4, 8), np.float32)
    x[0] = [5, 0, 6, 0, 0, 7, 0, 8]
    c = port.compress_with_flags(x, SparsityConfig(block_size=4), 0, [0])
    assert c.meta_pool[0] & 0xFF == 0xD8  # rows 1-3 are zero groups -> 0x44 above
    assert list(c.nnz_pool[:4]) == [5, 6, 7, 8]


# ------------------------------------------------------------------ pruner ----
def test_element_mask_and_loss_examples(port):
    # test_pruner.cpp:38-45 and :117-121: [1,-2,0.5,3] keeps {1,3}, loss 1.5
    x = np.zeros((4, 4), np.float32)
    x[0] = [1.0, -2.0, 0.5, 3.0]
    c = port.prune_compress(x, SparsityConfig(s_key=1, s_value=1, block_size=4), 0, 1.0,
                            element_mask=True)
    assert list(c.element_mask[0]) == [0, 1, 0, 1]
    assert c.losses[0] == 1.5


def test_sequence_axis_groups_run_down_rows(port):
    # test_pruner.cpp:56-69
    x = np.array([[1.0, 9.0], [-2.0, 0.1], [0.5, -8.0], [3.0, 0.2]], np.float32)
    x = np.concatenate([x, np.zeros((4, 2), np.float32)], axis=1)
    c = port.prune_compress(x, SparsityConfig(s_key=1, s_value=1, block_size=4), 1, 1.0,
                            element_mask=True)
    m = c.element_mask
    assert list(m[:, 0]) == [0, 1, 0, 1]
    assert list(m[:, 1]) == [1, 0, 1, 0]


def _loss_blocks(losses, block=4):
    """Blocks whose block_loss equals the given values: one group [t/2, t/2, 100, 100]."""
    x = np.zeros((block * len(losses), 4), np.float32)
    for b, t in enumerate(losses):
        x[b * block] = [t / 2, t / 2, 100.0, 100.0]
    return x


@pytest.mark.parametrize("losses,s,prefix,suffix,sparse", [
    ([5.0, 1.0, 3.0, 2.0], 0.5, 0, 0, [1, 3]),        # test_pruner.cpp:123-130
    ([1.0, 2.0, 3.0], 0.5, 0, 0, [0]),                # floor quota :132-136
    ([2.0, 1.0, 1.0, 3.0], 0.5, 0, 0, [1, 2]),        # ties :138-145
    ([1.0, 1.0, 1.0, 1.0], 0.25, 0, 0, [0]),
    ([5.0, 1.0, 3.0, 2.0], 1.0, 1, 0, [1, 2, 3]),     # protection :147-159
    ([0.0, 0.0, 0.0, 0.0], 1.0, 1, 1, [1, 2]),
])
def test_select_blocks_examples(port, losses, s, prefix, suffix, sparse):
    x = _loss_blocks(losses)
    cfg = SparsityConfig(s_key=s, s_value=s, block_size=4, sink_tokens=prefix * 4,
                         local_window=suffix * 4)
    c = port.prune_compress(x, cfg, 0, s)
    assert list(c.losses) == losses
    assert [b for b in range(len(losses)) if c.flags[b] == 0] == sparse


def test_protected_regions_round_up(port):
    # test_pruner.cpp:250-270: sink 1 -> 1 block, window 9 -> 2 blocks (B=8)
    cfg = SparsityConfig(s_key=1, s_value=1, block_size=8, sink_tokens=1, local_window=9)
    x = port.random_gaussian(48, 8, 1)
    c = port.prune_compress(x, cfg, 0, 1.0)
    assert list(c.flags) == [1, 0, 0, 0, 1, 1]
    assert list(c.index_map) == [1, -1, -2, -3, 2, 3]


def test_overlapping_protection_clamps(port):
    # test_pruner.cpp:272-288
    cfg = SparsityConfig(s_key=1, s_value=1, block_size=8, sink_tokens=64, local_window=64)
    c = port.prune_compress(port.random_gaussian(16, 8, 3), cfg, 0, 1.0)
    assert c.sparse_count == 0 and list(c.flags) == [1, 1]


def test_pool_counts_host_side(port):
    assert port.pool_counts(131072, 64, 1.0) == (0, 0, 2048)
    assert port.pool_counts(48, 8, 1.0, 1, 9) == (1, 2, 3)
    assert port.pool_counts(65536, 64, 0.75) == (0, 0, 768)
    with pytest.raises(ConfigError):
        port.pool_counts(100, 64, 0.5)


def test_bad_geometry_rejected(port):
    # test_pruner.cpp:290-296, test_compressor.cpp:190-202
    with pytest.raises(ConfigError):
        port.prune_compress(np.zeros((12, 8), np.float32), SparsityConfig(block_size=8), 0, 0.5)
    with pytest.raises(ConfigError):
        port.prune_compress(np.zeros((16, 6), np.float32), SparsityConfig(block_size=8), 0, 0.5)


# -------------------------------------------------------------- compressor ----
def test_index_maps(port):
    # test_compressor.cpp:37-65
    cfg = SparsityConfig(block_size=4)
    x = port.random_gaussian(12, 8, 1)
    assert list(port.compress_with_flags(x, cfg, 0, [1, 1, 1]).index_map) == [1, 2, 3]
    assert list(port.compress_with_flags(x, cfg, 0, [0, 0, 0]).index_map) == [-1, -2, -3]
    assert list(port.compress_with_flags(x, cfg, 0, [1, 0, 1]).index_map) == [1, -1, 2]


def test_value_blocks_stored_transposed(port):
    # test_compressor.cpp:82-92
    x = port.random_gaussian(4, 8, 4)
    c = port.compress_with_flags(x, SparsityConfig(block_size=4), 1, [1])
    assert (c.dense_pool.reshape(8, 4) == x.T).all()
    assert (port.decompress(c) == x).all()


def test_measure_size_breakdowns(port):
    # test_compressor.cpp:151-174
    x = port.random_gaussian(128, 128, 8)
    cfg = SparsityConfig(block_size=64)
    assert port.compress_with_flags(x, cfg, 0, [1, 1]).size_breakdown() == dict(
        size_idx=4, size_den=32768, size_nnz=0, size_e=0)
    assert port.compress_with_flags(x, cfg, 0, [0, 0]).size_breakdown() == dict(
        size_idx=4, size_den=0, size_nnz=16384, size_e=2048)


def test_int16_pool_capacity(port):
    # test_compressor.cpp:176-188
    x = np.zeros((32768 * 4, 4), np.float32)
    with pytest.raises(ConfigError):
        port.compress_with_flags(x, SparsityConfig(block_size=4), 0, np.ones(32768, np.uint8))


def test_decompress_rejects_corrupt_maps(port):
    # test_compressor.cpp:220-236
    x = port.random_gaussian(8, 4, 11)
    c = port.compress_with_flags(x, SparsityConfig(block_size=4), 0, [1, 0])
    for idx, val in ((0, 0), (0, 2), (1, -5)):
        bad = CompressedCache(**{k: (v.copy() if isinstance(v, np.ndarray) else v)
                                 for k, v in c.__dict__.items() if not k.startswith("_")})
        bad.index_map[idx] = val
        with pytest.raises(DataError):
            port.decompress(bad)


# --------------------------------------------------------------- attention ----
def test_op_counts_closed_forms(port):
    # test_attention.cpp:410-424
    cfg = SparsityConfig(block_size=64)
    x = np.zeros((1024, 128), np.float32)
    kd = port.compress_with_flags(x, cfg, 0, np.ones(16, np.uint8))
    vd = port.compress_with_flags(x, cfg, 1, np.ones(16, np.uint8))
    assert port.flop_and_byte_count(1024, 128, kd, vd)[0] == 536870912
    ks = port.compress_with_flags(x, cfg, 0, np.zeros(16, np.uint8))
    vs = port.compress_with_flags(x, cfg, 1, np.zeros(16, np.uint8))
    assert port.flop_and_byte_count(1024, 128, ks, vs)[0] == 268435456


def test_decode_byte_count_config2(port):
    # 8 KV heads x 128K at S=1 -> 302,056,032 bytes
    cfg = SparsityConfig(block_size=64)
    x = np.zeros((131072, 128), np.float32)
    k = port.compress_with_flags(x, cfg, 0, np.zeros(2048, np.uint8))
    v = port.compress_with_flags(x, cfg, 1, np.zeros(2048, np.uint8))
    assert 8 * port.flop_and_byte_count(4, 128, k, v)[1] == 302056032


def test_dense_oracle_single_key(port):
    # test_attention.cpp:117-127
    q = port.random_gaussian(3, 4, 1)
    k = port.random_gaussian(1, 4, 2)
    v = port.random_gaussian(1, 4, 3)
    out = port.dense_attention(q, k, v, False, 0.5)
    assert np.allclose(out, np.repeat(v, 3, axis=0), atol=1e-7)


def test_decode_rejects_invalid(port):
    # test_attention.cpp:383-408
    cfg = SparsityConfig(block_size=16, s_key=0.5, s_value=0.5)
    k = port.prune_compress(port.random_gaussian(32, 32, 1), cfg, 0, 0.5)
    v = port.prune_compress(port.random_gaussian(32, 32, 2), cfg, 1, 0.5)
    with pytest.raises(ConfigError):
        port.decode(port.random_gaussian(4, 32, 3), k, v, scale=0.1, gqa_group=3)
    with pytest.raises(ConfigError):
        port.decode(port.random_gaussian(4, 32, 3), v, k, scale=0.1)


# ---------------------------------------------------- reference fixtures ----
def test_port_matches_committed_reference_vectors(port):
    g = np.load(GOLD)
    for i in range(3):
        seed = int(g[f"gauss_{i}_seed"])
        assert port.random_gaussian(4, 8, seed).tobytes() == g[f"gauss_{i}"].tobytes()
    assert port.head_seed(7, 3, 2) == int(g["head_seed_7_3_2"])
    to_f = lambda b: (b.astype(np.uint32) << 16).view(np.float32)  # noqa: E731
    key, val = to_f(g["key"]).reshape(-1, 128), to_f(g["val"]).reshape(-1, 128)
    L = 256
    for name in ("s50", "s100w", "s25"):
        caches = {}
        for axis, x in ((0, key), (1, val)):
            p = f"{name}_{'k' if axis == 0 else 'v'}"
            s, sink, window = g[p + "_cfg"]
            cfg = SparsityConfig(s, s, 64, int(sink), int(window))
            c = port.prune_compress(x[:L], cfg, axis, s)
            assert (c.index_map == g[p + "_index_map"]).all()
            assert (c.flags == g[p + "_flags"]).all()
            assert c.losses.tobytes() == g[p + "_losses"].tobytes()
            assert (to_f(g[p + "_dense_pool"]) == c.dense_pool).all()
            assert (to_f(g[p + "_nnz_pool"]) == c.nnz_pool).all()
            assert (c.meta_pool == g[p + "_meta_pool"]).all()
            caches[axis] = c
        scale = np.float32(1.0 / np.sqrt(128))
        out = port.decode(g[name + "_decode_q"], caches[0], caches[1], key[L:], val[L:], scale,
                          splits=3)
        assert out.tobytes() == g[name + "_decode_out"].tobytes()
        qp = port.round_to(port.random_gaussian(L + 17, 128, port.head_seed(7, 0, 2)), "bf16")
        out = port.prefill(qp, caches[0], caches[1], key[L:], val[L:], True, scale, 64)
        assert out.tobytes() == g[name + "_prefill_out"].tobytes()
        assert list(port.flop_and_byte_count(L + 17, 128, caches[0], caches[1], 17, True)) == \
            list(g[name + "_prefill_counts"])


# ------------------------------------------------ live reference cross-check ----
def test_port_equals_reference_random_compress(port, ref):
    rng = np.random.default_rng(0)
    for it in range(120):
        B = [4, 8, 16, 64][it % 4]
        nb = 1 + int(rng.integers(0, 6))
        cols = 4 * (1 + int(rng.integers(0, 8)))
        x = port.random_gaussian(nb * B, cols, int(rng.integers(1 << 62)))
        if it % 3 == 0:
            x = port.round_to(x, "bf16")
        if it % 5 == 0:
            x[:, :4] = 0.0
        cfg = SparsityConfig(0.5, 0.5, B, int(rng.integers(0, 2 * B)), int(rng.integers(0, 2 * B)))
        for axis in (0, 1):
            s = float(rng.integers(0, 5)) / 4
            a = port.prune_compress(x, cfg, axis, s, element_mask=True)
            b = ref.prune_compress(x, cfg, axis, s, fused=bool(it % 2), element_mask=True)
            for f in ("index_map", "dense_pool", "nnz_pool", "meta_pool", "flags", "losses",
                      "element_mask"):
                assert getattr(a, f).tobytes() == getattr(b, f).tobytes(), (it, axis, f)


def test_port_equals_reference_random_attention(port, ref):
    rng = np.random.default_rng(1)
    for it in range(40):
        B, nb = 16, 1 + int(rng.integers(0, 4))
        tail = int(rng.integers(0, B)) if it % 2 else 0
        d = 32 if it % 3 else 64
        cfg = SparsityConfig(block_size=B)
        sk, sv = float(rng.integers(0, 5)) / 4, float(rng.integers(0, 5)) / 4
        kc = port.prune_compress(port.random_gaussian(nb * B, d, it * 10 + 1), cfg, 0, sk)
        vc = port.prune_compress(port.random_gaussian(nb * B, d, it * 10 + 2), cfg, 1, sv)
        kt = port.random_gaussian(tail, d, it * 10 + 3) if tail else None
        vt = port.random_gaussian(tail, d, it * 10 + 4) if tail else None
        n_kv = nb * B + tail
        causal = bool(it % 2)
        n_q = 1 + int(rng.integers(0, n_kv)) if causal else 1 + int(rng.integers(0, 24))
        q = port.random_gaussian(n_q, d, it * 10 + 5)
        sc = np.float32(1 / np.sqrt(d))
        br = 1 + int(rng.integers(0, 24))
        assert port.prefill(q, kc, vc, kt, vt, causal, sc, br).tobytes() == \
            ref.prefill(q, kc, vc, kt, vt, causal, sc, br).tobytes()
        g = 1 + int(rng.integers(0, 4))
        qd = port.random_gaussian(g, d, it)
        spl = 1 + int(rng.integers(0, 6))
        assert port.decode(qd, kc, vc, kt, vt, sc, spl).tobytes() == \
            ref.decode(qd, kc, vc, kt, vt, sc, spl).tobytes()
        assert port.flop_and_byte_count(n_q, d, kc, vc, tail, causal) == \
            ref.flop_and_byte_count(n_q, d, kc, vc, tail, causal)


# ------------------------------------------------- compress (explicit mask) ----
def _masked_groups(rng, x, axis, block, cfg, port):
    """A valid HierarchicalMask from the pruner, then the flags it came with."""
    c = port.prune_compress(x, cfg, axis, cfg.s_key, element_mask=True)
    return c.element_mask.copy(), c.flags.copy()


@pytest.mark.parametrize("axis", [0, 1])
def test_compress_with_mask_equals_fused(port, ref, axis):
    """compress(cache, prune_cache mask) is field-identical to fused_magnitude_compress
    (test_compressor.cpp:114-134), in the port and in the reference."""
    rng = np.random.default_rng(3 + axis)
    x = port.round_to(rng.standard_normal((256, 32)).astype(np.float32), "bf16")
    cfg = SparsityConfig(0.5, 0.5, 16)
    em, flags = _masked_groups(rng, x, axis, 16, cfg, port)
    for o in (port, ref):
        a = o.compress_with_mask(x, cfg, axis, em, flags)
        b = o.compress_with_flags(x, cfg, axis, flags)
        assert (a.index_map == b.index_map).all() and (a.nnz_pool == b.nnz_pool).all()
        assert (a.meta_pool == b.meta_pool).all() and (a.dense_pool == b.dense_pool).all()


@pytest.mark.parametrize("axis", [0, 1])
def test_compress_with_mask_random_masks_port_equals_reference(port, ref, axis):
    """Arbitrary valid 2-of-4 masks (not magnitude-chosen): the port packs them
    exactly like the reference's compress."""
    rng = np.random.default_rng(11 + axis)
    rows, cols, B = 128, 16, 16
    x = rng.standard_normal((rows, cols)).astype(np.float32)
    em = np.zeros((rows, cols), np.uint8)
    pairs = [(0, 1), (0, 2), (0, 3), (1, 2), (1, 3), (2, 3)]
    for r in range(rows if axis == 0 else rows // 4):
        for g in range(cols // 4 if axis == 0 else cols):
            p = pairs[rng.integers(0, 6)]
            for i in p:
                if axis == 0:
                    em[r, 4 * g + i] = 1
                else:
                    em[4 * r + i, g] = 1
    flags = (rng.random(rows // B) < 0.3).astype(np.uint8)
    cfg = SparsityConfig(block_size=B)
    a, b = port.compress_with_mask(x, cfg, axis, em, flags), ref.compress_with_mask(x, cfg, axis, em, flags)
    for f in ("index_map", "dense_pool", "nnz_pool", "meta_pool"):
        assert (getattr(a, f) == getattr(b, f)).all(), f


@pytest.mark.parametrize("kept,msg", [(3, "more than n_keep"), (1, "fewer than n_keep"), (0, "fewer than n_keep")])
def test_compress_with_mask_rejects_bad_groups(port, ref, kept, msg):
    """compressed_cache.hpp:216-223: a sparse block's group keeping != 2 -> DataError."""
    x = np.arange(64, dtype=np.float32).reshape(16, 4)
    em = np.zeros((16, 4), np.uint8)
    em[:, :2] = 1
    em[5, :] = 0
    em[5, :kept] = 1
    for o in (port, ref):
        with pytest.raises(DataError, match=msg):
            o.compress_with_mask(x, SparsityConfig(block_size=4), 0, em, [0, 0, 0, 0])
    # the same group in a dense block is never consulted
    for o in (port, ref):
        o.compress_with_mask(x, SparsityConfig(block_size=4), 0, em, [0, 1, 0, 0])


def test_port_matches_small_shape_reference_fixtures(port):
    """The port at the reference's general (B, d) shapes reproduces the fixtures the
    compiled reference wrote (tests/golden/make_small_shapes.py)."""
    from oracle.oracle import SparsityConfig as OCfg
    g = np.load(os.path.join(os.path.dirname(GOLD), "small_shapes.npz"))
    f32 = lambda b: (b.astype(np.uint32) << 16).view(np.float32)  # noqa: E731
    for name in g["names"]:
        name = str(name)
        L, tail, d, B, gqa, n_q, sink, window = (int(x) for x in g[name + "_shape"])
        s = float(g[name + "_s"][0])
        key = f32(g[name + "_key"]).reshape(L + tail, d)
        val = f32(g[name + "_val"]).reshape(L + tail, d)
        cfg = OCfg(s, s, B, sink, window)
        kc = port.prune_compress(key[:L], cfg, 0, s)
        vc = port.prune_compress(val[:L], cfg, 1, s)
        for c, p in ((kc, name + "_k"), (vc, name + "_v")):
            assert (c.index_map == g[p + "_index_map"]).all(), name
            assert c.losses.tobytes() == g[p + "_losses"].tobytes(), name
            if c.sparse_count:
                assert (c.meta_pool == g[p + "_meta_pool"]).all(), name
        kt, vt = (key[L:], val[L:]) if tail else (None, None)
        scale = np.float32(1.0 / np.sqrt(d))
        out = port.decode(g[name + "_decode_q"], kc, vc, kt, vt, scale, 2)
        assert np.abs(out - g[name + "_decode_out"]).max() < 1e-5, name
