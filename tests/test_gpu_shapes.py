"""GPU parity at the reference's general shapes (block size B and head dim d any
multiples of the 2:4 group, masks.hpp:87 / pruner.hpp:172-173; GQA groups above
8 rows): the device path against fixtures produced by the UNMODIFIED reference
(tests/golden/small_shapes.npz, tests/golden/make_small_shapes.py) -- pools,
index maps, flags and losses bit-exact; decode / causal prefill with a ragged
dense tail within the north-star bar."""
import os

import numpy as np
import pytest

from tests.helpers import MAX_ABS_TOL, MEAN_REL_TOL, device_to_oracle, err_stats, to_torch

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "small_shapes.npz")


@pytest.fixture(scope="module")
def hs():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_2604_16864_b200 import hierasparse
    return hierasparse


@pytest.fixture(scope="module")
def gold():
    return np.load(GOLD)


def f32(bits):
    return (bits.astype(np.uint32) << 16).view(np.float32)


def caches(hs, g, name):
    L, tail, d, B, gqa, n_q, sink, window = (int(x) for x in g[name + "_shape"])
    s = float(g[name + "_s"][0])
    key = f32(g[name + "_key"]).reshape(L + tail, d)
    val = f32(g[name + "_val"]).reshape(L + tail, d)
    cfg = hs.SparsityConfig(s, s, B, sink, window)
    kc, vc = hs.prune_cache(to_torch(key[None, :L], "bf16"), to_torch(val[None, :L], "bf16"), cfg, with_losses=True)
    return key, val, kc, vc, (L, tail, d, B, gqa, n_q)


NAMES = ["b4d8", "b16d32", "b32d64", "b64d64", "b128d256", "b8d128", "b64d128g12"]


@pytest.mark.parametrize("name", NAMES)
def test_compression_matches_reference_fixture(hs, gold, name):
    _, _, kc, vc, _ = caches(hs, gold, name)
    for c, p in ((kc, name + "_k"), (vc, name + "_v")):
        got = device_to_oracle(c, 0)
        assert (got.index_map == gold[p + "_index_map"]).all()
        assert (got.flags == gold[p + "_flags"]).all()
        assert got.losses.tobytes() == gold[p + "_losses"].tobytes()
        if c.dense_count:
            assert (got.dense_pool == f32(gold[p + "_dense_pool"])).all()
        if c.sparse_count:
            assert (got.nnz_pool == f32(gold[p + "_nnz_pool"])).all()
            assert (got.meta_pool == gold[p + "_meta_pool"]).all()


@pytest.mark.parametrize("name", NAMES)
def test_decompress_and_recompress_general_shapes(hs, gold, port, name):
    from oracle.oracle import SparsityConfig as OCfg
    key, val, kc, vc, (L, tail, d, B, gqa, n_q) = caches(hs, gold, name)
    for c, x in ((kc, key[:L]), (vc, val[:L])):
        dec = hs.decompress(c).float().cpu().numpy()[0]
        want = port.decompress(device_to_oracle(c, 0))
        assert (dec == want).all()
        # decode-phase re-prune to S = 1 (pipeline.hpp:227-240), fused, vs the oracle chain
        cfg = hs.SparsityConfig(1.0, 1.0, B)
        r = hs.recompress(c, cfg, 1.0, with_losses=True)
        w = port.prune_compress(want, OCfg(1.0, 1.0, B), c.axis, 1.0)
        got = device_to_oracle(r, 0)
        assert (got.index_map == w.index_map).all() and (got.nnz_pool == w.nnz_pool).all()
        assert (got.meta_pool == w.meta_pool).all() and got.losses.tobytes() == w.losses.tobytes()
        del x


@pytest.mark.parametrize("name", NAMES)
def test_decode_matches_reference_fixture(hs, gold, name):
    key, val, kc, vc, (L, tail, d, B, gqa, n_q) = caches(hs, gold, name)
    q = gold[name + "_decode_q"]
    kt = to_torch(key[None, L:], "bf16") if tail else None
    vt = to_torch(val[None, L:], "bf16") if tail else None
    scale = float(np.float32(1.0 / np.sqrt(d)))
    got = hs.decode_attention(to_torch(q[None], "bf16"), kc, vc, kt, vt, scale=scale).cpu().numpy()[0]
    mx, mr = err_stats(got, gold[name + "_decode_out"])
    assert mx < MAX_ABS_TOL and mr < MEAN_REL_TOL, (mx, mr)
    for splits in (1, 3):
        got2 = hs.decode_attention(to_torch(q[None], "bf16"), kc, vc, kt, vt, scale=scale, splits=splits)
        mx, mr = err_stats(got2.cpu().numpy()[0], gold[name + "_decode_out"])
        assert mx < MAX_ABS_TOL and mr < MEAN_REL_TOL, (splits, mx, mr)


@pytest.mark.parametrize("name", NAMES)
def test_prefill_matches_reference_fixture(hs, gold, name):
    key, val, kc, vc, (L, tail, d, B, gqa, n_q) = caches(hs, gold, name)
    q = gold[name + "_prefill_q"]
    kt = to_torch(key[None, L:], "bf16") if tail else None
    vt = to_torch(val[None, L:], "bf16") if tail else None
    scale = float(np.float32(1.0 / np.sqrt(d)))
    got = hs.prefill_attention(to_torch(q[None, None], "bf16"), kc, vc, kt, vt, causal=True, scale=scale)
    mx, mr = err_stats(got.cpu().numpy()[0, 0], gold[name + "_prefill_out"])
    assert mx < MAX_ABS_TOL and mr < MEAN_REL_TOL, (mx, mr)


@pytest.mark.parametrize("name", ["b16d32", "b64d64"])
def test_decode_partial_combine_general_shapes(hs, gold, name):
    """attend_range partials over two block ranges + the LSE combine equal the
    one-pass decode (attention.hpp:380-407) at a generic shape."""
    import torch
    key, val, kc, vc, (L, tail, d, B, gqa, n_q) = caches(hs, gold, name)
    q = to_torch(gold[name + "_decode_q"][None], "bf16")
    nb = L // B
    kt = to_torch(key[None, L:], "bf16") if tail else None
    vt = to_torch(val[None, L:], "bf16") if tail else None
    parts = torch.stack([hs.decode_partial(q, kc, vc, 0, nb // 2, kt, vt, include_tail=False),
                         hs.decode_partial(q, kc, vc, nb // 2, nb, kt, vt, include_tail=True)])
    got = hs.decode_combine(parts).cpu().numpy()[0]
    mx, mr = err_stats(got, gold[name + "_decode_out"])
    assert mx < MAX_ABS_TOL and mr < MEAN_REL_TOL, (mx, mr)
