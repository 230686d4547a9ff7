"""GPU parity: hierarchical pruning + pooled 2:4 compression must match the
oracle bit for bit (index map, block flags, FP64 losses, dense / nnz / metadata
pools), through the C ABI (include/hierasparse_b200.h)."""
import os

import numpy as np
import pytest

from tests.helpers import device_to_oracle, gen_units, parallel, to_torch

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "reference_vectors.npz")


@pytest.fixture(scope="module")
def hs():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_2604_16864_b200 import hierasparse
    return hierasparse


def assert_cache_equal(dev, u, want, label=""):
    got = device_to_oracle(dev, u)
    assert got.dense_count == want.dense_count and got.sparse_count == want.sparse_count, label
    assert (got.index_map == want.index_map).all(), label
    assert (got.flags == want.flags).all(), label
    assert got.losses.tobytes() == want.losses.tobytes(), f"{label}: losses differ"
    if want.dense_count:
        assert (got.dense_pool == want.dense_pool).all(), f"{label}: dense pool"
    if want.sparse_count:
        assert (got.nnz_pool == want.nnz_pool).all(), f"{label}: nnz pool"
        assert (got.meta_pool == want.meta_pool).all(), f"{label}: meta pool"


CASES = [
    # rows, s, sink, window
    (4096, 1.0, 0, 0),
    (4096, 0.5, 64, 100),
    (2048, 0.25, 0, 0),
    (1024, 0.0, 0, 0),
    (512, 0.75, 1, 9),
    (640, 1.0, 70, 130),
]


@pytest.mark.parametrize("dtype", ["bf16", "f16"])
@pytest.mark.parametrize("rows,s,sink,window", CASES)
def test_prune_compress_matches_oracle(hs, port, dtype, rows, s, sink, window):
    from oracle.oracle import SparsityConfig as OCfg
    U = 3
    cfg = hs.SparsityConfig(s, s, 64, sink, window)
    ocfg = OCfg(s, s, 64, sink, window)
    for axis, role in ((0, 0), (1, 1)):
        x = gen_units(port, U, rows, 128, seed=11 + rows, role=role, dtype=dtype)
        dev = hs.prune_compress(to_torch(x, dtype), cfg, s, axis)
        wants = parallel(lambda u: port.prune_compress(x[u], ocfg, axis, s), range(U))
        for u in range(U):
            assert_cache_equal(dev, u, wants[u], f"axis={axis} unit={u}")
        # slot_block inverts the index map (dense slots first, then sparse slots)
        im = dev.index_map.cpu().numpy()
        sb = dev.slot_block.cpu().numpy()
        for u in range(U):
            for b, e in enumerate(im[u]):
                slot = e - 1 if e > 0 else dev.dense_count + (-e - 1)
                assert sb[u, slot] == b


@pytest.mark.parametrize("dtype", ["bf16", "f16"])
def test_ties_zeros_and_signed_zero(hs, port, dtype):
    from oracle.oracle import SparsityConfig as OCfg
    rng = np.random.default_rng(3)
    vals = np.array([0.0, -0.0, 1.0, -1.0, 2.0, -2.0, 0.5], np.float32)
    x = rng.choice(vals, size=(2, 1024, 128)).astype(np.float32)
    x[:, :64] = 0.0  # an all-zero block: ties keep positions {0, 1}
    for s in (1.0, 0.5):
        cfg, ocfg = hs.SparsityConfig(s, s, 64), OCfg(s, s, 64)
        for axis in (0, 1):
            dev = hs.prune_compress(to_torch(x, dtype), cfg, s, axis)
            for u in range(2):
                assert_cache_equal(dev, u, port.prune_compress(x[u], ocfg, axis, s), f"s={s} axis={axis}")


def test_loss_fallback_wide_dynamic_range(hs, port):
    """bf16 blocks whose pruned magnitudes span > 2^33 take the sequential
    FP64 path; losses must still be bit-identical to pruner.hpp:85-87."""
    from oracle.oracle import SparsityConfig as OCfg
    x = gen_units(port, 1, 512, 128, seed=5, role=0, dtype="bf16")
    x[0, ::7, ::5] *= np.float32(2.0 ** 60)
    x[0, 3::11, 1::3] *= np.float32(2.0 ** -60)
    x = port.round_to(x, "bf16")
    for s in (1.0, 0.5):
        for axis in (0, 1):
            dev = hs.prune_compress(to_torch(x, "bf16"), hs.SparsityConfig(s, s, 64), s, axis)
            assert_cache_equal(dev, 0, port.prune_compress(x[0], OCfg(s, s, 64), axis, s), f"axis={axis}")


def test_compress_with_flags(hs, port):
    import torch
    from oracle.oracle import SparsityConfig as OCfg
    x = gen_units(port, 2, 1024, 128, seed=9, role=0, dtype="bf16")
    flags = np.zeros((2, 16), np.uint8)
    flags[:, [0, 3, 4, 9, 15]] = 1
    for axis in (0, 1):
        dev = hs.fused_magnitude_compress(to_torch(x, "bf16"), torch.from_numpy(flags), hs.SparsityConfig(), axis)
        for u in range(2):
            want = port.compress_with_flags(x[u], OCfg(block_size=64), axis, flags[u])
            got = device_to_oracle(dev, u)
            assert (got.index_map == want.index_map).all()
            assert (got.dense_pool == want.dense_pool).all()
            assert (got.nnz_pool == want.nnz_pool).all()
            assert (got.meta_pool == want.meta_pool).all()


@pytest.mark.parametrize("s", [1.0, 0.5])
def test_decompress_matches_oracle(hs, port, s):
    from oracle.oracle import SparsityConfig as OCfg
    x = gen_units(port, 2, 2048, 128, seed=21, role=1, dtype="f16")
    for axis in (0, 1):
        dev = hs.prune_compress(to_torch(x, "f16"), hs.SparsityConfig(s, s, 64, 64, 64), s, axis)
        got = hs.decompress(dev).float().cpu().numpy()
        for u in range(2):
            want = port.decompress(port.prune_compress(x[u], OCfg(s, s, 64, 64, 64), axis, s))
            assert (got[u] == want).all()


def test_decompress_rejects_corrupt_index_map(hs, port):
    from paper_2604_16864_b200 import DataError
    x = gen_units(port, 1, 256, 128, seed=1, role=0, dtype="bf16")
    dev = hs.prune_compress(to_torch(x, "bf16"), hs.SparsityConfig(1, 1, 64), 1.0, 0)
    dev.index_map[0, 1] = 0
    with pytest.raises(DataError, match="index map holds a zero entry"):
        hs.decompress(dev)


def test_decompress_errors_in_reference_order(hs, port):
    """The first offending block in the reference's loop order decides the message
    (compressed_cache.hpp:277-287), whatever order the device blocks ran in; the
    messages are the oracle's.  The call itself never synchronises (check=False)."""
    import torch
    from oracle.oracle import SparsityConfig as OCfg
    x = gen_units(port, 2, 1024, 128, seed=2, role=1, dtype="bf16")
    dev = hs.prune_compress(to_torch(x, "bf16"), hs.SparsityConfig(0.5, 0.5, 64), 0.5, 1)
    dense_slot = int(dev.index_map[0][dev.index_map[0] > 0][0])
    sparse_b = int(torch.nonzero(dev.index_map[1] < 0)[0])
    dense_b = int(torch.nonzero(dev.index_map[1] > 0)[-1])
    dev.index_map[1, dense_b] = 100            # dangling dense offset (unit 1, late block)
    dev.meta_pool[1, -int(dev.index_map[1, sparse_b]) - 1, 5] = 0x0003  # codes (3, 0) in unit 1
    out = hs.decompress(dev, check=False)      # asynchronous: no raise, no sync
    first = "dangling dense offset" if dense_b < sparse_b else "codes not increasing"
    st = hs.StatusWord(out.device)
    hs.decompress(dev, check=False, status=st)
    with pytest.raises(hs.DataError, match=first):
        st.check()
    want_msg = None
    try:
        port.decompress(device_to_oracle(dev, 1))
    except Exception as e:  # noqa: BLE001
        want_msg = str(e)
    assert want_msg is not None and first in want_msg
    del dense_slot, out, OCfg


def test_dangling_sparse_offset_message(hs, port):
    x = gen_units(port, 1, 512, 128, seed=4, role=0, dtype="f16")
    dev = hs.prune_compress(to_torch(x, "f16"), hs.SparsityConfig(1, 1, 64), 1.0, 0)
    dev.index_map[0, 2] = -50
    with pytest.raises(hs.DataError, match="dangling sparse offset"):
        hs.decompress(dev)


@pytest.mark.parametrize("axis", [0, 1])
@pytest.mark.parametrize("dtype", ["bf16", "f16"])
def test_compress_with_element_mask_matches_oracle(hs, port, axis, dtype):
    """compress (compressed_cache.hpp:196-225) under an explicit HierarchicalMask:
    random valid 2-of-4 masks and a random block mask, bit-exact vs the oracle."""
    import torch
    from oracle.oracle import SparsityConfig as OCfg
    rng = np.random.default_rng(40 + axis)
    U, L, d = 2, 1024, 128
    x = gen_units(port, U, L, d, seed=17, role=axis, dtype=dtype)
    pairs = np.array([[1, 1, 0, 0], [1, 0, 1, 0], [1, 0, 0, 1], [0, 1, 1, 0], [0, 1, 0, 1], [0, 0, 1, 1]], np.uint8)
    if axis == 0:
        em = pairs[rng.integers(0, 6, (U, L, d // 4))].reshape(U, L, d)
    else:
        em = pairs[rng.integers(0, 6, (U, L // 4, d))].transpose(0, 1, 3, 2).reshape(U, L, d)
    nb = L // 64
    flags = np.zeros((U, nb), np.uint8)
    for u in range(U):
        flags[u, rng.choice(nb, 5, replace=False)] = 1
    dev = hs.compress(to_torch(x, dtype), torch.from_numpy(em), torch.from_numpy(flags), hs.SparsityConfig(), axis)
    for u in range(U):
        want = port.compress_with_mask(x[u], OCfg(block_size=64), axis, em[u], flags[u])
        got = device_to_oracle(dev, u)
        for f in ("index_map", "dense_pool", "nnz_pool", "meta_pool"):
            assert (getattr(got, f) == getattr(want, f)).all(), (u, f)


@pytest.mark.parametrize("axis", [0, 1])
def test_compress_with_element_mask_rejects_bad_groups(hs, port, axis):
    """The first group (unit, block, stored row, group order) keeping != 2 elements
    decides the DataError, as in the oracle; groups of dense blocks are ignored."""
    import torch
    from oracle.oracle import SparsityConfig as OCfg
    U, L, d = 1, 256, 128
    x = gen_units(port, U, L, d, seed=5, role=axis, dtype="bf16")
    em = np.zeros((U, L, d), np.uint8)
    if axis == 0:
        em[..., 0::4] = 1
        em[..., 1::4] = 1
    else:
        em[:, 0::4] = 1
        em[:, 1::4] = 1
    flags = np.array([[1, 0, 0, 0]], np.uint8)
    em[0, 10, 0:4] = 1 if axis == 0 else em[0, 10, 0:4]  # dense block 0: ignored
    if axis == 0:
        em[0, 64 + 3, 8:12] = [1, 1, 1, 0]    # block 1, stored row 3, group 2: three kept
        em[0, 128 + 1, 4:8] = [0, 1, 0, 0]    # block 2: one kept (later)
        msg = "more than n_keep"
    else:
        em[0, 64 + 4:64 + 8, 7] = [0, 0, 0, 1]  # block 1, channel 7, token group 1: one kept
        em[0, 128:132, 2] = [1, 1, 1, 1]        # block 2: four kept (later)
        msg = "fewer than n_keep"
    with pytest.raises(hs.DataError, match=msg):
        hs.compress(to_torch(x, "bf16"), torch.from_numpy(em), torch.from_numpy(flags), hs.SparsityConfig(), axis)
    with pytest.raises(Exception, match=msg):
        port.compress_with_mask(x[0], OCfg(block_size=64), axis, em[0], flags[0])


def test_block_mask_count_mismatch_is_config_error(hs, port):
    """Pooled units share one dense count: a unit whose BlockMask differs raises
    ConfigError from the device check, and no pool is written out of bounds."""
    import torch
    x = gen_units(port, 2, 512, 128, seed=6, role=0, dtype="bf16")
    flags = np.zeros((2, 8), np.uint8)
    flags[0, [1, 2]] = 1
    flags[1, [1, 2, 3, 4]] = 1
    with pytest.raises(hs.ConfigError, match="dense count"):
        hs.fused_magnitude_compress(to_torch(x, "bf16"), torch.from_numpy(flags), hs.SparsityConfig(), 0)


def test_golden_reference_vectors_on_gpu(hs):
    """Pools must equal the committed outputs of the compiled reference."""
    g = np.load(GOLD)
    to_f = lambda b: (b.astype(np.uint32) << 16).view(np.float32)  # noqa: E731
    key = to_f(g["key"]).reshape(-1, 128)[:256]
    val = to_f(g["val"]).reshape(-1, 128)[:256]
    for name in ("s50", "s100w", "s25"):
        for axis, x in ((0, key), (1, val)):
            p = f"{name}_{'k' if axis == 0 else 'v'}"
            s, sink, window = g[p + "_cfg"]
            dev = hs.prune_compress(to_torch(x[None], "bf16"), hs.SparsityConfig(s, s, 64, int(sink), int(window)),
                                    float(s), axis)
            got = device_to_oracle(dev, 0)
            assert (got.index_map == g[p + "_index_map"]).all()
            assert (got.flags == g[p + "_flags"]).all()
            assert got.losses.tobytes() == g[p + "_losses"].tobytes()
            if got.dense_count:
                assert (got.dense_pool == to_f(g[p + "_dense_pool"])).all()
            if got.sparse_count:
                assert (got.nnz_pool == to_f(g[p + "_nnz_pool"])).all()
                assert (got.meta_pool == g[p + "_meta_pool"]).all()


def test_golden_reference_attention_on_gpu(hs, port):
    """Decode (3 splits) and causal prefill with the 17-token dense tail against the
    reference's own committed outputs (tests/golden/make_golden.py), on the GPU box
    where /root/reference is absent."""
    import math
    from tests.helpers import MAX_ABS_TOL, MEAN_REL_TOL, err_stats
    g = np.load(GOLD)
    to_f = lambda b: (b.astype(np.uint32) << 16).view(np.float32)  # noqa: E731
    key = to_f(g["key"]).reshape(-1, 128)
    val = to_f(g["val"]).reshape(-1, 128)
    L = 256
    scale = 1.0 / math.sqrt(128)
    for name in ("s50", "s100w", "s25"):
        s, sink, window = g[name + "_k_cfg"]
        kc, vc = hs.prune_cache(to_torch(key[None, :L], "bf16"), to_torch(val[None, :L], "bf16"),
                                hs.SparsityConfig(float(s), float(s), 64, int(sink), int(window)))
        kt, vt = to_torch(key[None, L:], "bf16"), to_torch(val[None, L:], "bf16")
        out = hs.decode_attention(to_torch(g[name + "_decode_q"][None], "bf16"), kc, vc, kt, vt, scale=scale, splits=3)
        mx, mr = err_stats(out[0].cpu().numpy(), g[name + "_decode_out"])
        assert mx < MAX_ABS_TOL and mr < MEAN_REL_TOL, (name, "decode", mx, mr)
        # prefill queries: the generator stream of make_golden.py (role 2, seed 7), regenerated by the port
        qp = port.round_to(port.random_gaussian(L + 17, 128, port.head_seed(7, 0, 2)), "bf16")
        outp = hs.prefill_attention(to_torch(qp[None, None], "bf16"), kc, vc, kt, vt, causal=True, scale=scale)
        mx, mr = err_stats(outp[0, 0].cpu().numpy(), g[name + "_prefill_out"])
        assert mx < MAX_ABS_TOL and mr < MEAN_REL_TOL, (name, "prefill", mx, mr)


def test_config2_full_size_compression(hs, port):
    """Config 2 geometry (8 KV heads x 128K, S=1): bit-exact on two heads,
    structural properties on all (every sparse block decodes to a 2:4 pattern
    whose kept values are the group's two largest magnitudes)."""
    from oracle.oracle import SparsityConfig as OCfg
    import torch
    U, L = 8, 131072
    torch.manual_seed(0)
    x = torch.randn(U, L, 128, device="cuda").to(torch.bfloat16)
    for axis in (0, 1):
        dev = hs.prune_compress(x, hs.SparsityConfig(1, 1, 64), 1.0, axis)
        assert dev.sparse_count == 2048 and dev.dense_count == 0
        xs = x[[0, 5]].float().cpu().numpy()
        for i, u in enumerate((0, 5)):
            assert_cache_equal(dev, u, port.prune_compress(xs[i], OCfg(1, 1, 64), axis, 1.0), f"unit {u}")
        # round trip on every unit: decompress keeps exactly the top-2 per group
        dec = hs.decompress(dev).float()
        grp = (x.float().reshape(U, L, 32, 4) if axis == 0 else
               x.float().reshape(U, L // 4, 4, 128).transpose(2, 3))
        dgrp = (dec.reshape(U, L, 32, 4) if axis == 0 else dec.reshape(U, L // 4, 4, 128).transpose(2, 3))
        assert ((dgrp != 0).sum(-1) <= 2).all()
        kept = torch.where(dgrp != 0, grp.abs(), torch.zeros_like(grp)).sum(-1)
        top2 = grp.abs().topk(2, dim=-1).values.sum(-1)
        assert torch.equal(kept, top2)


@pytest.mark.parametrize("dtype", ["bf16", "f16"])
@pytest.mark.parametrize("s_pre,s_dec", [(0.0, 1.0), (0.5, 1.0), (0.25, 0.75)])
def test_decode_phase_recompress_matches_oracle(hs, port, dtype, s_pre, s_dec):
    """Prefill-sparsity caches re-pruned at the decode sparsity (pipeline.hpp:227-240):
    GPU recompress == oracle decompress -> prune_compress, bit for bit."""
    from oracle.oracle import SparsityConfig as OCfg
    U, L = 2, 1024
    kx = gen_units(port, U, L, 128, 21, 0, dtype)
    vx = gen_units(port, U, L, 128, 21, 1, dtype)
    kc, vc = hs.prune_cache(to_torch(kx, dtype), to_torch(vx, dtype), hs.SparsityConfig(s_pre, s_pre, 64))
    cfg_dec = hs.SparsityConfig(s_dec, s_dec, 64)
    k2, v2 = hs.recompress_pair(kc, vc, cfg_dec, with_losses=True)
    for dev_old, dev_new, axis in ((kc, k2, 0), (vc, v2, 1)):
        for u in range(U):
            dense = port.decompress(device_to_oracle(dev_old, u))
            want = port.prune_compress(dense, OCfg(s_dec, s_dec, 64), axis, s_dec)
            assert_cache_equal(dev_new, u, want, f"recompress axis={axis} unit={u}")


@pytest.mark.parametrize("dtype", ["bf16", "f16"])
@pytest.mark.parametrize("s_pre,s_dec", [(0.0, 0.5), (0.5, 0.25), (1.0, 1.0), (0.75, 0.0)])
def test_fused_recompress_equals_decompress_then_compress(hs, port, dtype, s_pre, s_dec):
    """hs_recompress (one pass over the input pools) == hs_decompress followed by
    hs_prune_compress on the device: pools, index map, flags and losses bit for
    bit, with sink / window protection in play."""
    import torch
    U, L = 3, 2048
    kx = gen_units(port, U, L, 128, 33, 0, dtype)
    vx = gen_units(port, U, L, 128, 33, 1, dtype)
    pre = hs.SparsityConfig(s_pre, s_pre, 64, sink_tokens=64, local_window=128)
    kc, vc = hs.prune_cache(to_torch(kx, dtype), to_torch(vx, dtype), pre)
    dec = hs.SparsityConfig(s_dec, s_dec, 64, sink_tokens=128, local_window=64)
    for c in (kc, vc):
        a = hs.recompress(c, dec, s_dec)
        b = hs.recompress_unfused(c, dec, s_dec)
        for name in ("index_map", "dense_pool", "nnz_pool", "meta_pool", "flags"):
            x, y = getattr(a, name), getattr(b, name)
            if x.is_floating_point():
                x, y = x.view(torch.int16), y.view(torch.int16)
            assert torch.equal(x, y), name
        if 0.0 < s_dec < 1.0:  # loss-driven selection computes every block's loss
            assert torch.equal(a.losses, b.losses)


@pytest.mark.parametrize("s_pre,s_dec", [(1.0, 1.0), (0.5, 1.0), (1.0, 0.5)])
def test_recompress_with_kept_zeros(hs, port, s_pre, s_dec):
    """Inputs with exact zeros (a third of the values): stored 2:4 groups keep
    zeros, so re-pruning may move their codes by the tie rule -- the blocks the
    stored-to-stored copy must not take.  Fused == the oracle chain, bit for bit."""
    import torch
    from oracle.oracle import SparsityConfig as OCfg
    rng = np.random.default_rng(77)
    U, L = 2, 2048
    kx = gen_units(port, U, L, 128, 34, 0, "bf16")
    vx = gen_units(port, U, L, 128, 34, 1, "bf16")
    for x in (kx, vx):
        x[rng.random(x.shape) < 0.35] = 0.0
        x[:, 640:704] = 0.0  # one all-zero block
    pre = hs.SparsityConfig(s_pre, s_pre, 64)
    kc, vc = hs.prune_cache(to_torch(kx, "bf16"), to_torch(vx, "bf16"), pre)
    dec = hs.SparsityConfig(s_dec, s_dec, 64)
    for c in (kc, vc):
        got = hs.recompress(c, dec, s_dec, with_losses=True)
        for u in range(U):
            want = port.prune_compress(port.decompress(device_to_oracle(c, u)), OCfg(s_dec, s_dec, 64), c.axis, s_dec)
            g = device_to_oracle(got, u)
            for f in ("index_map", "dense_pool", "nnz_pool", "meta_pool"):
                assert (getattr(g, f) == getattr(want, f)).all(), (u, f)
            assert g.losses.tobytes() == want.losses.tobytes()
    del torch


def test_recompress_rejects_corrupt_input(hs, port):
    """A zero index entry or non-increasing codes in the input: decompress's DataError."""
    U, L = 1, 512
    kx = gen_units(port, U, L, 128, 5, 0, "bf16")
    kc = hs.prune_compress(to_torch(kx, "bf16"), hs.SparsityConfig(1.0, 1.0, 64), 1.0, 0)
    bad = hs.recompress(kc, hs.SparsityConfig(1.0, 1.0, 64), 1.0)
    bad.index_map[0, 3] = 0
    with pytest.raises(hs.DataError, match="zero entry"):
        hs.recompress(bad, hs.SparsityConfig(0.5, 0.5, 64), 0.5)
    bad2 = hs.recompress(kc, hs.SparsityConfig(1.0, 1.0, 64), 1.0)
    bad2.meta_pool[0, 0, 0] = 0x0003  # first group codes (3, 0): not increasing
    with pytest.raises(hs.DataError, match="not increasing"):
        hs.recompress(bad2, hs.SparsityConfig(1.0, 1.0, 64), 1.0)


@pytest.mark.parametrize("dtype", ["bf16", "f16"])
@pytest.mark.parametrize("s_dec,tail_rows", [(1.0, 200), (0.5, 128), (0.25, 64)])
def test_absorb_tail_matches_oracle(hs, port, dtype, s_dec, tail_rows):
    """Dense-tail growth: the cache's blocks plus the tail's
    whole blocks re-pruned in one pass == oracle prune_compress of
    [decompress(cache); tail blocks], bit for bit; the partial block stays a tail."""
    import torch
    from oracle.oracle import SparsityConfig as OCfg
    U, L = 2, 1024
    kx = gen_units(port, U, L + tail_rows, 128, 41, 0, dtype)
    vx = gen_units(port, U, L + tail_rows, 128, 41, 1, dtype)
    kt, vt = to_torch(kx, dtype), to_torch(vx, dtype)
    kc, vc = hs.prune_cache(kt[:, :L].contiguous(), vt[:, :L].contiguous(), hs.SparsityConfig(0.5, 0.5, 64))
    cfg = hs.SparsityConfig(s_dec, s_dec, 64, sink_tokens=64)
    k2, v2, krest, vrest = hs.absorb_tail_pair(kc, vc, kt[:, L:], vt[:, L:], cfg, with_losses=True)
    full = (tail_rows // 64) * 64
    assert k2.logical_blocks == (L + full) // 64 and krest.shape[1] == tail_rows - full
    assert torch.equal(krest.view(torch.int16), kt[:, L + full:].view(torch.int16))
    for dev_old, dev_new, axis, src in ((kc, k2, 0, kx), (vc, v2, 1, vx)):
        for u in range(U):
            dense = port.decompress(device_to_oracle(dev_old, u))
            grown = np.concatenate([dense, np.asarray(src[u])[L:L + full]], axis=0)
            want = port.prune_compress(grown, OCfg(s_dec, s_dec, 64, sink_tokens=64), axis, s_dec)
            assert_cache_equal(dev_new, u, want, f"absorb_tail axis={axis} unit={u}")
    # the grown cache and its remaining tail decode like any other cache
    q = torch.randn(U, 4, 128, device="cuda").to(kt.dtype)
    out = hs.decode_attention(q, k2, v2, krest, vrest)
    assert torch.isfinite(out).all()


def test_absorb_tail_without_whole_block_is_a_noop(hs, port):
    import torch
    U, L = 1, 256
    kx = gen_units(port, U, L + 10, 128, 3, 0, "bf16")
    kt = to_torch(kx, "bf16")
    kc = hs.prune_compress(kt[:, :L].contiguous(), hs.SparsityConfig(1.0, 1.0, 64), 1.0, 0)
    k2, rest = hs.absorb_tail(kc, kt[:, L:], hs.SparsityConfig(1.0, 1.0, 64), 1.0)
    assert k2 is kc and rest.shape[1] == 10


@pytest.mark.parametrize("axis_name", ["key", "value"])
def test_nan_losses_flag_exactly_quota_blocks(hs, port, axis_name):
    """Blocks whose pruned values are NaN (an all-NaN token row, e.g. fp16 overflow)
    get a NaN loss.  Selection orders NaN as the largest loss, so exactly
    floor(S * prunable) blocks are sparse, the index map is a permutation of the
    pool slots and decompress reads it back without a DataError (ADVICE: a NaN
    rank once flagged extra blocks and packed past the sparse pool)."""
    import torch
    U, rows, s = 2, 2048, 0.5
    x = gen_units(port, U, rows, 128, 5, 0, "f16")
    # three NaN token rows inside one group of 4 tokens: NaN pruned values along both
    # axes (key: whole channel groups; value: 3 NaN of a 4-token group)
    x[0, 64 * 3 + 4:64 * 3 + 7, :] = np.nan    # block 3 of unit 0
    x[1, 64 * 10:64 * 10 + 3, :] = np.nan      # block 10 of unit 1
    xt = to_torch(x, "f16")
    cfg = hs.SparsityConfig(s, s, 64)
    axis = 0 if axis_name == "key" else 1
    c = hs.prune_compress(xt, cfg, s, axis)
    nb = rows // 64
    quota = int(np.floor(s * nb))
    im = c.index_map.cpu().numpy()
    for u in range(U):
        assert (im[u] < 0).sum() == quota and (im[u] > 0).sum() == nb - quota
        assert sorted(-im[u][im[u] < 0] - 1) == list(range(quota))
        assert sorted(im[u][im[u] > 0] - 1) == list(range(nb - quota))
    losses = c.losses.cpu().numpy()
    assert np.isnan(losses[0, 3]) and np.isnan(losses[1, 10])
    assert im[0, 3] > 0 and im[1, 10] > 0  # NaN loss = largest: kept dense
    out = hs.decompress(c)
    torch.cuda.synchronize()
    assert out.shape == xt.shape


@pytest.mark.parametrize("nb,prefix,suffix", [(2048, 0, 0), (3000, 5, 17), (16384, 1, 4), (40, 3, 2)])
@pytest.mark.parametrize("s", [0.0, 0.1, 0.5, 0.9, 1.0])
def test_select_blocks_radix_matches_stable_sort(hs, nb, prefix, suffix, s):
    """hs_select_blocks (radix select) against select_blocks' stable ascending sort
    (pruner.hpp:94-117): ties to the lower index (heavy ties drawn from a few values,
    -0.0 == +0.0), NaN above +inf, protected prefix/suffix dense, exactly
    floor(S * prunable) sparse."""
    import torch
    rng = np.random.default_rng(nb + int(100 * s))
    U = 3
    losses = rng.integers(0, 7, size=(U, nb)).astype(np.float64) * 0.25
    losses[0, rng.integers(0, nb, 5)] = np.nan
    losses[1, rng.integers(0, nb, 5)] = -0.0
    losses[2, rng.integers(0, nb, 5)] = np.inf
    sink, window = prefix * 64, suffix * 64
    cfg = hs.SparsityConfig(s, s, 64, sink, window)
    got = hs.select_blocks(torch.from_numpy(losses).cuda(), cfg, s).cpu().numpy()
    np_ = nb - prefix - suffix
    quota = int(np.floor(s * np_))
    for u in range(U):
        want = np.ones(nb, np.uint8)
        lp = losses[u, prefix:nb - suffix]
        order = np.lexsort((np.arange(np_), np.nan_to_num(lp, nan=0.0, posinf=np.inf), np.isnan(lp)))
        want[prefix + order[:quota]] = 0
        assert (got[u] == want).all(), (u, np.nonzero(got[u] != want)[0][:10])


def test_pair_entry_points_match_single_cache_calls(hs, port):
    """prune_cache / recompress_pair run the value cache on a side stream: results
    equal the single-cache calls on the caller's stream, bit for bit."""
    import torch
    U, rows = 3, 4096
    kx = to_torch(gen_units(port, U, rows, 128, 21, 0, "bf16"), "bf16")
    vx = to_torch(gen_units(port, U, rows, 128, 21, 1, "bf16"), "bf16")
    cfg = hs.SparsityConfig(0.5, 0.75, 64, 64, 128)
    kc, vc = hs.prune_cache(kx, vx, cfg)
    k1 = hs.prune_compress(kx, cfg, cfg.s_key, 0)
    v1 = hs.prune_compress(vx, cfg, cfg.s_value, 1)
    dec = hs.SparsityConfig(1.0, 1.0, 64, 64, 128)
    k2, v2 = hs.recompress_pair(kc, vc, dec)
    k3, v3 = hs.recompress(kc, dec, 1.0), hs.recompress(vc, dec, 1.0)
    torch.cuda.synchronize()
    for a, b in ((kc, k1), (vc, v1), (k2, k3), (v2, v3)):
        for u in range(U):
            assert_cache_equal(a, u, device_to_oracle(b, u))


@pytest.mark.parametrize("s", [1.0, 0.0])
def test_static_selection_skips_losses(hs, port, s):
    """A static selection (quota 0 or every prunable block) needs no block loss:
    prune_cache / recompress leave losses as NaN unless with_losses, and every
    pool, index entry and flag is identical either way."""
    import torch
    U, L = 2, 2048
    kx = to_torch(gen_units(port, U, L, 128, 61, 0, "bf16"), "bf16")
    vx = to_torch(gen_units(port, U, L, 128, 61, 1, "bf16"), "bf16")
    cfg = hs.SparsityConfig(s, s, 64, sink_tokens=64, local_window=128)
    fast = hs.prune_cache(kx, vx, cfg)
    full = hs.prune_cache(kx, vx, cfg, with_losses=True)
    for a, b in zip(fast, full):
        assert torch.isnan(a.losses).all() and not torch.isnan(b.losses).any()
        for name in ("index_map", "dense_pool", "nnz_pool", "meta_pool", "flags", "slot_block"):
            x, y = getattr(a, name), getattr(b, name)
            if x.is_floating_point():
                x, y = x.view(torch.int16), y.view(torch.int16)
            assert torch.equal(x, y), name
    r_fast, r_full = hs.recompress(full[0], cfg, s), hs.recompress(full[0], cfg, s, with_losses=True)
    assert torch.isnan(r_fast.losses).all() and not torch.isnan(r_full.losses).any()
    assert torch.equal(r_fast.nnz_pool.view(torch.int16), r_full.nnz_pool.view(torch.int16))
