"""GPU parity: tcgen05 Trans-Both prefill (attention.hpp:323-354) against the
fp32 oracle on identical 16-bit inputs, within max-abs 2e-2 / mean-rel 1e-3.
Large shapes are checked on sampled query rows through attend_range with
explicit positions (attention.hpp:249-253), exactly the reference arithmetic
restricted to those rows."""
import math

import numpy as np
import pytest

from tests.helpers import MAX_ABS_TOL, MEAN_REL_TOL, device_to_oracle, err_stats, gen_units, parallel, to_torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def hs():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_2604_16864_b200 import hierasparse
    return hierasparse


def setup(hs, port, U, L, s, dtype, gqa, n_q, sink=0, window=0, seed=3):
    kx = gen_units(port, U, L, 128, seed, 0, dtype)
    vx = gen_units(port, U, L, 128, seed, 1, dtype)
    kc, vc = hs.prune_cache(to_torch(kx, dtype), to_torch(vx, dtype), hs.SparsityConfig(s, s, 64, sink, window))
    # prefill Q streams: role 2 + g (pipeline.hpp:202-203), last n_q rows
    q = np.stack([np.stack([port.round_to(port.random_gaussian(n_q, 128, port.head_seed(seed, u, 2 + g)), dtype)
                            for g in range(gqa)]) for u in range(U)])
    return kc, vc, q


@pytest.mark.parametrize("dtype", ["f16", "bf16"])
@pytest.mark.parametrize("L,n_q,s,sink,window,causal", [
    (512, 512, 1.0, 0, 0, True),
    (512, 512, 0.0, 0, 0, True),
    (1024, 1024, 0.5, 64, 128, True),
    (1024, 300, 0.75, 0, 0, True),    # queries at the end of the sequence, partial tile
    (768, 256, 0.25, 0, 0, False),
    (640, 640, 1.0, 70, 200, True),   # odd block count, protected sink/window
])
def test_prefill_matches_oracle(hs, port, dtype, L, n_q, s, sink, window, causal):
    U, gqa = 2, 2
    kc, vc, q = setup(hs, port, U, L, s, dtype, gqa, n_q, sink, window)
    scale = np.float32(1.0 / math.sqrt(128))
    got = hs.prefill_attention(to_torch(q, dtype), kc, vc, causal=causal, scale=float(scale)).cpu().numpy()

    def one(ug):
        u, g = divmod(ug, gqa)
        return port.prefill(q[u, g], device_to_oracle(kc, u), device_to_oracle(vc, u), None, None, causal, scale, 64)
    want = np.stack(parallel(one, range(U * gqa))).reshape(U, gqa, n_q, 128)
    mx, mr = err_stats(got, want)
    assert mx < MAX_ABS_TOL and mr < MEAN_REL_TOL, (mx, mr)


@pytest.mark.parametrize("hg", [2, 4])
@pytest.mark.parametrize("dtype,L,n_q,s,causal", [
    ("f16", 1024, 1024, 1.0, True),
    ("f16", 1024, 300, 0.5, True),    # partial query tiles of every stacked head
    ("bf16", 768, 256, 0.25, False),
])
def test_prefill_gqa_stacked(hs, port, monkeypatch, hg, dtype, L, n_q, s, causal):
    """hg query heads of one KV head per CTA (HS_PREFILL_HG): column c of the
    128-column tile is head c / (128 / hg), query c % (128 / hg)."""
    monkeypatch.setenv("HS_PREFILL_HG", str(hg))
    U, gqa = 2, 4
    kc, vc, q = setup(hs, port, U, L, s, dtype, gqa, n_q)
    scale = np.float32(1.0 / math.sqrt(128))
    got = hs.prefill_attention(to_torch(q, dtype), kc, vc, causal=causal, scale=float(scale)).cpu().numpy()

    def one(ug):
        u, g = divmod(ug, gqa)
        return port.prefill(q[u, g], device_to_oracle(kc, u), device_to_oracle(vc, u), None, None, causal, scale, 64)
    want = np.stack(parallel(one, range(U * gqa))).reshape(U, gqa, n_q, 128)
    mx, mr = err_stats(got, want)
    assert mx < MAX_ABS_TOL and mr < MEAN_REL_TOL, (mx, mr)


@pytest.mark.parametrize("s", [1.0, 0.5])
def test_prefill_sampled_rows_8k(hs, port, s):
    """8K causal prefill; 96 sampled query rows per head (block boundaries,
    first/last rows, random) through the oracle's attend_range."""
    U, gqa, L = 1, 2, 8192
    kc, vc, q = setup(hs, port, U, L, s, "f16", gqa, L, seed=5)
    scale = np.float32(1.0 / math.sqrt(128))
    got = hs.prefill_attention(to_torch(q, "f16"), kc, vc, causal=True, scale=float(scale)).cpu().numpy()
    rng = np.random.default_rng(0)
    rows = sorted(set([0, 1, 63, 64, 127, 128, 4095, 4096, L - 1] + list(rng.integers(0, L, 87))))
    k0, v0 = device_to_oracle(kc, 0), device_to_oracle(vc, 0)

    def one(g):
        qr = q[0, g][rows]
        out_t, m, l = port.attend_rows(qr, k0, v0, None, None, 0, k0.logical_blocks, True, scale,
                                       np.array(rows, np.int64))
        return (out_t / l[None, :]).T
    want = np.stack(parallel(one, range(gqa)))
    mx, mr = err_stats(got[0][:, rows], want)
    assert mx < MAX_ABS_TOL and mr < MEAN_REL_TOL, (mx, mr)


@pytest.mark.parametrize("dtype", ["f16", "bf16"])
@pytest.mark.parametrize("s,causal", [(1.0, True), (0.5, True), (0.0, False)])
def test_prefill_growing_scores(hs, port, dtype, s, causal):
    """Keys scaled by a ramp along the sequence (and one hot block late in it),
    so column maxima grow tile after tile: exercises the lazy-rescale slow path
    (running max update, O^T / l rescale) against the oracle."""
    U, gqa, L, n_q = 1, 2, 2048, 2048
    kx = np.stack([port.random_gaussian(L, 128, port.head_seed(11, u, 0)) for u in range(U)])
    ramp = (1.0 + 3.0 * np.arange(L, dtype=np.float32) / L)[None, :, None]
    kx = kx * ramp
    kx[:, 1600:1664] *= 4.0
    kx = port.round_to(kx.astype(np.float32), dtype)
    vx = gen_units(port, U, L, 128, 11, 1, dtype)
    kc, vc = hs.prune_cache(to_torch(kx, dtype), to_torch(vx, dtype), hs.SparsityConfig(s, s, 64))
    q = np.stack([np.stack([port.round_to(port.random_gaussian(n_q, 128, port.head_seed(11, u, 2 + g)) * 2.0, dtype)
                            for g in range(gqa)]) for u in range(U)])
    scale = np.float32(1.0 / math.sqrt(128))
    got = hs.prefill_attention(to_torch(q, dtype), kc, vc, causal=causal, scale=float(scale)).cpu().numpy()

    def one(g):
        return port.prefill(q[0, g], device_to_oracle(kc, 0), device_to_oracle(vc, 0), None, None, causal, scale, 64)
    want = np.stack(parallel(one, range(gqa)))[None]
    mx, mr = err_stats(got, want)
    assert mx < MAX_ABS_TOL and mr < MEAN_REL_TOL, (mx, mr)


@pytest.mark.parametrize("dtype", ["f16", "bf16"])
@pytest.mark.parametrize("qscale,negative", [(24.0, False), (24.0, True), (0.01, False)])
def test_prefill_logit_ranges(hs, port, dtype, qscale, negative):
    """Very large logits (|s| ~ 10^3: the running max lives in the 16-bit bias
    operand of GEMM1, rounded), all-negative large logits (every column's max far
    below zero) and near-uniform attention (tiny logits): the stabiliser may be any
    representable value as long as P and the rescale factors use it consistently."""
    U, gqa, L, n_q = 1, 2, 1024, 1024
    kx = gen_units(port, U, L, 128, 13, 0, dtype)
    vx = gen_units(port, U, L, 128, 13, 1, dtype)
    if negative:  # one shared direction pushed far negative for every key
        kx = kx.copy()
        kx[..., 0] = -40.0
    kx = port.round_to(kx.astype(np.float32), dtype)
    kc, vc = hs.prune_cache(to_torch(kx, dtype), to_torch(vx, dtype), hs.SparsityConfig(1.0, 1.0, 64))
    q = np.stack([np.stack([port.random_gaussian(n_q, 128, port.head_seed(13, u, 2 + g)) * qscale
                            for g in range(gqa)]) for u in range(U)]).astype(np.float32)
    if negative:
        q[..., 0] = np.abs(q[..., 0]) + 30.0
    q = port.round_to(q, dtype)
    scale = np.float32(1.0 / math.sqrt(128))
    got = hs.prefill_attention(to_torch(q, dtype), kc, vc, causal=True, scale=float(scale)).cpu().numpy()
    assert np.isfinite(got).all()

    def one(g):
        return port.prefill(q[0, g], device_to_oracle(kc, 0), device_to_oracle(vc, 0), None, None, True, scale, 64)
    want = np.stack(parallel(one, range(gqa)))[None]
    mx, mr = err_stats(got, want)
    assert mx < MAX_ABS_TOL and mr < MEAN_REL_TOL, (mx, mr)


@pytest.mark.parametrize("dtype", ["f16", "bf16"])
@pytest.mark.parametrize("L,tail,n_q,s,causal", [
    (512, 17, 529, 1.0, True),     # golden-vector shape: 4 blocks + 17-token tail, every query
    (1024, 64, 300, 0.5, True),    # whole tail block, queries at the end
    (768, 100, 868, 0.25, True),   # two tail blocks (the second one partial)
    (512, 130, 200, 1.0, False),   # three tail blocks, non-causal
    (0, 37, 37, 0.0, True),        # tail only (no compressed prefix)
])
def test_prefill_with_dense_tail(hs, port, dtype, L, tail, n_q, s, causal):
    """prefill_attention with CacheView::dense_tail (attention.hpp:19-31, :289-297)."""
    U, gqa = 2, 2
    kx = gen_units(port, U, L + tail, 128, 13, 0, dtype)
    vx = gen_units(port, U, L + tail, 128, 13, 1, dtype)
    if L == 0:  # CacheView{compressed = nullptr, dense_tail} (attention.hpp:22-31)
        kc = vc = None
    else:
        kc, vc = hs.prune_cache(to_torch(kx[:, :L], dtype), to_torch(vx[:, :L], dtype), hs.SparsityConfig(s, s, 64))
    q = np.stack([np.stack([port.round_to(port.random_gaussian(n_q, 128, port.head_seed(13, u, 2 + g)), dtype)
                            for g in range(gqa)]) for u in range(U)])
    scale = np.float32(1.0 / math.sqrt(128))
    got = hs.prefill_attention(to_torch(q, dtype), kc, vc, to_torch(kx[:, L:], dtype), to_torch(vx[:, L:], dtype),
                               causal=causal, scale=float(scale)).cpu().numpy()

    def one(ug):
        u, g = divmod(ug, gqa)
        if kc is None:  # the tail alone: the reference's dense oracle over the tail tokens
            return port.dense_attention(q[u, g], kx[u, L:], vx[u, L:], causal, scale)
        return port.prefill(q[u, g], device_to_oracle(kc, u), device_to_oracle(vc, u), kx[u, L:], vx[u, L:], causal,
                            scale, 64)
    want = np.stack(parallel(one, range(U * gqa))).reshape(U, gqa, n_q, 128)
    mx, mr = err_stats(got, want)
    assert mx < MAX_ABS_TOL and mr < MEAN_REL_TOL, (mx, mr)


def test_attention_rejects_mismatched_queries(hs, port):
    """Queries are validated against the caches (dtype, units, head_dim, device)
    instead of being reinterpreted (fp32 queries are a natural reference call)."""
    import torch
    kc, vc, q = setup(hs, port, 2, 256, 1.0, "f16", 1, 64)
    qt = to_torch(q, "f16")
    bad = [qt.float(), qt.to(torch.bfloat16), qt[:1], qt[..., :64].contiguous(), qt.cpu()]
    for b in bad:
        with pytest.raises(hs.ConfigError):
            hs.prefill_attention(b, kc, vc)
        with pytest.raises(hs.ConfigError):
            hs.decode_attention(b[:, 0, :4], kc, vc)
    with pytest.raises(hs.ConfigError):
        hs.prefill_attention(qt, kc, vc, out=torch.empty(2, 1, 64, 64, device="cuda"))


def test_prefill_rejects_invalid(hs, port):
    from paper_2604_16864_b200 import ConfigError
    kc, vc, q = setup(hs, port, 1, 256, 1.0, "f16", 1, 256)
    with pytest.raises(ConfigError):
        hs.prefill_attention(to_torch(q, "f16"), vc, kc)  # swapped caches
    big = np.zeros((1, 1, 512, 128), np.float32)
    with pytest.raises(ConfigError):
        hs.prefill_attention(to_torch(big, "f16"), kc, vc, causal=True)  # n_q > n_kv


@pytest.mark.parametrize("seed", [7, 8])
def test_prefill_random_shapes(hs, port, seed):
    """Randomised shapes (sequence length, query count, sparsity, protection,
    causality, units, GQA) on the fp16 ping-pong path against the oracle."""
    rng = np.random.default_rng(seed)
    for i in range(4):
        L = int(rng.choice([128, 256, 384, 640, 1024]))
        n_q = int(rng.integers(1, L + 1))
        s = float(rng.choice([0.0, 0.25, 0.5, 0.75, 1.0]))
        sink, window = int(rng.choice([0, 64, 100])), int(rng.choice([0, 128, 200]))
        causal = bool(rng.integers(0, 2))
        U, gqa = int(rng.integers(1, 3)), int(rng.integers(1, 3))
        kc, vc, q = setup(hs, port, U, L, s, "f16", gqa, n_q, sink, window, seed=seed * 10 + i)
        scale = np.float32(1.0 / math.sqrt(128))
        got = hs.prefill_attention(to_torch(q, "f16"), kc, vc, causal=causal, scale=float(scale)).cpu().numpy()

        def one(ug):
            u, g = divmod(ug, gqa)
            return port.prefill(q[u, g], device_to_oracle(kc, u), device_to_oracle(vc, u), None, None, causal,
                                scale, 64)
        want = np.stack(parallel(one, range(U * gqa))).reshape(U, gqa, n_q, 128)
        mx, mr = err_stats(got, want)
        assert mx < MAX_ABS_TOL and mr < MEAN_REL_TOL, (L, n_q, s, sink, window, causal, U, gqa, mx, mr)


@pytest.mark.parametrize("dtype", ["f16", "bf16"])
@pytest.mark.parametrize("s", [1.0, 0.5])
def test_prefill_safe_pass(hs, port, dtype, s, monkeypatch):
    """The SAFE pass (race-free running-max exchange, every CTA recomputed) on
    growing scores and random shapes: the ping-pong kernel re-runs the CTAs whose
    rows came out non-finite through it, so it must match the oracle on its own."""
    monkeypatch.setenv("HS_PREFILL_FORCE_SAFE", "1")
    test_prefill_growing_scores(hs, port, dtype, s, True)
    kc, vc, q = setup(hs, port, 2, 1024, s, dtype, 2, 700, 64, 128, seed=5)
    scale = np.float32(1.0 / math.sqrt(128))
    got = hs.prefill_attention(to_torch(q, dtype), kc, vc, causal=True, scale=float(scale)).cpu().numpy()

    def one(ug):
        u, g = divmod(ug, 2)
        return port.prefill(q[u, g], device_to_oracle(kc, u), device_to_oracle(vc, u), None, None, True, scale, 64)
    want = np.stack(parallel(one, range(4))).reshape(2, 2, 700, 128)
    mx, mr = err_stats(got, want)
    assert mx < MAX_ABS_TOL and mr < MEAN_REL_TOL, (mx, mr)


@pytest.mark.parametrize("dtype", ["f16", "bf16"])
def test_prefill_extreme_jumps(hs, port, dtype):
    """Column maxima that jump by hundreds of log2 units late in the sequence
    (hot key blocks scaled far above the rest): whichever group sees the jump
    first, the result (fast pass plus the SAFE pass it may trigger) matches."""
    U, gqa, L, n_q = 1, 2, 2048, 2048
    kx = np.stack([port.random_gaussian(L, 128, port.head_seed(21, u, 0)) for u in range(U)])
    for b0 in (640, 1216, 1792):
        kx[:, b0:b0 + 64] *= 48.0
    kx = port.round_to(kx.astype(np.float32), dtype)
    vx = gen_units(port, U, L, 128, 21, 1, dtype)
    kc, vc = hs.prune_cache(to_torch(kx, dtype), to_torch(vx, dtype), hs.SparsityConfig(1.0, 1.0, 64))
    q = np.stack([np.stack([port.round_to(port.random_gaussian(n_q, 128, port.head_seed(21, u, 2 + g)) * 6.0, dtype)
                            for g in range(gqa)]) for u in range(U)])
    scale = np.float32(1.0 / math.sqrt(128))
    got = hs.prefill_attention(to_torch(q, dtype), kc, vc, causal=True, scale=float(scale)).cpu().numpy()
    assert np.isfinite(got).all()

    def one(g):
        return port.prefill(q[0, g], device_to_oracle(kc, 0), device_to_oracle(vc, 0), None, None, True, scale, 64)
    want = np.stack(parallel(one, range(gqa)))[None]
    mx, mr = err_stats(got, want)
    assert mx < MAX_ABS_TOL and mr < MEAN_REL_TOL, (mx, mr)
