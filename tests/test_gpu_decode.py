"""GPU parity: split-KV sparse decode (attention.hpp:360-409) against the fp32
oracle on identical 16-bit inputs, within the north-star bar
(max-abs 2e-2, mean-rel = sum|e| / sum|ref| 1e-3)."""
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


def build_caches(hs, port, U, L, s, dtype, sink=0, window=0, seed=1):
    kx = gen_units(port, U, L, 128, seed, 0, dtype)
    vx = gen_units(port, U, L, 128, seed, 1, dtype)
    cfg = hs.SparsityConfig(s, s, 64, sink, window)
    kc, vc = hs.prune_cache(to_torch(kx, dtype), to_torch(vx, dtype), cfg)
    return kx, vx, kc, vc


def decode_queries(port, U, gqa, dtype, seed=1):
    # decode Q streams: role 32 + g (pipeline.hpp:249)
    q = np.stack([np.stack([port.random_gaussian(1, 128, port.head_seed(seed, u, 32 + g))[0]
                            for g in range(gqa)]) for u in range(U)])
    return port.round_to(q, dtype).reshape(U, gqa, 128)


def oracle_decode(port, kc, vc, q, scale, splits, k_tail=None, v_tail=None):
    U = q.shape[0]

    def one(u):
        kt = None if k_tail is None else k_tail[u]
        vt = None if v_tail is None else v_tail[u]
        return port.decode(q[u], device_to_oracle(kc, u), device_to_oracle(vc, u), kt, vt, scale, splits)
    return np.stack(parallel(one, range(U)))


@pytest.mark.parametrize("dtype", ["bf16", "f16"])
@pytest.mark.parametrize("L,s,sink,window,gqa,tail", [
    (4096, 1.0, 0, 0, 1, 0),     # config 1: single head, 4K, 2:4 K+V
    (4096, 1.0, 0, 0, 4, 0),
    (4096, 0.5, 64, 256, 4, 0),  # mixed dense/sparse, protected sink + window
    (2048, 0.0, 0, 0, 4, 0),     # all dense
    (1024, 0.75, 0, 0, 8, 17),   # ragged dense tail, 8 query rows
    (64, 1.0, 0, 0, 4, 63),      # one block + tail
])
def test_decode_matches_oracle(hs, port, dtype, L, s, sink, window, gqa, tail):
    U = 3
    kx, vx, kc, vc = build_caches(hs, port, U, L, s, dtype, sink, window)
    q = decode_queries(port, U, gqa, dtype)
    scale = np.float32(1.0 / math.sqrt(128))
    kt = vt = None
    if tail:
        kt = gen_units(port, U, tail, 128, 77, 0, dtype)
        vt = gen_units(port, U, tail, 128, 77, 1, dtype)
    want = oracle_decode(port, kc, vc, q, scale, 4, kt, vt)
    for splits in (0, 1, 7):
        got = hs.decode_attention(to_torch(q, dtype), kc, vc,
                                  None if kt is None else to_torch(kt, dtype),
                                  None if vt is None else to_torch(vt, dtype),
                                  float(scale), splits=splits).cpu().numpy()
        mx, mr = err_stats(got, want)
        assert mx < MAX_ABS_TOL and mr < MEAN_REL_TOL, (splits, mx, mr)


def test_decode_gqa_rows_independent(hs, port):
    """Each GQA row equals its own single-row decode (test_attention.cpp:356-364),
    within float rounding of the kernel."""
    U, L = 2, 2048
    kx, vx, kc, vc = build_caches(hs, port, U, L, 1.0, "f16")
    q = decode_queries(port, U, 4, "f16")
    full = hs.decode_attention(to_torch(q, "f16"), kc, vc, splits=3).cpu().numpy()
    for g in range(4):
        one = hs.decode_attention(to_torch(q[:, g:g + 1], "f16"), kc, vc, splits=3).cpu().numpy()
        assert np.abs(one[:, 0] - full[:, g]).max() < 1e-6


def test_decode_partial_and_combine(hs, port):
    """Sequence split across 'devices': partials over contiguous block ranges,
    LSE-combined, equal the single decode (attention.hpp:380-407)."""
    import torch
    U, L = 2, 8192
    kx, vx, kc, vc = build_caches(hs, port, U, L, 1.0, "bf16")
    q = to_torch(decode_queries(port, U, 4, "bf16"), "bf16")
    kt = to_torch(gen_units(port, U, 5, 128, 3, 0, "bf16"), "bf16")
    vt = to_torch(gen_units(port, U, 5, 128, 3, 1, "bf16"), "bf16")
    ref = hs.decode_attention(q, kc, vc, kt, vt)
    nb, parts = kc.logical_blocks, 4
    ps = [hs.decode_partial(q, kc, vc, nb * r // parts, nb * (r + 1) // parts, kt, vt, include_tail=(r == parts - 1))
          for r in range(parts)]
    out = hs.decode_combine(torch.stack(ps))
    assert (out - ref).abs().max().item() < 1e-5


def test_decode_config2_full_size(hs, port):
    """Config 2: 8 KV heads x 128K tokens, GQA 4, S_K = S_V = 1, bf16 — every
    head against the oracle's decode_attention."""
    U, L = 8, 131072
    kx, vx, kc, vc = build_caches(hs, port, U, L, 1.0, "bf16", seed=2)
    q = decode_queries(port, U, 4, "bf16", seed=2)
    scale = np.float32(1.0 / math.sqrt(128))
    got = hs.decode_attention(to_torch(q, "bf16"), kc, vc, scale=float(scale)).cpu().numpy()
    want = oracle_decode(port, kc, vc, q, scale, 1)
    mx, mr = err_stats(got, want)
    assert mx < MAX_ABS_TOL and mr < MEAN_REL_TOL, (mx, mr)


def test_decode_rejects_invalid(hs, port):
    from paper_2604_16864_b200 import ConfigError
    U = 1
    kx, vx, kc, vc = build_caches(hs, port, U, 512, 1.0, "bf16")
    q = to_torch(decode_queries(port, U, 4, "bf16"), "bf16")
    with pytest.raises(ConfigError):
        hs.decode_attention(q, vc, kc)          # swapped caches (test_attention.cpp:392-395)
    with pytest.raises(ConfigError):
        hs.decode_attention(q[:, :, :64].contiguous(), kc, vc)  # head_dim mismatch


def test_decode_gqa_above_eight_rows(hs, port):
    """GQA groups above the mma.sp kernel's 8 stacked rows run in row chunks with
    the group's strides: 12 and 16 rows against the oracle."""
    U, L = 2, 4096
    kx, vx, kc, vc = build_caches(hs, port, U, L, 0.5, "bf16", seed=6)
    scale = np.float32(1.0 / math.sqrt(128))
    for gqa in (12, 16):
        q = decode_queries(port, U, gqa, "bf16", seed=6)
        got = hs.decode_attention(to_torch(q, "bf16"), kc, vc, scale=float(scale)).cpu().numpy()
        want = oracle_decode(port, kc, vc, q, scale, 1)
        mx, mr = err_stats(got, want)
        assert mx < MAX_ABS_TOL and mr < MEAN_REL_TOL, (gqa, mx, mr)


def test_decode_fixed_splits_deterministic(hs, port):
    """An explicit split count is the static partition: bitwise identical across
    runs (acceptance.cpp:518-543 determinism); auto splits (dynamic block claims)
    agree to float rounding."""
    U, L = 4, 8192
    kx, vx, kc, vc = build_caches(hs, port, U, L, 1.0, "bf16")
    q = to_torch(decode_queries(port, U, 4, "bf16"), "bf16")
    runs = [hs.decode_attention(q, kc, vc, splits=7).cpu().numpy() for _ in range(3)]
    assert all((r == runs[0]).all() for r in runs[1:])
    auto = [hs.decode_attention(q, kc, vc).cpu().numpy() for _ in range(3)]
    assert max(np.abs(a - runs[0]).max() for a in auto) < 1e-5


def test_decode_concurrent_streams(hs, port):
    """Two full-machine decodes (auto splits: the cooperative combine) launched on
    two streams at once never deadlock and each equals its single-stream result:
    the cooperative launch guarantees co-residency instead of assuming it."""
    import torch
    U, L = 8, 16384
    kx, vx, kc, vc = build_caches(hs, port, U, L, 1.0, "bf16", seed=3)
    kx2, vx2, kc2, vc2 = build_caches(hs, port, U, L, 0.5, "bf16", seed=4)
    q = to_torch(decode_queries(port, U, 4, "bf16"), "bf16")
    want1 = hs.decode_attention(q, kc, vc).clone()
    want2 = hs.decode_attention(q, kc2, vc2).clone()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    outs1, outs2 = [], []
    torch.cuda.synchronize()
    for _ in range(20):
        with torch.cuda.stream(s1):
            outs1.append(hs.decode_attention(q, kc, vc))
        with torch.cuda.stream(s2):
            outs2.append(hs.decode_attention(q, kc2, vc2))
    torch.cuda.synchronize()
    for a in outs1:
        assert (a - want1).abs().max().item() < 1e-5
    for b in outs2:
        assert (b - want2).abs().max().item() < 1e-5


def test_decode_plans_own_their_workspaces(hs, port):
    """DecodePlan graphs replayed interleaved (and on recycled stream handles)
    share no split partials or arrival counters (hs_decode_ws)."""
    import torch
    U = 4
    plans, wants = [], []
    for i, L in enumerate((4096, 32768, 8192)):
        kx, vx, kc, vc = build_caches(hs, port, U, L, 1.0, "bf16", seed=10 + i)
        q = to_torch(decode_queries(port, U, 4, "bf16", seed=10 + i), "bf16")
        wants.append(hs.decode_attention(q, kc, vc).clone())
        plans.append(hs.DecodePlan(q, kc, vc))
    # a later, larger decode on the default path must not disturb the plans
    kx, vx, kcb, vcb = build_caches(hs, port, 8, 65536, 1.0, "bf16", seed=20)
    hs.decode_attention(to_torch(decode_queries(port, 8, 8, "bf16"), "bf16"), kcb, vcb)
    for _ in range(5):
        for p, w in zip(plans, wants):
            p()
        torch.cuda.synchronize()
        for p, w in zip(plans, wants):
            assert (p.out - w).abs().max().item() < 1e-5


def test_decode_mailbox_after_other_modes(hs, port, monkeypatch):
    """The cooperative combine's tagged mailbox must read empty before every launch:
    plain split partials of a larger, non-cooperative decode on the same stream
    (and a plan's row chunks of different widths in one workspace) never land on
    it, so later cooperative decodes and plan replays stay exact."""
    import torch
    kx, vx, kcb, vcb = build_caches(hs, port, 8, 65536, 1.0, "bf16", seed=41)
    qb = to_torch(decode_queries(port, 8, 8, "bf16", seed=41), "bf16")
    U, L = 4, 8192
    kx, vx, kc, vc = build_caches(hs, port, U, L, 0.5, "bf16", seed=42)
    q = to_torch(decode_queries(port, U, 4, "bf16", seed=42), "bf16")
    want = hs.decode_attention(q, kc, vc, splits=7).clone()
    monkeypatch.setenv("HS_DECODE_COOP", "0")
    hs.decode_attention(qb, kcb, vcb)  # plain partials over the whole decode workspace
    monkeypatch.delenv("HS_DECODE_COOP")
    for _ in range(3):
        assert (hs.decode_attention(q, kc, vc) - want).abs().max().item() < 1e-5
    q12 = to_torch(decode_queries(port, U, 12, "bf16", seed=43), "bf16")
    want12 = hs.decode_attention(q12, kc, vc).clone()
    plan = hs.DecodePlan(q12, kc, vc)
    for _ in range(3):
        plan()
        torch.cuda.synchronize()
        assert (plan.out - want12).abs().max().item() < 1e-5


def test_decode_plan_host_io(hs, port):
    """DecodePlan(host_io=True): one graph replay copies the pinned host queries in,
    decodes and copies the output to pinned host memory; fresh queries written to
    q_host between replays are picked up, matching decode_attention."""
    import torch
    U, L = 4, 8192
    kx, vx, kc, vc = build_caches(hs, port, U, L, 1.0, "bf16", seed=31)
    q0 = to_torch(decode_queries(port, U, 4, "bf16", seed=31), "bf16")
    q1 = to_torch(decode_queries(port, U, 4, "bf16", seed=32), "bf16")
    plan = hs.DecodePlan(q0, kc, vc, host_io=True)
    for q in (q0, q1, q0):
        out = plan(q.cpu())
        torch.cuda.synchronize()
        want = hs.decode_attention(q, kc, vc).cpu()
        assert out.device.type == "cpu" and out.is_pinned()
        assert (out - want).abs().max().item() < 1e-5


def test_decode_pinned_host_queries_and_output(hs, port):
    """decode_attention on a pinned host q with a pinned host out (zero-copy) equals
    the device-resident call; a pageable host q is rejected."""
    import torch
    U, L = 3, 4096
    kx, vx, kc, vc = build_caches(hs, port, U, L, 0.5, "bf16", seed=41)
    q = to_torch(decode_queries(port, U, 12, "bf16", seed=41), "bf16")  # 12 rows: two row chunks
    want = hs.decode_attention(q, kc, vc).cpu()
    out = torch.empty(want.shape, dtype=torch.float32).pin_memory()
    hs.decode_attention(q.cpu().pin_memory(), kc, vc, out=out)
    torch.cuda.synchronize()
    assert (out - want).abs().max().item() < 1e-5
    with pytest.raises(hs.ConfigError):
        hs.decode_attention(q.cpu(), kc, vc)


@pytest.mark.parametrize("tail", [1, 37, 200])
def test_decode_tail_only_view(hs, port, tail):
    """CacheView{compressed = nullptr, dense_tail} (attention.hpp:22-31): decode over
    the tail alone equals the reference's dense oracle on the tail tokens."""
    U, gqa = 2, 4
    kx = gen_units(port, U, tail, 128, 8, 0, "bf16")
    vx = gen_units(port, U, tail, 128, 8, 1, "bf16")
    q = decode_queries(port, U, gqa, "bf16", seed=8)
    scale = np.float32(1.0 / math.sqrt(128))
    got = hs.decode_attention(to_torch(q, "bf16"), None, None, to_torch(kx, "bf16"), to_torch(vx, "bf16"),
                              scale=float(scale)).cpu().numpy()
    want = np.stack([port.dense_attention(q[u], kx[u], vx[u], False, scale) for u in range(U)])
    mx, mr = err_stats(got, want)
    assert mx < MAX_ABS_TOL and mr < MEAN_REL_TOL, (mx, mr)


@pytest.mark.parametrize("env", [{"HS_DECODE_INTERLEAVE": "0"}, {"HS_DECODE_MAILBOX": "0"},
                                 {"HS_DECODE_COOP": "0"}, {"HS_DECODE_DYNAMIC": "0"}])
def test_decode_launch_variants_agree(hs, port, monkeypatch, env):
    """The legacy / fallback launch shapes kept behind switches -- the 2-D (split,
    unit) grid, the counter hand-off instead of the tagged mailbox, the last-CTA
    ticket combine, static split ranges -- give the default path's result."""
    U, L = 8, 16384
    kx, vx, kc, vc = build_caches(hs, port, U, L, 0.5, "bf16", seed=51)
    q = to_torch(decode_queries(port, U, 4, "bf16", seed=51), "bf16")
    want = hs.decode_attention(q, kc, vc).clone()
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    for _ in range(2):
        got = hs.decode_attention(q, kc, vc)
        assert (got - want).abs().max().item() < 1e-5
    for k in env:
        monkeypatch.delenv(k)
    assert (hs.decode_attention(q, kc, vc) - want).abs().max().item() < 1e-5
