"""GPU parity of the sequence-split decode (config 5) with the shards simulated
on one device: each shard is compressed on its own (as its rank would), the
per-shard SplitPartials (hs_decode_partial) are stacked in rank order and merged
by hs_decode_combine; the result must match the oracle's decode_attention over
the whole sequence (attention.hpp:360-409).  Also checks unit sharding: a rank's
decode over its unit range equals the same rows of the all-unit decode."""
import math

import numpy as np
import pytest

from tests.helpers import MAX_ABS_TOL, MEAN_REL_TOL, device_to_oracle, err_stats, gen_units, to_torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def hs():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_2604_16864_b200 import hierasparse
    return hierasparse


@pytest.mark.parametrize("world,L,tail", [(2, 4096, 0), (4, 8192, 21), (8, 16384, 0)])
def test_sequence_split_matches_whole_sequence(hs, port, world, L, tail):
    import torch
    from paper_2604_16864_b200 import distributed as D
    U, gqa, d = 2, 4, 128
    kx = gen_units(port, U, L + tail, d, 5, 0, "bf16")
    vx = gen_units(port, U, L + tail, d, 5, 1, "bf16")
    q = np.stack([port.round_to(np.stack([port.random_gaussian(1, d, port.head_seed(5, u, 32 + g))[0]
                                          for g in range(gqa)]), "bf16") for u in range(U)])
    scale = float(np.float32(1 / math.sqrt(d)))
    cfg = hs.SparsityConfig(1.0, 1.0, 64)
    nb = L // 64
    parts = []
    for r in range(world):
        sh = D.sequence_shard(nb, world, r)
        ks, vs = hs.prune_cache(to_torch(kx[:, sh.begin * 64:sh.end * 64], "bf16"),
                                to_torch(vx[:, sh.begin * 64:sh.end * 64], "bf16"), cfg)
        last = r == world - 1
        kt = to_torch(kx[:, L:], "bf16") if (last and tail) else None
        vt = to_torch(vx[:, L:], "bf16") if (last and tail) else None
        parts.append(hs.decode_partial(to_torch(q, "bf16"), ks, vs, 0, sh.size, kt, vt, include_tail=last,
                                       scale=scale))
    got = hs.decode_combine(torch.stack(parts)).cpu().numpy()
    kf, vf = hs.prune_cache(to_torch(kx[:, :L], "bf16"), to_torch(vx[:, :L], "bf16"), cfg)
    want = np.stack([port.decode(q[u], device_to_oracle(kf, u), device_to_oracle(vf, u),
                                 kx[u, L:] if tail else None, vx[u, L:] if tail else None, np.float32(scale), 1)
                     for u in range(U)])
    mx, mr = err_stats(got, want)
    assert mx < MAX_ABS_TOL and mr < MEAN_REL_TOL, (mx, mr)


def test_unit_shards_equal_rows_of_full_decode(hs, port):
    from paper_2604_16864_b200 import distributed as D
    U, L, gqa, world = 8, 2048, 4, 4
    kx = gen_units(port, U, L, 128, 9, 0, "f16")
    vx = gen_units(port, U, L, 128, 9, 1, "f16")
    q = np.stack([port.round_to(np.stack([port.random_gaussian(1, 128, port.head_seed(9, u, 32 + g))[0]
                                          for g in range(gqa)]), "f16") for u in range(U)])
    cfg = hs.SparsityConfig(0.5, 1.0, 64)
    kc, vc = hs.prune_cache(to_torch(kx, "f16"), to_torch(vx, "f16"), cfg)
    full = hs.decode_attention(to_torch(q, "f16"), kc, vc).cpu().numpy()
    for r in range(world):
        sh = D.unit_shard(1, U, world, r)
        ks, vs = hs.prune_cache(to_torch(kx[sh.begin:sh.end], "f16"), to_torch(vx[sh.begin:sh.end], "f16"), cfg)
        got = hs.decode_attention(to_torch(q[sh.begin:sh.end], "f16"), ks, vs).cpu().numpy()
        mx, _ = err_stats(got, full[sh.begin:sh.end])
        assert mx < 1e-5, (r, mx)


@pytest.mark.parametrize("world", [2, 4, 8])
def test_prefill_kv_head_shards_equal_rows_of_full_prefill(hs, port, world):
    """configs[2] over N GPUs: rank r prefills the KV heads
    heads_of_rank(8, N, r) with their GQA query heads -- compressed and attended on
    their own -- and must reproduce the same heads of the single-GPU prefill (the
    bench's prefill leg runs exactly this per rank; no collective)."""
    from paper_2604_16864_b200 import distributed as D
    U, L, gqa = 8, 1024, 4
    kx = gen_units(port, U, L, 128, 13, 0, "f16")
    vx = gen_units(port, U, L, 128, 13, 1, "f16")
    q = np.stack([np.stack([port.round_to(port.random_gaussian(L, 128, port.head_seed(13, u, 2 + g)), "f16")
                            for g in range(gqa)]) for u in range(U)])
    cfg = hs.SparsityConfig(0.5, 0.5, 64, 64, 128)
    kc, vc = hs.prune_cache(to_torch(kx, "f16"), to_torch(vx, "f16"), cfg)
    full = hs.prefill_attention(to_torch(q, "f16"), kc, vc, causal=True).cpu().numpy()
    for r in range(world):
        sh = D.heads_of_rank(U, world, r)
        ks, vs = hs.prune_cache(to_torch(kx[sh.begin:sh.end], "f16"), to_torch(vx[sh.begin:sh.end], "f16"), cfg)
        got = hs.prefill_attention(to_torch(q[sh.begin:sh.end], "f16"), ks, vs, causal=True).cpu().numpy()
        mx, _ = err_stats(got, full[sh.begin:sh.end])
        assert mx < 1e-3, (r, mx)  # same arithmetic per head; the running max is per CTA


@pytest.mark.parametrize("world,s,sink,window", [(2, 0.5, 64, 256), (4, 0.25, 100, 70), (8, 0.75, 0, 512)])
def test_sharded_pruning_equals_whole_sequence(hs, port, world, s, sink, window):
    """prune_cache_sharded's device steps per simulated rank (block losses of the
    shard, global select_blocks over the gathered losses, compress the slice)
    reproduce prune_cache of the whole sequence sliced by block range, bit for
    bit, and the split decode matches the whole-sequence decode."""
    import torch
    from paper_2604_16864_b200 import distributed as D
    U, gqa, d, L, B = 3, 4, 128, 8192, 64
    kx = gen_units(port, U, L, d, 12, 0, "bf16")
    vx = gen_units(port, U, L, d, 12, 1, "bf16")
    q = np.stack([port.round_to(np.stack([port.random_gaussian(1, d, port.head_seed(12, u, 32 + g))[0]
                                          for g in range(gqa)]), "bf16") for u in range(U)])
    cfg = hs.SparsityConfig(s, s, B, sink, window)
    nb = L // B
    kf, vf = hs.prune_cache(to_torch(kx, "bf16"), to_torch(vx, "bf16"), cfg)
    shards = [D.sequence_shard(nb, world, r) for r in range(world)]
    out = {}
    for x, full, axis, sv in ((kx, kf, 0, s), (vx, vf, 1, s)):
        xs = [to_torch(x[:, sh.begin * B:sh.end * B], "bf16") for sh in shards]
        losses = torch.cat([hs.block_losses(t, cfg, axis) for t in xs], dim=1)  # = gather_block_losses
        assert losses.cpu().numpy().tobytes() == full.losses.cpu().numpy().tobytes()
        flags = hs.select_blocks(losses, cfg, sv)
        assert (flags == full.flags).all()
        caches = [hs.fused_magnitude_compress(t, flags[:, sh.begin:sh.end], cfg, axis, capacity=True)
                  for t, sh in zip(xs, shards)]
        for c, sh in zip(caches, shards):
            for u in range(U):
                got = device_to_oracle(c, u)
                dense = port.decompress(got)
                want = port.decompress(device_to_oracle(full, u))[sh.begin * B:sh.end * B]
                assert (dense == want).all()
        out[axis] = caches
    parts = [hs.decode_partial(to_torch(q, "bf16"), out[0][r], out[1][r], 0, sh.size, include_tail=False)
             for r, sh in enumerate(shards)]
    got = hs.decode_combine(torch.stack(parts)).cpu().numpy()
    want = hs.decode_attention(to_torch(q, "bf16"), kf, vf).cpu().numpy()
    mx, mr = err_stats(got, want)
    assert mx < 1e-4 and mr < 1e-5, (mx, mr)


def test_prune_cache_sharded_single_rank(hs, port):
    """world 1: prune_cache_sharded == prune_cache (flags and pools)."""
    from paper_2604_16864_b200 import distributed as D
    U, L = 2, 4096
    kx = gen_units(port, U, L, 128, 13, 0, "f16")
    vx = gen_units(port, U, L, 128, 13, 1, "f16")
    cfg = hs.SparsityConfig(0.5, 0.75, 64, 64, 128)
    kt, vt = to_torch(kx, "f16"), to_torch(vx, "f16")
    kc, vc, kfl, vfl = D.prune_cache_sharded(kt, vt, cfg, L // 64)
    kf, vf = hs.prune_cache(kt, vt, cfg)
    assert (kfl == kf.flags).all() and (vfl == vf.flags).all()
    for a, b in ((kc, kf), (vc, vf)):
        assert (a.index_map == b.index_map).all()
        for u in range(U):
            ga, gb = device_to_oracle(a, u), device_to_oracle(b, u)
            assert (port.decompress(ga) == port.decompress(gb)).all()
