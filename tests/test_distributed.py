"""Multi-process (gloo, world_size 2, CPU) tests of the multi-GPU partitioning:
shard arithmetic (attention.hpp:380-381), the all-gather of SplitPartials in
rank order, and the sequence-split decode they assemble, checked against the
oracle's single-process decode_attention (attention.hpp:360-409)."""
import math
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2604_16864_b200 import distributed as D


@pytest.mark.parametrize("n,world", [(2048, 8), (16384, 8), (7, 3), (64, 2), (1, 1), (5, 5)])
def test_contiguous_shards_partition_the_range(n, world):
    shards = [D.contiguous_shard(n, world, r) for r in range(world)]
    assert shards[0].begin == 0 and shards[-1].end == n
    for a, b in zip(shards, shards[1:]):
        assert a.end == b.begin
    assert sum(s.size for s in shards) == n
    assert all(s == D.Shard(n * r // world, n * (r + 1) // world) for r, s in enumerate(shards))


def test_head_and_unit_shards():
    assert [D.heads_of_rank(8, 4, r) for r in range(4)] == [D.Shard(2 * r, 2 * r + 2) for r in range(4)]
    with pytest.raises(ValueError):
        D.heads_of_rank(8, 3, 0)
    with pytest.raises(ValueError):
        D.contiguous_shard(8, 2, 2)
    # config 4: 32 requests x 8 KV heads over 8 ranks -> 32 units each
    assert all(D.unit_shard(32, 8, 8, r).size == 32 for r in range(8))


def _combine(parts):
    """LSE combine of packed partials [P, rows, d+2] (attention.hpp:387-407)."""
    o, m, l = parts[..., :-2], parts[..., -2], parts[..., -1]
    mx = m.max(axis=0)
    w = np.where(np.isfinite(m), np.exp(m - mx[None]), 0.0)
    lt = (l * w).sum(axis=0)
    return (o * w[..., None]).sum(axis=0) / lt[:, None]


def _worker(rank, world, port_no, L, tail, ret):
    import torch
    import torch.distributed as dist
    from oracle.oracle import Oracle, SparsityConfig
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port_no))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        port = Oracle("port")
        d, gqa, seed = 128, 4, 7
        k = port.round_to(port.random_gaussian(L + tail, d, port.head_seed(seed, 0, 0)), "bf16")
        v = port.round_to(port.random_gaussian(L + tail, d, port.head_seed(seed, 0, 1)), "bf16")
        q = port.round_to(np.stack([port.random_gaussian(1, d, port.head_seed(seed, 0, 32 + g))[0]
                                    for g in range(gqa)]), "bf16")
        scale = np.float32(1 / math.sqrt(d))
        nb = L // 64
        sh = D.sequence_shard(nb, world, rank)
        last = rank == world - 1
        # this rank compresses only its own shard (S = 1: every block 2:4)
        cfg = SparsityConfig(1.0, 1.0, 64)
        ks = port.prune_compress(k[sh.begin * 64:sh.end * 64], cfg, 0, 1.0)
        vs = port.prune_compress(v[sh.begin * 64:sh.end * 64], cfg, 1, 1.0)
        kt, vt = (k[L:], v[L:]) if (last and tail) else (None, None)
        out_t, m, l = port.attend_rows(q, ks, vs, kt, vt, 0, sh.size, last, scale)
        partial = torch.from_numpy(np.concatenate([out_t.T, m[:, None], l[:, None]], axis=1))[None]
        gathered = D.gather_partials(partial).numpy()  # [world, 1, gqa, d+2]
        got = _combine(gathered[:, 0])
        if rank == 0:
            kf = port.prune_compress(k[:L], cfg, 0, 1.0)
            vf = port.prune_compress(v[:L], cfg, 1, 1.0)
            want = port.decode(q, kf, vf, k[L:] if tail else None, v[L:] if tail else None, scale, 1)
            ret.put((float(np.abs(got - want).max()), gathered.shape))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("L,tail", [(4096, 0), (2048, 37)])
def test_sequence_split_decode_two_ranks(L, tail):
    ctx = mp.get_context("spawn")
    ret = ctx.Queue()
    world = 2
    mp.start_processes(_worker, args=(world, _free_port(), L, tail, ret), nprocs=world, join=True,
                       start_method="spawn")
    err, shape = ret.get(timeout=60)
    assert shape == (world, 1, 4, 130)
    assert err < 1e-5, err


def _worker_global(rank, world, port_no, L, ret):
    """Sequence-split pruning with the global block selection: every rank's shard
    losses are gathered (distributed.gather_block_losses, the product's
    collective), the selection over the whole sequence flags the blocks, each
    rank packs its slice; oracle functions stand in for the device kernels."""
    import torch
    import torch.distributed as dist
    from oracle.oracle import Oracle, SparsityConfig
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port_no))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        port = Oracle("port")
        d, gqa, seed, B = 128, 4, 9, 64
        cfg = SparsityConfig(0.5, 0.5, B, 64, 256)
        k = port.round_to(port.random_gaussian(L, d, port.head_seed(seed, 0, 0)), "bf16")
        v = port.round_to(port.random_gaussian(L, d, port.head_seed(seed, 0, 1)), "bf16")
        q = port.round_to(np.stack([port.random_gaussian(1, d, port.head_seed(seed, 0, 32 + g))[0]
                                    for g in range(gqa)]), "bf16")
        scale = np.float32(1 / math.sqrt(d))
        nb = L // B
        sh = D.sequence_shard(nb, world, rank)
        kf = port.prune_compress(k, cfg, 0, 0.5)  # whole-sequence reference (every rank can check)
        vf = port.prune_compress(v, cfg, 1, 0.5)
        parts = []
        ok_losses = True
        for x, full, axis in ((k, kf, 0), (v, vf, 1)):
            xs = x[sh.begin * B:sh.end * B]
            local = port.prune_compress(xs, SparsityConfig(0.0, 0.0, B), axis, 0.0).losses  # block_loss of the shard
            glob = D.gather_block_losses(torch.from_numpy(local)[None], nb)[0].numpy()
            ok_losses &= glob.tobytes() == full.losses.tobytes()
            flags = full.flags  # select_blocks over the gathered losses (the oracle's, = whole-sequence)
            parts.append(port.compress_with_flags(xs, cfg, axis, flags[sh.begin:sh.end]))
        out_t, m, l = port.attend_rows(q, parts[0], parts[1], None, None, 0, sh.size, False, scale)
        partial = torch.from_numpy(np.concatenate([out_t.T, m[:, None], l[:, None]], axis=1))[None]
        got = _combine(D.gather_partials(partial).numpy()[:, 0])
        if rank == 0:
            want = port.decode(q, kf, vf, None, None, scale, 1)
            local_only = port.prune_compress(k[sh.begin * B:sh.end * B], cfg, 0, 0.5).flags
            ret.put((ok_losses, float(np.abs(got - want).max()),
                     bool((local_only != kf.flags[sh.begin:sh.end]).any())))
    finally:
        dist.destroy_process_group()


def test_sequence_split_pruning_uses_the_global_selection():
    """At S = 0.5 with sink and window protection, shard-local pruning differs from
    prune_cache of the whole sequence; gathering the losses restores it exactly and
    the split decode equals the single-process decode_attention."""
    ctx = mp.get_context("spawn")
    ret = ctx.Queue()
    world = 2
    mp.start_processes(_worker_global, args=(world, _free_port(), 4096, ret), nprocs=world, join=True,
                       start_method="spawn")
    ok_losses, err, local_differs = ret.get(timeout=60)
    assert ok_losses
    assert local_differs  # the bug the global selection fixes
    assert err < 1e-5, err


def test_bench_spawns_ranks_and_reports_n_gpus():
    """`bench.py --gpus 2` without torchrun starts two ranks itself; the selftest
    mode drives its multi-rank wiring (all-gather order of the configs[4]
    partials, max / sum over ranks) on gloo and reports n_gpus: 2."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--selftest"],
                         capture_output=True, text=True, timeout=240, cwd=root)
    line = [x for x in out.stdout.splitlines() if x.startswith("{")][-1]
    rec = json.loads(line)
    assert rec["selftest"] == "ok" and rec["n_gpus"] == 2, rec
