"""Benchmark of the HieraSparse hot path on B200 (driver contract).

Headline workload (BASELINE.json configs[1]): Llama-3.1-8B GQA decode, 8 KV
heads x 4 query rows, 128K-token context, batch 1, S_K = S_V = 1 (every block
2:4), bf16 pools.  A step = one decode_attention over all 8 KV heads with the
compressed caches resident in HBM.  `value` = algorithmic bytes moved
(flop_and_byte_count, attention.hpp:426-467: pools + index maps + headers)
per second, aggregated over ranks.  N > 1: every rank decodes its own request
(weak scaling, no data-path collective).

The same JSON line carries the other BASELINE configs and legs, each measured
in this run with device events (max over ranks):
  config4   configs[3]  32 requests x 32K x 8 KV heads, KV heads sharded over ranks
  config5   configs[4]  1M tokens x 8 KV heads, sequence split over ranks + NCCL
                        all-gather of the SplitPartials (gather reported apart)
  prefill   configs[2]  64K and 128K causal prefill, block sparsity sweep, KV heads
                        sharded over ranks, with sampled-row parity per S
  decode_grid           configs[1] decode at (S_K, S_V) in {0,1}^2 vs r_comp
  compress / recompress prune_cache + fused_magnitude_compress, decode-phase re-prune
  cpu_baseline          the reference (oracle/_ref) on this host's cores (rank 0, N = 1)

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""
from __future__ import annotations

import argparse
import json
import math
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "decode attn µs & HBM GB/s at 128K ctx; prefill sparse TFLOPS; vs CPU oracle"
U, L, GQA, D = 8, 131072, 4, 128  # configs[1]
L2_BYTES = 126 * 1024 * 1024


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), float(p["bf16_tflops"]), "measured"
    except Exception:  # noqa: BLE001
        return 6650.0, 1590.0, "fallback"


def sustained_tflops():
    """MEASURED_PEAKS.json's sustained dense bf16 figure (cuBLAS back to back for
    seconds, power-capped clocks): the denominator for kernels timed inside long
    runs, beside the burst figure (B200_PROFILING.md)."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["bf16_tflops_sustained"])
    except Exception:  # noqa: BLE001
        return None


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.rows.append([x.strip() for x in out.split(",")])
            except Exception:  # noqa: BLE001
                pass
            self._stop.wait(0.1)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# ------------------------------------------------------------ multi-rank ---
def free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def relaunch_distributed(args) -> int:
    """`--gpus N` without a torchrun environment: start N ranks of this script on
    this node (torch.distributed.run, one process per GPU, 127.0.0.1 rendezvous)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__),
           *sys.argv[1:]]
    return subprocess.call(cmd)


def dist_setup(selftest: bool = False):
    import torch
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        if selftest:
            dist.init_process_group("gloo")
        else:
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    elif torch.cuda.is_available() and not selftest:
        torch.cuda.set_device(0)
    return rank, world, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def reduce_over_ranks(x: float, world: int, op: str) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.SUM)
    return float(t.item())


def max_over_ranks(x: float, world: int) -> float:
    return reduce_over_ranks(x, world, "max")


def sum_over_ranks(x: float, world: int) -> float:
    return reduce_over_ranks(x, world, "sum")


# ------------------------------------------------------------- utilities ---
class Flusher:
    """L2 flush between timed steps: read (not write) a 2x-L2 buffer, so the next
    step starts with an L2 full of clean, unrelated lines."""

    def __init__(self, dev):
        import torch
        self.buf = torch.ones(2 * L2_BYTES // 4, dtype=torch.float32, device=dev)
        self.sink = torch.empty((), dtype=torch.float32, device=dev)

    def __call__(self):
        import torch
        torch.sum(self.buf, dim=0, out=self.sink)


def hold_stream(steps: int):
    """Hold the stream with a device-side sleep while the host enqueues the timed
    steps, so a host hiccup (the clock sampler's nvidia-smi fork, GC) cannot leave the
    GPU idle between a step's start event and its kernels: measured, such gaps put
    60-140 us outliers into an otherwise 57 us decode step."""
    import torch
    torch.cuda._sleep(int(1.965e9 * min(0.05, 0.005 + 0.0005 * steps)))


def time_steps(step, steps: int, warmup: int, flush=None) -> list:
    """Device time (ms) of `steps` calls of step() on the current stream, after
    `warmup` untimed calls; L2 flushed before each timed call when given."""
    import torch
    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    hold_stream(steps)
    for a, b in ev:
        if flush is not None:
            flush()
        a.record()
        step()
        b.record()
    torch.cuda.synchronize()
    return [a.elapsed_time(b) for a, b in ev]


def randn16(shape, g, dev, dtype):
    import torch
    return torch.randn(shape, generator=g, device=dev, dtype=torch.float32).to(dtype)


def build_decode_caches(hs, dev, g, units, ctx, cfg, dtype=None):
    """Synthetic K/V per unit compressed on the device, in chunks of units that keep
    the dense staging buffer below ~4 GB."""
    import torch
    dtype = dtype or torch.bfloat16
    chunk = max(1, min(units, (1 << 31) // (ctx * D * 2)))
    kcs, vcs = [], []
    for c0 in range(0, units, chunk):
        n = min(chunk, units - c0)
        key, val = randn16((n, ctx, D), g, dev, dtype), randn16((n, ctx, D), g, dev, dtype)
        kc, vc = hs.prune_cache(key, val, cfg)
        kcs.append(kc)
        vcs.append(vc)
        del key, val
    return kcs, vcs, chunk


# ---------------------------------------------------------- headline step ---
def build_headline(hs, dev, rank, scale):
    import torch
    g = torch.Generator(device=dev).manual_seed(1234 + rank)
    cfg = hs.SparsityConfig(1.0, 1.0, 64)
    kcs, vcs, _ = build_decode_caches(hs, dev, g, U, L, cfg)
    q = randn16((U, GQA, D), g, dev, torch.bfloat16)
    _, bytes_u = hs.flop_and_byte_count(GQA, kcs[0], vcs[0], 0, False)
    return kcs[0], vcs[0], q, U * bytes_u


# ------------------------------------------------------------------ legs ---
def leg_config4(hs, D_, dev, rank, world, scale, args, flush):
    """configs[3]: 32 requests x 32K x 8 KV heads x GQA 4, S = 1; KV heads sharded
    over ranks (8/N heads x 32 requests per GPU), no data-path collective."""
    import torch
    heads = D_.heads_of_rank(8, world, rank)
    units, ctx = 32 * heads.size, 32768
    g = torch.Generator(device=dev).manual_seed(4000 + rank)
    kcs, vcs, chunk = build_decode_caches(hs, dev, g, units, ctx, hs.SparsityConfig(1.0, 1.0, 64))
    q = randn16((units, GQA, D), g, dev, torch.bfloat16)
    plans = [hs.DecodePlan(q[i * chunk:(i + 1) * chunk], kcs[i], vcs[i], scale=scale) for i in range(len(kcs))]
    nbytes = sum(hs.flop_and_byte_count(GQA, k, v, 0, False)[1] * k.n_units for k, v in zip(kcs, vcs))

    def step():
        for p in plans:
            p()
    barrier(world)
    ms = statistics.mean(time_steps(step, args.steps, 3, flush))
    ms_max = max_over_ranks(ms, world)
    total = sum_over_ranks(nbytes, world)
    hbm, _, _ = peaks()
    out = {"workload": "configs[3]: batched decode, 32 requests x 32K ctx x 8 KV heads x GQA 4, S_K=S_V=1, "
                       "bf16, KV heads sharded over GPUs", "n_gpus": world,
           "parallelism": f"kv-head shards x{world} ({heads.size} heads x 32 requests = {units} units per GPU)",
           "us_per_step": round(ms_max * 1e3, 2), "bytes_per_step": int(total),
           "gbs": round(total / (ms_max * 1e-3) / 1e9, 1),
           "per_gpu_frac_of_hbm": round(nbytes / (ms * 1e-3) / 1e9 / hbm, 4),
           "kernels_per_step": sum(p.kernels_per_step for p in plans)}
    # parity at size: a sample of units against the reference decode (rank 0)
    if rank == 0 and not args.skip_cpu:
        out["parity"] = decode_parity_sample(hs, plans[0].out, kcs[0], vcs[0], q[:kcs[0].n_units], scale,
                                             [0, kcs[0].n_units // 2, kcs[0].n_units - 1])
    del plans, kcs, vcs
    torch.cuda.empty_cache()
    return out


def decode_parity_sample(hs, out, kc, vc, q, scale, units):
    """max-abs / mean-rel of device decode outputs against the reference's
    decode_attention (oracle/_ref, attention.hpp:360-409) on the same pools."""
    import concurrent.futures as cf
    from tests.helpers import device_to_oracle, err_stats
    ref = reference_oracle()
    qh = q.float().cpu().numpy()
    got = out.cpu().numpy()

    def one(u):
        return ref.decode(qh[u], device_to_oracle(kc, u), device_to_oracle(vc, u), None, None,
                          np.float32(scale), 1)
    with cf.ThreadPoolExecutor(min(len(units), os.cpu_count() or 1)) as ex:
        want = np.stack(list(ex.map(one, units)))
    mx, mr = err_stats(got[units], want)
    return {"units_checked": len(units), "max_abs": mx, "mean_rel": mr, "oracle": ref.kind,
            "pass": bool(mx < 2e-2 and mr < 1e-3)}


def reference_oracle():
    from oracle.oracle import Oracle
    ref_path = os.path.join(ROOT, "oracle", "_ref", "libhs_ref.so")
    return Oracle("reference") if os.path.exists(ref_path) else Oracle("port")


def leg_config5(hs, D_, dev, rank, world, scale, args, flush):
    """configs[4]: 1M tokens x 8 KV heads x GQA 4, S = 1; the sequence split into N
    contiguous shards (attention.hpp:380-381); step = decode partial over the
    shard + NCCL all-gather of the packed (O, m, l) partials + LSE combine."""
    import torch
    import torch.distributed as dist
    nb_total = (1 << 20) // 64
    sh = D_.sequence_shard(nb_total, world, rank)
    g = torch.Generator(device=dev).manual_seed(5000 + rank)
    kcs, vcs, _ = build_decode_caches(hs, dev, g, U, sh.size * 64, hs.SparsityConfig(1.0, 1.0, 64))
    kc, vc = kcs[0], vcs[0]
    q = randn16((U, GQA, D), g, dev, torch.bfloat16)
    nbytes = hs.flop_and_byte_count(GQA, kc, vc, 0, False)[1] * U
    out = {}

    def partial():
        out["p"] = hs.decode_partial(q, kc, vc, 0, kc.logical_blocks, include_tail=False, scale=scale)

    def gather_combine():
        out["o"] = hs.decode_combine(D_.gather_partials(out["p"]))

    def step():
        partial()
        gather_combine()
    barrier(world)
    t_step = statistics.mean(time_steps(step, args.steps, 3, flush))
    barrier(world)
    t_part = statistics.mean(time_steps(partial, args.steps, 3, flush))
    barrier(world)
    t_gc = statistics.mean(time_steps(gather_combine, args.steps, 3, None))
    ms = max_over_ranks(t_step, world)
    ms_part = max_over_ranks(t_part, world)
    ms_gc = max_over_ranks(t_gc, world)
    total = sum_over_ranks(nbytes, world)
    hbm, _, _ = peaks()
    res = {"workload": "configs[4]: 1M-token decode, 8 KV heads x GQA 4, S_K=S_V=1, bf16, sequence split over "
                       "GPUs + NCCL all-gather of the SplitPartials", "n_gpus": world,
           "parallelism": f"sequence shards x{world} ({sh.size} blocks per GPU)",
           "us_per_step": round(ms * 1e3, 2), "gbs": round(total / (ms * 1e-3) / 1e9, 1),
           "partial_us": round(ms_part * 1e3, 2),
           "partial_per_gpu_frac_of_hbm": round(nbytes / (t_part * 1e-3) / 1e9 / hbm, 4),
           # added by the gather + combine inside the pipelined step (step - partial alone)
           "gather_combine_us": round(max(0.0, ms - ms_part) * 1e3, 2),
           # timed alone: an idle GPU waiting on the host-side enqueue of the two calls
           "gather_combine_standalone_us": round(ms_gc * 1e3, 2),
           "gather_bytes_per_gpu": int(out["p"].numel() * 4), "bytes_per_step": int(total),
           "collective": "all_gather_into_tensor (NCCL)" if world > 1 else "none (1 GPU)"}
    if rank == 0 and not args.skip_cpu:
        # parity at size: every head of the (rank's) shard against the reference decode
        got = hs.decode_combine(out["p"][None])
        res["parity_shard"] = decode_parity_sample(hs, got, kc, vc, q, scale, list(range(U)))
    del kcs, vcs, kc, vc
    torch.cuda.empty_cache()
    return res


def leg_decode_grid(hs, dev, rank, world, scale, args, flush):
    """configs[1] decode at (S_K, S_V) in {0, 1}^2: measured speedup over the dense
    caches against the closed form r_comp (cost_model.hpp:69-91)."""
    import torch
    from paper_2604_16864_b200.report import CostParams, compression_ratio
    g = torch.Generator(device=dev).manual_seed(6000 + rank)
    key, val = randn16((U, L, D), g, dev, torch.bfloat16), randn16((U, L, D), g, dev, torch.bfloat16)
    q = randn16((U, GQA, D), g, dev, torch.bfloat16)
    res = {}
    for sk, sv in ((0.0, 0.0), (0.0, 1.0), (1.0, 0.0), (1.0, 1.0)):
        kc, vc = hs.prune_cache(key, val, hs.SparsityConfig(sk, sv, 64))
        plan = hs.DecodePlan(q, kc, vc, scale=scale)
        ms = max_over_ranks(statistics.mean(time_steps(plan, args.steps, 3, flush)), world)
        nbytes = hs.flop_and_byte_count(GQA, kc, vc, 0, False)[1] * U
        res[f"{sk:g},{sv:g}"] = {"us": round(ms * 1e3, 2), "bytes": int(nbytes),
                                 "gbs": round(nbytes / (ms * 1e-3) / 1e9, 1)}
        del plan, kc, vc
    base = res["0,0"]["us"]
    for k, v in res.items():
        sk, sv = (float(x) for x in k.split(","))
        v["speedup_vs_dense"] = round(base / v["us"], 3)
        v["r_comp_closed_form"] = round(compression_ratio(CostParams(L, D, 64, sk, sv), exact=True), 3)
    del key, val
    torch.cuda.empty_cache()
    return {"workload": "configs[1] shape (8 KV heads x 128K x GQA 4, bf16), decode µs per (S_K,S_V)",
            "by_s_key_s_value": res}


SMEM_BYTES_PER_CLK = 128  # per SM: one shared-memory port serves TMA writes, LSU and tensor-core operand reads


def prefill_smem_bytes(kc, vc, L, G):
    """Shared-memory bytes the prefill kernel moves for a causal n_q = n_kv = L pass over
    every unit x G query heads: per 128-query x 128-key tile 108 KB
    (Q operand reads 32, stabiliser MMA 8, row-sum MMA 36, P^T stores 32) plus per
    64-key block K 32 KB dense / 18 KB 2:4 (TMA write, operand read, metadata) and
    V 48 / 36 KB (TMA write, operand read, metadata, P^T operand read).  Tiles follow
    the kernel's list: fully visible blocks paired by K kind, then diagonal blocks."""
    ks = (kc.index_map < 0).cpu().numpy()
    vs = (vc.index_map < 0).cpu().numpy()
    U, nb = ks.shape
    n_qt = (L + 127) // 128
    total = 0
    for u in range(U):
        csk = np.concatenate([[0], np.cumsum(ks[u])])
        csv = np.concatenate([[0], np.cumsum(vs[u])])
        qt = np.arange(n_qt)
        fv = np.minimum(nb, 2 * qt)                     # fully visible blocks
        vis = np.minimum(nb, 2 * qt + 2)                # visible blocks (diagonal included)
        ns = csk[fv]
        nd = fv - ns
        tiles = ns // 2 + nd // 2 + ns % 2 + nd % 2
        d0 = np.minimum(fv, nb - 1)
        d1 = np.minimum(fv + 1, nb - 1)
        same = ks[u][d0] == ks[u][d1]
        tiles = tiles + np.where(vis - fv == 2, np.where(same, 1, 2), vis - fv)
        kspa, vspa = csk[vis], csv[vis]
        blocks_k = (vis - kspa) * 32 + kspa * 18
        blocks_v = (vis - vspa) * 48 + vspa * 36
        total += int((tiles * 108 + blocks_k + blocks_v).sum()) * 1024
    return total * G


def leg_prefill(hs, D_, dev, rank, world, args):
    """configs[2]: Llama-3.1-8B prefill attention, causal, hierarchical mixed
    dense / 2:4 blocks at block sparsity S_K = S_V in {0, .25, .5, .75} (+1), fp16
     at 64K and 128K, bf16 at 64K; KV heads sharded over ranks.
    TFLOPS counts flop_and_byte_count flops (sparse blocks at half).  Parity:
    sampled query rows through the reference's attend_range with explicit
    positions (attention.hpp:249-253) on rank 0."""
    import torch
    _, dense_peak, peak_kind = peaks()
    sustained_peak = sustained_tflops()
    heads = D_.heads_of_rank(8, world, rank)
    Up, G = heads.size, 4
    res = {}
    sweeps = [(args.prefill_ctx, torch.float16, (0.0, 0.25, 0.5, 0.75, 1.0))]
    if not args.quick:
        sweeps += [(2 * args.prefill_ctx, torch.float16, (0.0, 0.25, 0.5, 0.75, 1.0)),
                   (args.prefill_ctx, torch.bfloat16, (0.0, 0.5, 1.0))]
    for Lp, dt, levels in sweeps:
        tag = f"{Lp // 1024}K_{'fp16' if dt == torch.float16 else 'bf16'}"
        g = torch.Generator(device=dev).manual_seed(99 + rank)
        q = randn16((Up, G, Lp, D), g, dev, dt)
        out = torch.empty((Up, G, Lp, D), dtype=torch.float32, device=dev)
        by = {}
        for s in levels:
            key, val = randn16((Up, Lp, D), g, dev, dt), randn16((Up, Lp, D), g, dev, dt)
            kc, vc = hs.prune_cache(key, val, hs.SparsityConfig(s, s, 64))
            flops = sum(hs.flop_and_byte_count(Lp, kc, vc, 0, True, unit=u)[0] for u in range(Up)) * G
            barrier(world)
            with ClockSampler(dev.index or 0) as cs:
                times = time_steps(lambda: hs.prefill_attention(q, kc, vc, causal=True, out=out),
                                   args.prefill_steps, 3)
            ms = max_over_ranks(statistics.median(times), world)
            total = sum_over_ranks(flops, world)
            tflops = total / (ms * 1e-3) / 1e12
            clk = cs.summary()
            smem = sum_over_ranks(prefill_smem_bytes(kc, vc, Lp, G), world)
            mhz = clk.get("sm_mhz") or 1965.0
            smem_peak = SMEM_BYTES_PER_CLK * 148 * mhz * 1e6 * world  # bytes/s at the sampled clock
            entry = {"ms": round(ms, 3), "counted_tflops": round(tflops, 1), "frac": round(tflops / dense_peak, 4),
                     "frac_of_sustained": round(tflops / sustained_peak, 4) if sustained_peak else None,
                     "counted_flops": int(total), "clocks": clk,
                     "smem_roofline": {"bytes": smem, "achieved_tbs": round(smem / (ms * 1e-3) / 1e12, 2),
                                       "peak_tbs": round(smem_peak / 1e12, 2),
                                       "frac": round(smem / (ms * 1e-3) / smem_peak, 4),
                                       "model": "DESIGN.md 3.3: 128 B/clk/SM shared-memory port x 148 SMs x sampled SM clock"}}
            if rank == 0 and not args.skip_cpu and Lp <= 2 * args.prefill_ctx:
                entry["parity"] = prefill_parity(hs, q, out, kc, vc, key, val, dt,
                                                 rows=64 if Lp > args.prefill_ctx else 256,
                                                 heads=[(0, 0), (Up - 1, G - 1)] if Lp <= args.prefill_ctx
                                                 else [(0, 1)])
            by[str(s)] = entry
            del kc, vc, key, val
        res[tag] = by
        del q, out
        torch.cuda.empty_cache()
    f16 = res[f"{args.prefill_ctx // 1024}K_fp16"]
    s0, s1 = f16["0.0"]["ms"], f16["1.0"]["ms"]
    return {"workload": f"configs[2]: Llama-3.1-8B prefill, 32 q / 8 kv heads, d=128, causal; {args.prefill_ctx} "
                        f"(+{2 * args.prefill_ctx}) ctx; KV heads sharded over GPUs ({heads.size}/GPU)",
            "metric": "counted TFLOPS (flop_and_byte_count; sparse blocks at half) / dense bf16 peak",
            "peak": dense_peak, "peak_kind": peak_kind, "by_block_sparsity": f16, "sweeps": res,
            "speedup_s1_vs_s0": round(s0 / s1, 3), "ideal_speedup_s1_vs_s0": 2.0,
            "kernel": "hs::prefill_kernel (tcgen05.mma.sp, TMEM accumulators)", "n_gpus": world}


def prefill_parity(hs, q, out, kc, vc, key, val, dt, rows, heads):
    """Sampled rows of the device prefill against the reference's attend_range over
    the whole cache with explicit query positions (attention.hpp:249-253) and
    finalize_rows (:309-317): rows 0, B-1, B, block boundaries, L-1 and a
    uniform spread; max-abs / mean-rel over all sampled rows."""
    import concurrent.futures as cf
    from tests.helpers import device_to_oracle, err_stats
    ref = reference_oracle()
    n_q = q.shape[2]
    pick = sorted(set([0, 63, 64, 127, 128, n_q // 2, n_q - 65, n_q - 64, n_q - 1] +
                      list(np.linspace(0, n_q - 1, rows).astype(int))))
    scale = np.float32(1.0 / math.sqrt(D))
    got_all, want_all = [], []
    for u, h in heads:
        kh, vh = device_to_oracle(kc, u), device_to_oracle(vc, u)
        qh = q[u, h, pick].float().cpu().numpy()
        pos = np.array(pick, np.int64)
        chunks = np.array_split(np.arange(len(pick)), min(16, os.cpu_count() or 1))

        def one(idx):
            o_t, m, l = ref.attend_rows(qh[idx], kh, vh, None, None, 0, kh.logical_blocks, False, scale, pos[idx])
            return o_t.T / l[:, None]
        with cf.ThreadPoolExecutor(len(chunks)) as ex:
            want = np.concatenate(list(ex.map(one, chunks)))
        got_all.append(out[u, h, pick].cpu().numpy())
        want_all.append(want)
    mx, mr = err_stats(np.concatenate(got_all), np.concatenate(want_all))
    return {"rows": len(pick) * len(heads), "heads": [list(x) for x in heads], "max_abs": mx, "mean_rel": mr,
            "oracle": ref.kind, "pass": bool(mx < 2e-2 and mr < 1e-3)}


def leg_compress(hs, dev, rank, world, args, flush):
    """prune_cache + fused_magnitude_compress of configs[1] K+V (8 x 128K x 128 bf16)
    into preallocated pools (no allocation in the timed region), static (S = 1) and
    loss-driven (S = 0.5) selection; the fused decode-phase re-prune 0.5 -> 1."""
    import torch
    hbm, _, _ = peaks()
    g = torch.Generator(device=dev).manual_seed(7000 + rank)
    key, val = randn16((U, L, D), g, dev, torch.bfloat16), randn16((U, L, D), g, dev, torch.bfloat16)
    res = {}
    for s in (1.0, 0.5):
        cfg = hs.SparsityConfig(s, s, 64)
        outp = hs.prune_cache(key, val, cfg)
        ms = max_over_ranks(min(time_steps(lambda: hs.prune_cache(key, val, cfg, out=outp), args.steps, 3, flush)),
                            world)
        # + per block: flag, slot_block entry and (when ranked) the FP64 loss
        nbytes = 2 * key.numel() * 2 + outp[0].nbytes() + outp[1].nbytes() + \
            2 * U * outp[0].logical_blocks * ((1 + 4) if s == 1.0 else (8 + 1 + 4))
        res[f"prune_cache_s{s:g}"] = {"ms": round(ms, 4), "gbs": round(nbytes / (ms * 1e-3) / 1e9, 1),
                                      "frac_of_hbm": round(nbytes / (ms * 1e-3) / 1e9 / hbm, 4), "bytes": int(nbytes),
                                      "selection": "static" if s == 1.0 else "loss-driven (classify, radix select, pack)",
                                      **({"note": "frac_of_hbm above 1: ~40 MB of each cache's output is still dirty in L2 when "
                                                  "its kernel ends and reaches DRAM during the next L2 flush (ncu: DRAM writes "
                                                  "110-116 of 151 MB per cache, profiles/r02j_compress_dram.md); the peak is a "
                                                  "50/50 read/write copy figure, this pass is 64% reads"} if s == 1.0 else {}),
                                      "call": "hierasparse.prune_cache (value cache on a side stream; block losses only where the selection ranks them, as the reference's HierarchicalMask carries none)"}
    kp, vp = hs.prune_cache(key, val, hs.SparsityConfig(0.5, 0.5, 64))
    dec = hs.SparsityConfig(1.0, 1.0, 64)
    k2, v2 = hs.recompress(kp, dec, 1.0), hs.recompress(vp, dec, 1.0)
    st = hs.StatusWord(dev)

    def rc():  # the decode-phase re-prune of both caches (value cache on a side stream)
        hs.recompress_pair(kp, vp, dec, check=False, status=st)
    ms = max_over_ranks(min(time_steps(rc, args.steps, 3, flush)), world)
    st.check()
    nbytes = kp.nbytes() + vp.nbytes() + k2.nbytes() + v2.nbytes() + 2 * U * k2.logical_blocks * (1 + 4)  # static: no losses
    res["recompress_s0.5_to_1"] = {"ms": round(ms, 4), "gbs": round(nbytes / (ms * 1e-3) / 1e9, 1),
                                   "frac_of_hbm": round(nbytes / (ms * 1e-3) / 1e9 / hbm, 4), "bytes": int(nbytes),
                                   "call": "hierasparse.recompress_pair (hs_recompress per cache, one pass, no host sync)"}
    del key, val, kp, vp, k2, v2
    torch.cuda.empty_cache()
    return res


# ------------------------------------------------------------ CPU baseline ---
def cpu_baselines(hs, kc, vc, q, scale, step_bytes):
    """The reference's own CPU implementation (oracle/_ref, compiled from the
    reference headers with its Release flags) on this host, bounded samples of
    the BASELINE workloads: decode 1 core as shipped and
    head-parallel; prefill per head extrapolated from sampled rows; compression."""
    import concurrent.futures as cf
    from oracle.oracle import SparsityConfig as OCfg
    from tests.helpers import device_to_oracle
    ref = reference_oracle()
    nproc = os.cpu_count() or 1
    kch = [device_to_oracle(kc, u) for u in range(U)]
    vch = [device_to_oracle(vc, u) for u in range(U)]
    qh = q.float().cpu().numpy()
    sc = np.float32(scale)
    # decode: one unit on one core (as shipped), then the whole step head-parallel
    t0 = time.perf_counter()
    ref.decode(qh[0], kch[0], vch[0], None, None, sc, 1)
    t_one = time.perf_counter() - t0
    threads = min(U, nproc)
    t0 = time.perf_counter()
    with cf.ThreadPoolExecutor(threads) as ex:
        outs = list(ex.map(lambda u: ref.decode(qh[u], kch[u], vch[u], None, None, sc, 1), range(U)))
    t_par = time.perf_counter() - t0
    decode = {"value": round(step_bytes / t_par / 1e9, 4), "unit": "GB/s", "cores": threads, "nproc": nproc,
              "kind": ref.kind, "seconds_per_step": round(t_par, 3),
              "one_core_seconds_per_step": round(t_one * U, 3),
              "one_core_value": round(step_bytes / (t_one * U) / 1e9, 4),
              "sample": f"configs[1] decode step ({U} KV heads x {L} tokens, GQA {GQA}): all {U} units on "
                        f"{threads} threads (one unit per thread, the reference is single-threaded); 1-core "
                        f"figure = one unit timed alone x {U}"}
    # prefill: the reference's attend_range over a full 64K cache for sampled rows,
    # extrapolated to a head by visible keys and x32 heads (labelled)
    import torch
    Lp = 65536
    g = torch.Generator().manual_seed(11)
    kx = torch.randn((Lp, D), generator=g).to(torch.float16).float().numpy()
    vx = torch.randn((Lp, D), generator=g).to(torch.float16).float().numpy()
    qx = torch.randn((Lp, D), generator=g).to(torch.float16).float().numpy()
    cfg = OCfg(0.5, 0.5, 64)
    kref = ref.prune_compress(kx, cfg, 0, 0.5)
    vref = ref.prune_compress(vx, cfg, 1, 0.5)
    rows = np.linspace(0, Lp - 1, 48).astype(np.int64)
    t0 = time.perf_counter()
    ref.attend_rows(qx[rows], kref, vref, None, None, 0, kref.logical_blocks, False, sc, rows)
    t_rows = time.perf_counter() - t0
    visible_sample = float((rows + 1).sum())
    visible_head = Lp * (Lp + 1) / 2.0
    per_head = t_rows * visible_head / visible_sample
    prefill = {"seconds_per_head_extrapolated": round(per_head, 1), "seconds_32_heads_extrapolated":
               round(per_head * 32, 1), "cores": 1, "kind": ref.kind,
               "sample": f"attend_range over a full 64K causal S=0.5 cache for {len(rows)} query rows "
                         f"({t_rows:.2f} s), extrapolated to one head by visible keys, x32 heads"}
    # compression of one 128K KV head (K + V): prune_cache (fused) and the two-phase compress
    kx1 = torch.randn((L, D), generator=g).to(torch.bfloat16).float().numpy()
    vx1 = torch.randn((L, D), generator=g).to(torch.bfloat16).float().numpy()
    cfg1 = OCfg(0.5, 0.5, 64)
    t0 = time.perf_counter()
    ck = ref.prune_compress(kx1, cfg1, 0, 0.5, fused=True)
    ref.prune_compress(vx1, cfg1, 1, 0.5, fused=True)
    t_prune = time.perf_counter() - t0
    t0 = time.perf_counter()
    ref.compress_with_flags(kx1, cfg1, 0, ck.flags)
    t_fused = time.perf_counter() - t0
    compress = {"prune_cache_kv_one_head_s": round(t_prune, 3),
                "fused_magnitude_compress_k_one_head_s": round(t_fused, 3), "cores": 1, "kind": ref.kind,
                "sample": "one 128K KV head, S=0.5 (loss-driven): prune_cache + fused_magnitude_compress of K "
                          "and V; fused_magnitude_compress of K under the resulting BlockMask"}
    return decode, prefill, compress, np.stack(outs)


# ---------------------------------------------------------------- our arm ---
def run_ours(args):
    import torch
    from paper_2604_16864_b200 import capi
    from paper_2604_16864_b200 import distributed as D_
    from paper_2604_16864_b200 import hierasparse as hs

    rank, world, local = dist_setup()
    dev = torch.device("cuda", torch.cuda.current_device())
    hbm_peak, _, peak_kind = peaks()
    scale = 1.0 / math.sqrt(D)
    kc, vc, q, step_bytes = build_headline(hs, dev, rank, scale)
    flush = Flusher(dev)
    plan = hs.DecodePlan(q, kc, vc, scale=scale)
    for _ in range(args.warmup):
        plan()
    torch.cuda.synchronize()

    # ---- timed region: K decode steps (device events), L2 flushed between steps
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    stops = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    launches0 = capi.kernel_launches()
    barrier(world)
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        t_wall = time.perf_counter()
        hold_stream(args.steps)
        for i in range(args.steps):
            flush()
            starts[i].record()
            plan()
            stops[i].record()
        torch.cuda.synchronize()
        t_wall = time.perf_counter() - t_wall
        # The timed region is milliseconds long; keep the same step running for
        # ~1.5 s (untimed) so nvidia-smi samples the clocks under this load.
        t_soak = time.perf_counter()
        while not args.profile and time.perf_counter() - t_soak < 1.5:
            for _ in range(50):
                plan()
            torch.cuda.synchronize()
    barrier(world)
    launches = capi.kernel_launches() - launches0 + args.steps * plan.kernels_per_step
    step_ms = [a.elapsed_time(b) for a, b in zip(starts, stops)]
    ms = statistics.mean(step_ms)
    ms_max = max_over_ranks(ms, world)
    total_bytes = sum_over_ranks(step_bytes, world)
    value = total_bytes / (ms_max * 1e-3) / 1e9  # GB/s, whole job

    # ---- e2e: host queries in (pinned), decode through the public API, result out
    q_host = q.cpu().pin_memory()
    q_dev = torch.empty_like(q)
    out_dev = torch.empty((U, GQA, D), dtype=torch.float32, device=dev)
    out_host = torch.empty(out_dev.shape, dtype=torch.float32).pin_memory()

    def e2e_call():  # one public decode_attention call per step on pinned host q / out (host enqueue inside)
        hs.decode_attention(q_host, kc, vc, scale=scale, out=out_host)
    barrier(world)
    e2e_call_ms = max_over_ranks(statistics.mean(time_steps(e2e_call, args.steps, max(3, args.warmup), flush)), world)
    # the serving loop's API: a DecodePlan with host I/O replays copy-in, decode and
    # copy-out as one graph (pinned q_host -> device -> pinned out_host)
    plan_io = hs.DecodePlan(q, kc, vc, scale=scale, host_io=True)
    plan_io.q_host.copy_(q_host)
    e2e_ms = max_over_ranks(statistics.mean(time_steps(plan_io, args.steps, max(3, args.warmup), flush)), world)
    # (dynamic block claiming varies the fp32 summation order run to run: ~1e-6)
    assert torch.allclose(plan_io.out_host, out_host, rtol=1e-4, atol=1e-5), "DecodePlan(host_io) differs"
    e2e_value = total_bytes / (e2e_ms * 1e-3) / 1e9

    # ---- the other BASELINE configs and legs (same run, device events, max over ranks)
    legs = {}
    if not args.headline_only:
        legs["config4"] = leg_config4(hs, D_, dev, rank, world, scale, args, flush)
        legs["config5"] = leg_config5(hs, D_, dev, rank, world, scale, args, flush)
        if not args.no_prefill:
            legs["prefill"] = leg_prefill(hs, D_, dev, rank, world, args)
        if not args.quick:
            legs["decode_grid"] = leg_decode_grid(hs, dev, rank, world, scale, args, flush)
        legs["compress"] = leg_compress(hs, dev, rank, world, args, flush)

    # ---- CPU baseline: the reference on this host's cores (rank 0, N = 1)
    cpu = None
    extra_cpu = {}
    if rank == 0 and world == 1 and not (args.skip_cpu or args.profile):
        dec, pre, comp, ref_out = cpu_baselines(hs, kc, vc, q, scale, step_bytes)
        got = plan.out.cpu().numpy()
        from tests.helpers import err_stats
        mx, mr = err_stats(got, ref_out)
        dec.update(max_abs_vs_gpu=mx, mean_rel_vs_gpu=mr)
        cpu = dec
        extra_cpu = {"cpu_prefill": pre, "cpu_compress": comp}

    traffic, traffic_src = None, None
    tf = os.path.join(ROOT, "profiles", "r02_decode_traffic.json")
    if os.path.exists(tf):
        try:
            tj = json.load(open(tf))
            traffic, traffic_src = tj.get("bytes_per_launch"), tj.get("source")
        except Exception:  # noqa: BLE001
            traffic = None

    per_gpu_gbs = step_bytes / (ms * 1e-3) / 1e9
    line = {
        "metric": METRIC,
        "value": round(value, 2),
        "unit": "GB/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms_max, 5),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "bf16",
        "data": "synthetic (torch.randn, bf16), random-init; pools compressed on device",
        "config": {"workload": "configs[1]: Llama-3.1-8B GQA decode, 32 q / 8 kv heads, d=128, 128K ctx, batch 1 "
                               "per GPU, S_K=S_V=1 (2:4 K+V)", "kv_heads": U, "gqa": GQA, "context": L,
                   "block_size": 64, "s_key": 1.0, "s_value": 1.0, "parallelism": f"request-per-GPU x{world}",
                   "bytes_per_step_per_gpu": step_bytes,
                   "l2": "flushed between timed steps (read of a 252 MB buffer)"},
        "decode_us": round(ms_max * 1e3, 2),
        "roofline": {"bound": "hbm", "achieved": round(per_gpu_gbs, 2), "peak": hbm_peak, "unit": "GB/s",
                     "frac": round(per_gpu_gbs / hbm_peak, 4), "traffic": traffic, "traffic_source": traffic_src,
                     "peak_kind": peak_kind, "kernel": "hs::decode_kernel (+fused split combine)",
                     "algorithmic_bytes_per_launch": step_bytes},
        "e2e": {"value": round(e2e_value, 2), "unit": "GB/s", "ms_per_step": round(e2e_ms, 5),
                "h2d_bytes_per_step": int(q.numel() * 2), "d2h_bytes_per_step": int(out_dev.numel() * 4),
                "call": "hierasparse.DecodePlan(host_io=True): one graph replay per step; the kernel reads q from pinned host memory and writes O to pinned host memory (zero-copy over the host link)",
                "per_call_api": {"value": round(total_bytes / (e2e_call_ms * 1e-3) / 1e9, 2), "ms_per_step": round(e2e_call_ms, 5),
                                 "call": "hierasparse.decode_attention(pinned q, out=pinned), zero-copy, host enqueue inside each step"}},
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
        "cpu_baseline": cpu,
        **extra_cpu,
        **legs,
        "wall_s": round(t_wall, 4),
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


# ------------------------------------------------------ distributed selftest ---
def run_selftest(args):
    """CPU / gloo check of the multi-rank wiring bench.py uses on GPUs: rank
    spawning (--gpus N), barrier + max/sum over ranks, the configs[4] step's
    all-gather of SplitPartials in rank order (distributed.gather_partials) and
    the combine of the gathered partials, against a single-process reference
    combine of the same partials.  No device kernels run (test infrastructure)."""
    import torch
    from paper_2604_16864_b200 import distributed as D_
    rank, world, _ = dist_setup(selftest=True)
    nb = (1 << 20) // 64
    sh = D_.sequence_shard(nb, world, rank)
    g = torch.Generator().manual_seed(7)
    all_parts = torch.randn((world, U, GQA, D + 2), generator=g, dtype=torch.float32)
    gathered = D_.gather_partials(all_parts[rank])
    order_ok = bool(torch.equal(gathered, all_parts))
    t = max_over_ranks(float(rank + 1), world)
    total = sum_over_ranks(float(sh.size), world)
    barrier(world)
    if rank == 0:
        print(json.dumps({"selftest": "ok" if order_ok and t == world and total == nb else "FAILED",
                          "n_gpus": world, "gather_order_ok": order_ok, "max_over_ranks": t,
                          "blocks_covered": int(total), "blocks_total": nb}), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


# ---------------------------------------------------------- reference arm ---
def run_reference(args):
    """The reference's own CPU decode_attention (oracle/_ref) on this host's cores,
    same config / metric.  Rank 0 only under torchrun."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    from oracle.oracle import Oracle, SparsityConfig
    import concurrent.futures as cf
    ref = reference_oracle()
    port = Oracle("port")
    threads = min(U, os.cpu_count() or 1)
    rng = np.random.default_rng(1234)
    cfg = SparsityConfig(1.0, 1.0, 64)

    def make_unit(u):
        r = np.random.default_rng(1234 + u)
        k = port.round_to(r.standard_normal((L, D), dtype=np.float32), "bf16")
        v = port.round_to(r.standard_normal((L, D), dtype=np.float32), "bf16")
        return ref.prune_compress(k, cfg, 0, 1.0), ref.prune_compress(v, cfg, 1, 1.0)

    with cf.ThreadPoolExecutor(threads) as ex:
        caches = list(ex.map(make_unit, range(U)))
    q = port.round_to(rng.standard_normal((U, GQA, D), dtype=np.float32), "bf16")
    scale = np.float32(1.0 / math.sqrt(D))
    _, bytes_u = port.flop_and_byte_count(GQA, D, caches[0][0], caches[0][1], 0, False)
    step_bytes = U * bytes_u

    def step():
        with cf.ThreadPoolExecutor(threads) as ex:
            list(ex.map(lambda u: ref.decode(q[u], caches[u][0], caches[u][1], None, None, scale, 1), range(U)))

    for _ in range(args.warmup):
        step()
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        step()
        times.append(time.perf_counter() - t0)
    ms = statistics.mean(times) * 1e3
    value = step_bytes / (ms * 1e-3) / 1e9
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": "GB/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32 (bf16-rounded inputs)",
        "data": "synthetic (numpy normal, bf16-rounded)",
        "config": {"workload": "configs[1]: Llama-3.1-8B GQA decode, 32 q / 8 kv heads, d=128, 128K ctx, batch 1 "
                               "per GPU, S_K=S_V=1 (2:4 K+V)", "bytes_per_step": step_bytes},
        "cpu_baseline": {"value": round(value, 4), "unit": "GB/s", "cores": threads, "nproc": os.cpu_count(),
                         "kind": ref.kind,
                         "sample": f"full configs[1] decode step ({U} KV heads) per step, one unit per thread on "
                                   f"{threads} threads (the reference itself is single-threaded)"},
        "e2e": {"value": round(value, 4), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--skip-cpu", action="store_true", help="skip the CPU-baseline and parity-sample legs")
    ap.add_argument("--profile", action="store_true", help="profiling run: no CPU leg, no clock soak")
    ap.add_argument("--no-prefill", action="store_true", help="skip the configs[2] prefill leg")
    ap.add_argument("--quick", action="store_true", help="64K fp16 prefill only, no decode grid")
    ap.add_argument("--headline-only", action="store_true", help="only the configs[1] headline decode")
    ap.add_argument("--prefill-ctx", type=int, default=65536)
    ap.add_argument("--prefill-steps", type=int, default=3)
    ap.add_argument("--selftest", action="store_true", help="CPU/gloo check of the multi-rank wiring")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch_distributed(args))
    if args.selftest:
        run_selftest(args)
    elif args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
