"""Benchmark of the HieraSparse hot path on B200 (driver contract).

Headline workload (BASELINE.json configs[1]): Llama-3.1-8B GQA decode, 8 KV
heads x 4 query rows, 128K-token context, batch 1, S_K = S_V = 1 (every block
2:4), bf16 pools.  A step = one decode_attention over all 8 KV heads with the
compressed caches resident in HBM.  `value` = algorithmic bytes moved
(flop_and_byte_count, attention.hpp:426-467: pools + index maps + headers)
per second, aggregated over ranks.  N > 1: every rank decodes its own request
(weak scaling, no data-path collective).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import math
import os
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


def dist_setup(n_gpus):
    import torch
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    elif torch.cuda.is_available():
        torch.cuda.set_device(0)
    return rank, world, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t)
    return float(t.item())


# --------------------------------------------------------------- CPU legs ---
def cpu_reference_decode(kc_host, vc_host, q, scale, threads):
    """The reference's own decode_attention (oracle/_ref, compiled from the
    reference headers) over every unit, head-parallel on `threads` cores."""
    import concurrent.futures as cf
    from oracle.oracle import Oracle
    ref = Oracle("reference") if os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libhs_ref.so")) \
        else Oracle("port")
    t0 = time.perf_counter()
    with cf.ThreadPoolExecutor(threads) as ex:
        outs = list(ex.map(lambda u: ref.decode(q[u], kc_host[u], vc_host[u], None, None, scale, 1),
                           range(len(kc_host))))
    return time.perf_counter() - t0, np.stack(outs), ref.kind


def host_caches(dev, units):
    from tests.helpers import device_to_oracle
    return [device_to_oracle(dev, u) for u in units]


# ---------------------------------------------------------------- our arm ---
def build_workload(args, hs, dev, rank, world, scale):
    """The decode workload this rank runs (synthetic bf16 K/V, compressed on device):

    config2 (headline, BASELINE configs[1]): this rank's own request, 8 KV heads x
        GQA 4 x 128K, S_K=S_V=1 — weak scaling over ranks, no collective.
    config4 (configs[3]): 32 requests x 32K x 8 KV heads, KV heads sharded over the
        ranks (each rank: 8/N heads x 32 requests = 256/N units) — strong scaling.
    config5 (configs[4]): 1 request x 1M tokens x 8 KV heads, the sequence split
        into N contiguous shards (distributed.sequence_shard); each step = decode
        partial over the shard + NCCL all-gather of the (O, m, l) partials +
        LSE combine — strong scaling."""
    import torch
    from paper_2604_16864_b200 import distributed as Dd
    cfg = hs.SparsityConfig(1.0, 1.0, 64)
    g = torch.Generator(device=dev).manual_seed(1234 + rank)
    if args.workload == "config2":
        units, L_ctx, blocks = U, L, L // 64
        desc = {"workload": "configs[1]: Llama-3.1-8B GQA decode, 32 q / 8 kv heads, d=128, 128K ctx, batch 1 "
                            "per GPU, S_K=S_V=1 (2:4 K+V)", "kv_heads": U, "gqa": GQA, "context": L,
                "block_size": 64, "s_key": 1.0, "s_value": 1.0, "parallelism": f"request-per-GPU x{world}"}
        scaling = "weak"
    elif args.workload == "config4":
        heads = Dd.heads_of_rank(8, world, rank)
        units, L_ctx, blocks = 32 * heads.size, 32768, 32768 // 64
        desc = {"workload": "configs[3]: batched decode, 32 requests x 32K ctx x 8 KV heads x GQA 4, S_K=S_V=1, "
                            "KV heads sharded over GPUs", "requests": 32, "kv_heads": 8, "gqa": GQA,
                "context": 32768, "parallelism": f"kv-head shards x{world} ({heads.size} heads/GPU)"}
        scaling = "strong"
    elif args.workload == "config5":
        sh = Dd.sequence_shard(1 << 14, world, rank)
        units, L_ctx, blocks = U, sh.size * 64, sh.size
        desc = {"workload": "configs[4]: 1M-token decode, 8 KV heads x GQA 4, S_K=S_V=1, sequence split over "
                            "GPUs + NCCL all-gather of partials", "kv_heads": U, "gqa": GQA, "context": 1 << 20,
                "parallelism": f"sequence shards x{world} ({sh.size} blocks/GPU)"}
        scaling = "strong"
    else:
        raise SystemExit(f"unknown workload {args.workload}")
    # compress in chunks of units to bound the dense staging buffer (<= 4 GB)
    chunk = max(1, min(units, (1 << 31) // (L_ctx * D * 2)))
    kcs, vcs = [], []
    comp_ms = []
    comp_bytes = 0
    rc_ms, rc_bytes = [], 0
    for c0 in range(0, units, chunk):
        n = min(chunk, units - c0)
        key = torch.randn((n, L_ctx, D), generator=g, device=dev, dtype=torch.float32).to(torch.bfloat16)
        val = torch.randn((n, L_ctx, D), generator=g, device=dev, dtype=torch.float32).to(torch.bfloat16)
        if c0 == 0:  # compression (prune_cache + fused_magnitude_compress) timed on the first chunk
            for _ in range(3):
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                kc0, vc0 = hs.prune_cache(key, val, cfg)
                e1.record()
                torch.cuda.synchronize()
                comp_ms.append(e0.elapsed_time(e1))
            comp_bytes = 2 * key.numel() * 2 + kc0.nbytes() + vc0.nbytes() + 2 * n * kc0.logical_blocks * (8 + 1 + 4)
            # decode-phase re-prune (pipeline.hpp:227-240) of prefill-sparsity caches
            # (S = 0.5) to the decode sparsity, fused over the compressed pools
            kp, vp = hs.prune_cache(key, val, hs.SparsityConfig(0.5, 0.5, 64))
            for _ in range(3):
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                k2, v2 = hs.recompress(kp, cfg, cfg.s_key), hs.recompress(vp, cfg, cfg.s_value)
                e1.record()
                torch.cuda.synchronize()
                rc_ms.append(e0.elapsed_time(e1))
            rc_bytes = (kp.nbytes() + vp.nbytes() + k2.nbytes() + v2.nbytes() +
                        2 * n * k2.logical_blocks * (8 + 1 + 4))
            del kp, vp, k2, v2
            kcs.append(kc0)
            vcs.append(vc0)
        else:
            kc0, vc0 = hs.prune_cache(key, val, cfg)
            kcs.append(kc0)
            vcs.append(vc0)
        del key, val
    q = torch.randn((units, GQA, D), generator=g, device=dev, dtype=torch.float32).to(torch.bfloat16)
    _, bytes_u = hs.flop_and_byte_count(GQA, kcs[0], vcs[0], 0, False)
    step_bytes = units * bytes_u
    wl = {"kc": kcs[0], "vc": vcs[0], "q": q, "bytes": step_bytes, "config": desc, "scaling": scaling,
          "comp_ms": comp_ms, "comp_bytes": comp_bytes, "rc_ms": rc_ms, "rc_bytes": rc_bytes, "plan": None}
    if args.workload == "config5":
        last = rank == world - 1

        def call(qd):
            return Dd.sequence_split_decode(qd, kcs[0], vcs[0], is_last=last, scale=scale)
        wl["step"] = lambda: call(q)
        wl["e2e_call"] = call
        wl["e2e_name"] = "distributed.sequence_split_decode (decode_partial + all-gather + decode_combine)"
        return wl
    # one CUDA graph per chunk of units (the decode step of every unit of this rank)
    plans = [hs.DecodePlan(q[i * chunk:(i + 1) * chunk], kcs[i], vcs[i], scale=scale) for i in range(len(kcs))]

    class MultiPlan:
        kernels_per_step = sum(p.kernels_per_step for p in plans)
        out = plans[0].out

        def __call__(self):
            for p in plans:
                p()
    wl["plan"] = MultiPlan()
    wl["step"] = wl["plan"]
    outs = [torch.empty((kc.n_units, GQA, D), dtype=torch.float32, device=dev) for kc in kcs]

    def call(qd):
        for i in range(len(kcs)):
            hs.decode_attention(qd[i * chunk:(i + 1) * chunk], kcs[i], vcs[i], scale=scale, out=outs[i])
        return outs[0] if len(outs) == 1 else torch.cat(outs)
    wl["e2e_call"] = call
    wl["e2e_name"] = "hierasparse.decode_attention"
    return wl


def run_ours(args):
    import torch
    from paper_2604_16864_b200 import capi
    from paper_2604_16864_b200 import hierasparse as hs

    rank, world, local = dist_setup(args.gpus)
    dev = torch.device("cuda", torch.cuda.current_device())
    hbm_peak, _, peak_kind = peaks()
    scale = 1.0 / math.sqrt(D)
    wl = build_workload(args, hs, dev, rank, world, scale)
    kc, vc, q, step_bytes = wl["kc"], wl["vc"], wl["q"], wl["bytes"]
    comp_ms, comp_bytes = wl["comp_ms"], wl["comp_bytes"]
    # L2 flush between timed steps: read (not write) a 2x-L2 buffer, so the next
    # step starts with an L2 full of clean, unrelated lines (a write flush would
    # charge ~126 MB of dirty-line writebacks to the timed kernel).
    flush = torch.ones(2 * L2_BYTES // 4, dtype=torch.float32, device=dev)
    flush_sink = torch.empty((), dtype=torch.float32, device=dev)

    def flush_l2():
        torch.sum(flush, dim=0, out=flush_sink)

    plan = wl["plan"]
    step = wl["step"]
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    # ---- timed region: K decode steps (device events), L2 flushed between steps
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    stops = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    launches0 = capi.kernel_launches()
    barrier(world)
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        t_wall = time.perf_counter()
        for i in range(args.steps):
            flush_l2()
            starts[i].record()
            step()
            stops[i].record()
        torch.cuda.synchronize()
        t_wall = time.perf_counter() - t_wall
        # The timed region is milliseconds long; keep the same step running for
        # ~1.5 s (untimed) so nvidia-smi samples the clocks under this load.
        t_soak = time.perf_counter()
        while not args.profile and time.perf_counter() - t_soak < 1.5:
            for _ in range(50):
                step()
            torch.cuda.synchronize()
    barrier(world)
    launches = capi.kernel_launches() - launches0 + (args.steps * plan.kernels_per_step if plan else 0)
    step_ms = [a.elapsed_time(b) for a, b in zip(starts, stops)]
    ms = statistics.mean(step_ms)
    ms_max = max_over_ranks(ms, world)
    total_bytes = sum_over_ranks(step_bytes, world)
    value = total_bytes / (ms_max * 1e-3) / 1e9  # GB/s, whole job

    # ---- e2e: host queries in (pinned), decode through the public API, result out
    q_host = q.cpu().pin_memory()
    q_dev = torch.empty_like(q)
    e2e_call = wl["e2e_call"]
    out = e2e_call(q_dev)
    out_host = torch.empty(out.shape, dtype=out.dtype).pin_memory()
    for _ in range(max(3, args.warmup)):
        q_dev.copy_(q_host, non_blocking=True)
        out = e2e_call(q_dev)
        out_host.copy_(out, non_blocking=True)
    torch.cuda.synchronize()
    e_s = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    e_t = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    barrier(world)
    for i in range(args.steps):
        flush_l2()
        e_s[i].record()
        q_dev.copy_(q_host, non_blocking=True)
        out = e2e_call(q_dev)
        out_host.copy_(out, non_blocking=True)
        e_t[i].record()
    torch.cuda.synchronize()
    e2e_ms = max_over_ranks(statistics.mean(a.elapsed_time(b) for a, b in zip(e_s, e_t)), world)
    e2e_value = total_bytes / (e2e_ms * 1e-3) / 1e9

    # ---- prefill (configs[2]): 32 q / 8 kv heads, 64K causal, S in {0,.25,.5,.75}
    prefill = None if (args.no_prefill or args.workload != "config2") else run_prefill(hs, dev, rank, args)

    # ---- CPU baseline: the reference's decode on this host's cores (rank 0, N=1)
    cpu = None
    if rank == 0 and world == 1 and args.workload == "config2" and not (args.skip_cpu or args.profile):
        threads = min(16, os.cpu_count() or 1)
        units = list(range(U))
        kch, vch = host_caches(kc, units), host_caches(vc, units)
        qh = q.float().cpu().numpy()
        secs, ref_out, kind = cpu_reference_decode(kch, vch, qh, np.float32(scale), threads)
        got = plan.out.cpu().numpy()
        err = float(np.abs(got - ref_out).max())
        cpu = {"value": round(step_bytes / secs / 1e9, 4), "unit": "GB/s", "cores": threads,
               "kind": kind, "seconds": round(secs, 3), "max_abs_vs_gpu": err,
               "sample": f"one full configs[1] decode step ({U} KV heads x {L} tokens, GQA {GQA}) "
                         f"head-parallel on {threads} threads"}

    traffic = None
    tf = os.path.join(ROOT, "profiles", "decode_traffic.json")
    if os.path.exists(tf):
        try:
            traffic = json.load(open(tf)).get("bytes_per_launch")
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
        "scaling": wl["scaling"],
        "vs_baseline": None,
        "dtype": "bf16",
        "data": "synthetic (torch.randn, bf16), random-init; pools compressed on device",
        "config": dict(wl["config"], bytes_per_step_per_gpu=step_bytes,
                       l2="flushed between timed steps (read of a 252 MB buffer)"),
        "decode_us": round(ms_max * 1e3, 2),
        "roofline": {"bound": "hbm", "achieved": round(per_gpu_gbs, 2), "peak": hbm_peak, "unit": "GB/s",
                     "frac": round(per_gpu_gbs / hbm_peak, 4), "traffic": traffic,
                     "peak_kind": peak_kind, "kernel": "hs::decode_kernel (+fused split combine)"}
        if args.workload == "config2" else None,
        "e2e": {"value": round(e2e_value, 2), "unit": "GB/s", "ms_per_step": round(e2e_ms, 5),
                "h2d_bytes_per_step": int(q.numel() * 2), "d2h_bytes_per_step": int(out.numel() * 4),
                "call": wl["e2e_name"]},
        "compress": {"ms": round(min(comp_ms), 4), "gbs": round(comp_bytes / (min(comp_ms) * 1e-3) / 1e9, 2),
                     "bytes": int(comp_bytes)},
        "recompress": {"from_s": 0.5, "to_s": 1.0, "ms": round(min(wl["rc_ms"]), 4),
                       "gbs": round(wl["rc_bytes"] / (min(wl["rc_ms"]) * 1e-3) / 1e9, 2),
                       "bytes": int(wl["rc_bytes"]), "call": "hierasparse.recompress x2 (hs_recompress, one pass)"}
        if wl.get("rc_ms") else None,
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
        "cpu_baseline": cpu,
        "prefill": prefill,
        "wall_s": round(t_wall, 4),
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def run_prefill(hs, dev, rank, args):
    """configs[2]: Llama-3.1-8B prefill attention at 64K context, causal,
    hierarchical mixed dense/2:4 blocks at block sparsity S_K = S_V in
    {0, .25, .5, .75}; fp16 (P in fp16 meets the 1e-3 bar).
    TFLOPS counts flop_and_byte_count flops (sparse blocks at half)."""
    import torch
    _, dense_peak, peak_kind = peaks()
    Lp, Up, G = args.prefill_ctx, 8, 4
    g = torch.Generator(device=dev).manual_seed(99 + rank)
    q = torch.randn((Up, G, Lp, D), generator=g, device=dev, dtype=torch.float32).half()
    out = torch.empty((Up, G, Lp, D), dtype=torch.float32, device=dev)
    res = {}
    for s in (0.0, 0.25, 0.5, 0.75, 1.0):
        key = torch.randn((Up, Lp, D), generator=g, device=dev, dtype=torch.float32).half()
        val = torch.randn((Up, Lp, D), generator=g, device=dev, dtype=torch.float32).half()
        kc, vc = hs.prune_cache(key, val, hs.SparsityConfig(s, s, 64))
        del key, val
        flops = sum(hs.flop_and_byte_count(Lp, kc, vc, 0, True, unit=u)[0] for u in range(Up)) * G
        hs.prefill_attention(q, kc, vc, causal=True, out=out)
        torch.cuda.synchronize()
        times = []
        for _ in range(args.prefill_steps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            hs.prefill_attention(q, kc, vc, causal=True, out=out)
            e1.record()
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
        ms = statistics.median(times)
        tflops = flops / (ms * 1e-3) / 1e12
        res[str(s)] = {"ms": round(ms, 3), "counted_tflops": round(tflops, 1),
                       "frac": round(tflops / dense_peak, 4), "counted_flops": flops}
        del kc, vc
    return {"workload": f"configs[2]: Llama-3.1-8B prefill, 32 q / 8 kv heads, d=128, {Lp} ctx, causal, fp16",
            "metric": "counted TFLOPS (flop_and_byte_count; sparse blocks at half) / dense bf16 peak",
            "peak": dense_peak, "peak_kind": peak_kind, "by_block_sparsity": res,
            "kernel": "hs::prefill_kernel (tcgen05.mma.sp, TMEM accumulators)"}


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
    ref_path = os.path.join(ROOT, "oracle", "_ref", "libhs_ref.so")
    ref = Oracle("reference") if os.path.exists(ref_path) else Oracle("port")
    port = Oracle("port")
    threads = min(16, os.cpu_count() or 1)
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
        "config": {"workload": "configs[1]: Llama-3.1-8B GQA decode, 8 kv heads x GQA 4, d=128, 128K ctx, "
                               "S_K=S_V=1", "bytes_per_step": step_bytes},
        "cpu_baseline": {"value": round(value, 4), "unit": "GB/s", "cores": threads, "kind": ref.kind,
                         "sample": f"full configs[1] decode step ({U} KV heads) per step, head-parallel on "
                                   f"{threads} threads"},
        "e2e": {"value": round(value, 4), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--skip-cpu", action="store_true", help="skip the CPU-baseline leg")
    ap.add_argument("--profile", action="store_true", help="profiling run: no CPU leg, no clock soak")
    ap.add_argument("--no-prefill", action="store_true", help="skip the configs[2] prefill leg")
    ap.add_argument("--prefill-ctx", type=int, default=65536)
    ap.add_argument("--prefill-steps", type=int, default=3)
    ap.add_argument("--workload", default="config2", choices=["config2", "config4", "config5"],
                    help="config2 (headline) | config4 batched KV-head sharding | config5 1M sequence split")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
