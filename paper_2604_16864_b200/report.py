"""Closed-form cost model and a run_pipeline-shaped report fed by B200 results.

Cost model (cost_model.hpp:17-137, restated as host arithmetic): analytic cache
sizes (Eq. 5), the compression ratio r_comp, the ideal prefill / decode speedups
and the GEMM-orientation design-space table.

`run_pipeline` mirrors pipeline.hpp:137-299 on the device: synthetic K/V per KV
head, prune + compress at the prefill sparsities, causal prefill over the
compressed caches, re-prune at the decode sparsities, one decode step per KV
head, operation counts (flop_and_byte_count) and the closed forms, in the JSON
schema of report_json.hpp:55-84, extended with a "b200" section: measured device
times, achieved GB/s / TFLOP/s, roofline fractions and the measured speedup of
each phase against the same run with dense caches (S = 0).  Accuracy is taken
against a PyTorch fp32 two-pass softmax attention over the decompressed caches
(dense_attention_oracle semantics, attention.hpp:84-115).

    python -m paper_2604_16864_b200.report cost --s-key 1 --s-value 1
    python -m paper_2604_16864_b200.report run --seq-len 8192 --heads 8 --gqa 4 --out report.json

Exit codes follow bench_cli.cpp:21-23: 2 ConfigError, 3 IoError, 4 DataError.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys
from dataclasses import asdict, dataclass

from .errors import ConfigError, DataError, IoError

# --------------------------------------------------------------- cost model ---


@dataclass
class CostParams:
    """cost_model.hpp:17-35."""

    seq_len: int = 4096
    hidden_dim: int = 128
    block_size: int = 64
    s_key: float = 0.0
    s_value: float = 0.0
    dense_throughput: float = 1.0
    metadata_fraction: float = 1.0 / 16.0
    nnz_fraction: float = 1.0 / 2.0

    def validate(self) -> None:
        if not (self.seq_len > 0 and self.hidden_dim > 0 and self.block_size > 0):
            raise ConfigError("CostParams: L, D, B must be positive")
        if not (0.0 <= self.s_key <= 1.0 and 0.0 <= self.s_value <= 1.0):
            raise ConfigError("CostParams: sparsities outside [0, 1]")
        if not self.dense_throughput > 0.0:
            raise ConfigError("CostParams: dense_throughput must be positive")


def analytic_sizes(p: CostParams) -> dict:
    """Eq. 5 sizes in bytes, both caches (cost_model.hpp:51-61)."""
    p.validate()
    ld = float(p.seq_len) * float(p.hidden_dim)
    s = p.s_key + p.s_value
    sizes = {"size_idx": 2.0 * p.seq_len / p.block_size * 2.0, "size_den": ld * (2.0 - s) * 2.0,
             "size_nnz": ld * s * p.nnz_fraction * 2.0, "size_e": ld * s * p.metadata_fraction * 2.0}
    sizes["total"] = sizes["size_idx"] + sizes["size_den"] + sizes["size_nnz"] + sizes["size_e"]
    return sizes


def compression_ratio(p: CostParams, exact: bool) -> float:
    """r_comp (cost_model.hpp:69-77)."""
    p.validate()
    savings = (1.0 - p.nnz_fraction - p.metadata_fraction) / 2.0
    denom = 1.0 - savings * (p.s_key + p.s_value)
    if exact:
        denom += 1.0 / (float(p.block_size) * float(p.hidden_dim))
    return 1.0 / denom


def prefill_speedup(p: CostParams) -> float:
    """4 / (4 - S_K - S_V) (cost_model.hpp:82-85)."""
    p.validate()
    return 4.0 / (4.0 - (p.s_key + p.s_value))


def decode_speedup(p: CostParams) -> float:
    """= approximate r_comp (cost_model.hpp:89-91)."""
    return compression_ratio(p, exact=False)


def design_space_table() -> list:
    """cost_model.hpp:107-114."""
    return [{"config": "Naive", "sparse_operands": ["Q", "P"], "ideal_prefill": 2.0, "ideal_decode": 1.0},
            {"config": "Trans-K", "sparse_operands": ["K", "P"], "ideal_prefill": 2.0, "ideal_decode": 1.5},
            {"config": "Trans-V", "sparse_operands": ["Q", "V"], "ideal_prefill": 2.0, "ideal_decode": 1.5},
            {"config": "Trans-Both", "sparse_operands": ["K", "V"], "ideal_prefill": 2.0, "ideal_decode": 2.0}]


def cost_report(p: CostParams) -> dict:
    """cost_report + to_json(CostReport) (cost_model.hpp:127-137, report_json.hpp:88-108)."""
    return {"params": {"seq_len": p.seq_len, "hidden_dim": p.hidden_dim, "block_size": p.block_size,
                       "s_key": p.s_key, "s_value": p.s_value},
            "sizes": {k: v for k, v in analytic_sizes(p).items() if k != "total"},
            "r_comp_exact": compression_ratio(p, True), "r_comp_approx": compression_ratio(p, False),
            "speedup_prefill": prefill_speedup(p), "speedup_decode": decode_speedup(p),
            "design_space": design_space_table()}


# -------------------------------------------------------------- run report ---


@dataclass
class RunConfig:
    """pipeline.hpp:22-54 (device kernels: head_dim 128, block_size 64)."""

    seq_len: int = 4096
    head_dim: int = 128
    heads: int = 1
    gqa_group: int = 4
    block_size: int = 64
    s_key_prefill: float = 0.5
    s_value_prefill: float = 0.5
    s_key_decode: float = 0.5
    s_value_decode: float = 0.5
    sink_tokens: int = 0
    local_window: int = 0
    splits: int = 0
    seed: int = 1
    dtype: str = "f16"
    output_path: str = ""

    def validate(self) -> None:
        if self.seq_len <= 0:
            raise ConfigError("RunConfig: seq_len must be positive")
        if self.head_dim != 128 or self.block_size != 64:
            raise ConfigError("RunConfig: the device kernels take head_dim 128 and block_size 64")
        if self.seq_len % self.block_size:
            raise ConfigError("RunConfig: seq_len must be a multiple of block_size on the device path")
        if self.heads <= 0 or self.gqa_group <= 0:
            raise ConfigError("RunConfig: heads and gqa_group must be positive")
        for s in (self.s_key_prefill, self.s_value_prefill, self.s_key_decode, self.s_value_decode):
            if not 0.0 <= s <= 1.0:
                raise ConfigError("RunConfig: sparsities must lie in [0, 1]")
        if self.dtype not in ("f16", "bf16"):
            raise ConfigError("RunConfig: dtype must be f16 or bf16")


def _attention_fp32(q, k, v, causal: bool, scale: float):
    """dense_attention_oracle semantics (attention.hpp:84-115) in fp32 torch."""
    import torch
    s = (q.float() @ k.float().transpose(-1, -2)) * scale
    if causal:
        n_q, n_kv = s.shape[-2], s.shape[-1]
        qpos = torch.arange(n_q, device=s.device)[:, None] + (n_kv - n_q)
        s = s.masked_fill(torch.arange(n_kv, device=s.device)[None, :] > qpos, float("-inf"))
    return torch.softmax(s, dim=-1) @ v.float()


def _acc(got, want) -> dict:
    d = (got.double() - want.double()).abs()
    return {"max_abs": float(d.max()), "mean_abs": float(d.mean())}


def _time(fn, reps: int = 3) -> float:
    import torch
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return sorted(ts)[len(ts) // 2]


def run_pipeline(cfg: RunConfig, accuracy_rows: int = 256) -> dict:
    """pipeline.hpp:137-299 on the device; returns the report dict."""
    import torch
    from . import hierasparse as hs
    cfg.validate()
    dev = torch.device("cuda", torch.cuda.current_device())
    dt = torch.float16 if cfg.dtype == "f16" else torch.bfloat16
    H, G, L, d = cfg.heads, cfg.gqa_group, cfg.seq_len, cfg.head_dim
    g = torch.Generator(device=dev).manual_seed(cfg.seed)
    key = torch.randn((H, L, d), generator=g, device=dev).to(dt)
    val = torch.randn((H, L, d), generator=g, device=dev).to(dt)
    qp = torch.randn((H, G, L, d), generator=g, device=dev).to(dt)
    qd = torch.randn((H, G, d), generator=g, device=dev).to(dt)
    scale = 1.0 / math.sqrt(d)

    def phase(sk, sv):
        c = hs.SparsityConfig(sk, sv, cfg.block_size, cfg.sink_tokens, cfg.local_window)
        ms_c = _time(lambda: hs.prune_cache(key, val, c))
        kc, vc = hs.prune_cache(key, val, c)
        return c, kc, vc, ms_c

    pcfg, kc, vc, ms_compress = phase(cfg.s_key_prefill, cfg.s_value_prefill)
    ms_prefill = _time(lambda: hs.prefill_attention(qp, kc, vc, causal=True, scale=scale), reps=1)
    out_p = hs.prefill_attention(qp, kc, vc, causal=True, scale=scale)
    dcfg = hs.SparsityConfig(cfg.s_key_decode, cfg.s_value_decode, cfg.block_size, cfg.sink_tokens,
                             cfg.local_window)
    kd, vd = hs.recompress_pair(kc, vc, dcfg)
    plan = hs.DecodePlan(qd, kd, vd, scale=scale, splits=cfg.splits)  # graph replay: device time only
    ms_decode = _time(plan, reps=5)
    out_d = hs.decode_attention(qd, kd, vd, scale=scale, splits=cfg.splits)
    # dense baselines (S = 0) of the same shapes, for the measured speedups
    _, k0, v0, _ = phase(0.0, 0.0)
    ms_prefill_dense = _time(lambda: hs.prefill_attention(qp, k0, v0, causal=True, scale=scale), reps=1)
    plan0 = hs.DecodePlan(qd, k0, v0, scale=scale, splits=cfg.splits)
    ms_decode_dense = _time(plan0, reps=5)
    del k0, v0, plan0

    # accuracy on the last `accuracy_rows` prefill rows and every decode row
    kdec, vdec = hs.decompress(kc), hs.decompress(vc)
    kdd, vdd = hs.decompress(kd), hs.decompress(vd)
    rows = min(accuracy_rows, L)
    acc = {"prefill_vs_decompressed": {"max_abs": 0.0, "mean_abs": 0.0},
           "prefill_vs_raw": {"max_abs": 0.0, "mean_abs": 0.0},
           "decode_vs_decompressed": {"max_abs": 0.0, "mean_abs": 0.0},
           "decode_vs_raw": {"max_abs": 0.0, "mean_abs": 0.0}}

    def merge(name, a):
        acc[name]["max_abs"] = max(acc[name]["max_abs"], a["max_abs"])
        acc[name]["mean_abs"] += a["mean_abs"] / H

    for h in range(H):
        qr = qp[h, :, L - rows:]
        merge("prefill_vs_decompressed", _acc(out_p[h, :, L - rows:], _attention_fp32(qr, kdec[h], vdec[h], True,
                                                                                        scale)))
        merge("prefill_vs_raw", _acc(out_p[h, :, L - rows:], _attention_fp32(qr, key[h], val[h], True, scale)))
        merge("decode_vs_decompressed", _acc(out_d[h], _attention_fp32(qd[h], kdd[h], vdd[h], False, scale)))
        merge("decode_vs_raw", _acc(out_d[h], _attention_fp32(qd[h], key[h], val[h], False, scale)))

    sizes = {k: 0 for k in ("size_idx", "size_den", "size_nnz", "size_e")}
    for c in (kc, vc):
        for k, v in c.measure_size().items():
            sizes[k] += v * H
    baseline = 2 * L * d * 2 * H
    measured_total = sum(sizes.values())
    fp, bp = 0, 0
    fd, bd = 0, 0
    for u in range(H):
        f, b = hs.flop_and_byte_count(L, kc, vc, 0, True, unit=u)
        fp, bp = fp + f * G, bp + b * G
        f, b = hs.flop_and_byte_count(G, kd, vd, 0, False, unit=u)
        fd, bd = fd + f, bd + b
    cp_pre = CostParams(L, d, cfg.block_size, cfg.s_key_prefill, cfg.s_value_prefill)
    cp_dec = CostParams(L, d, cfg.block_size, cfg.s_key_decode, cfg.s_value_decode)
    try:
        root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
        with open(os.path.join(root, "MEASURED_PEAKS.json")) as f:
            peaks = json.load(f)
        hbm, tf = float(peaks["hbm_gbs"]), float(peaks["bf16_tflops"])
    except (OSError, KeyError, ValueError):
        hbm, tf = 6650.0, 1590.0  # B200_PROFILING.md fallback
    report = {
        "schema_version": 1,
        "config": asdict(cfg),
        "compression": {"measured_sizes": sizes, "dense_baseline_bytes": baseline,
                        "r_comp_measured": baseline / measured_total,
                        "r_comp_model_exact": compression_ratio(cp_pre, True),
                        "r_comp_model_approx": compression_ratio(cp_pre, False)},
        "accuracy": acc,
        "counts": {"prefill": {"flops": fp, "bytes_moved": bp}, "decode": {"flops": fd, "bytes_moved": bd},
                   "model_speedup_prefill": prefill_speedup(cp_pre),
                   "model_speedup_decode": decode_speedup(cp_dec)},
        "b200": {
            "compress_ms": ms_compress, "prefill_ms": ms_prefill, "decode_ms": ms_decode,
            "prefill_counted_tflops": fp / (ms_prefill * 1e-3) / 1e12,
            "prefill_frac_of_dense_peak": fp / (ms_prefill * 1e-3) / 1e12 / tf,
            "decode_gbs": bd / (ms_decode * 1e-3) / 1e9,
            "decode_frac_of_hbm": bd / (ms_decode * 1e-3) / 1e9 / hbm,
            "measured_speedup_prefill": ms_prefill_dense / ms_prefill,
            "measured_speedup_decode": ms_decode_dense / ms_decode,
            "peaks": {"hbm_gbs": hbm, "dense_tflops": tf},
        },
    }
    if cfg.output_path:
        try:
            with open(cfg.output_path, "w") as f:
                json.dump(report, f, indent=2)
        except OSError as e:
            raise IoError(f"cannot write '{cfg.output_path}': {e}") from e
    return report


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="hierasparse-b200", description=__doc__.split("\n\n")[0])
    sub = ap.add_subparsers(dest="cmd", required=True)
    c = sub.add_parser("cost", help="closed-form cost report (cost_model.hpp)")
    c.add_argument("--seq-len", type=int, default=4096)
    c.add_argument("--hidden-dim", type=int, default=128)
    c.add_argument("--block-size", type=int, default=64)
    c.add_argument("--s-key", type=float, default=0.5)
    c.add_argument("--s-value", type=float, default=0.5)
    r = sub.add_parser("run", help="device pipeline report (pipeline.hpp)")
    for name, typ, dflt in (("seq-len", int, 4096), ("heads", int, 1), ("gqa", int, 4), ("s-key-prefill", float, .5),
                            ("s-value-prefill", float, .5), ("s-key-decode", float, .5),
                            ("s-value-decode", float, .5), ("sink", int, 0), ("window", int, 0), ("splits", int, 0),
                            ("seed", int, 1), ("dtype", str, "f16"), ("out", str, "")):
        r.add_argument("--" + name, type=typ, default=dflt)
    a = ap.parse_args(argv)
    try:
        if a.cmd == "cost":
            print(json.dumps(cost_report(CostParams(a.seq_len, a.hidden_dim, a.block_size, a.s_key, a.s_value)),
                             indent=2))
        else:
            cfg = RunConfig(seq_len=a.seq_len, heads=a.heads, gqa_group=a.gqa, s_key_prefill=a.s_key_prefill,
                            s_value_prefill=a.s_value_prefill, s_key_decode=a.s_key_decode,
                            s_value_decode=a.s_value_decode, sink_tokens=a.sink, local_window=a.window,
                            splits=a.splits, seed=a.seed, dtype=a.dtype, output_path=a.out)
            print(json.dumps(run_pipeline(cfg), indent=2))
    except ConfigError as e:
        print(f"config error: {e}", file=sys.stderr)
        return 2
    except IoError as e:
        print(f"io error: {e}", file=sys.stderr)
        return 3
    except DataError as e:
        print(f"data error: {e}", file=sys.stderr)
        return 4
    return 0


if __name__ == "__main__":
    sys.exit(main())
