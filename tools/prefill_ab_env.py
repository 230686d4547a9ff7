"""A/B of prefill run-time switches (environment variables read per call) in one process.

    python tools/prefill_ab_env.py L "S1,S2,..." "VAR=a;VAR2=c|VAR=b|..." [reps]

AB_SLEEP=<s>: idle that long before every timed run (equal power state; with it the
runs repeat to ~0.3%, without it the 1000 W cap moves them by up to 10%).

Caches per S are built once; the variants alternate within each repetition so
clock drift cancels.  configs[2] shape: 8 KV heads x GQA 4, causal, fp16.
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2604_16864_b200 import hierasparse as hs

L = int(sys.argv[1])
spars = [float(x) for x in sys.argv[2].split(",")]
variants = sys.argv[3].split("|")
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
dtype = torch.bfloat16 if os.environ.get("AB_BF16") else torch.half
U, G = 8, 4
torch.manual_seed(0)
q = torch.randn(U, G, L, 128, device="cuda").to(dtype)
out = torch.empty(U, G, L, 128, device="cuda")
ref = torch.empty_like(out)


def set_env(v):
    for kv in v.split(";"):
        if not kv:
            continue
        k, val = kv.split("=")
        if val == "":
            os.environ.pop(k, None)
        else:
            os.environ[k] = val


def clear(vs):
    for v in vs:
        for kv in v.split(";"):
            if kv:
                os.environ.pop(kv.split("=")[0], None)


for s in spars:
    k = torch.randn(U, L, 128, device="cuda").to(dtype)
    v = torch.randn(U, L, 128, device="cuda").to(dtype)
    kc, vc = hs.prune_cache(k, v, hs.SparsityConfig(s, s, 64))
    del k, v
    fl = sum(hs.flop_and_byte_count(L, kc, vc, 0, True, unit=u)[0] for u in range(U)) * G
    res = {vv: [] for vv in variants}
    for vv in variants:  # warm-up + agreement with the first variant
        clear(variants)
        set_env(vv)
        hs.prefill_attention(q, kc, vc, causal=True, out=out)
        torch.cuda.synchronize()
        if vv == variants[0]:
            ref.copy_(out)
        else:
            d = (out - ref).abs().max().item()
            print(f"  S={s} {vv}: max |diff| vs {variants[0]} = {d:.3e}", flush=True)
    for _ in range(reps):
        for vv in variants:
            clear(variants)
            set_env(vv)
            if os.environ.get("AB_SLEEP"):  # equal power / thermal state before every timed run
                time.sleep(float(os.environ["AB_SLEEP"]))
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record()
            hs.prefill_attention(q, kc, vc, causal=True, out=out)
            e1.record()
            torch.cuda.synchronize()
            res[vv].append(e0.elapsed_time(e1))
    for vv in variants:
        ms = min(res[vv])
        print(f"L={L} S={s} [{vv}]: best {ms:.3f} ms ({fl / ms / 1e9:.1f} counted TFLOPS), all "
              + " ".join(f"{x:.2f}" for x in res[vv]), flush=True)
    del kc, vc
    torch.cuda.empty_cache()
clear(variants)
