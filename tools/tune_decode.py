"""Decode kernel tuning sweep on configs[1] (8 KV heads x 128K, GQA 4, S=1).
Prints µs and GB/s per (warps, ctas/SM, slots/warp, splits) variant."""
import math
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_16864_b200 import hierasparse as hs  # noqa: E402

U, L, GQA, D = 8, 131072, 4, 128
dtype = torch.bfloat16 if "--f16" not in sys.argv else torch.float16
torch.manual_seed(0)
key = torch.randn(U, L, D, device="cuda").to(dtype)
val = torch.randn(U, L, D, device="cuda").to(dtype)
q = torch.randn(U, GQA, D, device="cuda").to(dtype)
kc, vc = hs.prune_cache(key, val, hs.SparsityConfig(1, 1, 64))
del key, val
nbytes = U * hs.flop_and_byte_count(GQA, kc, vc)[1]
out = torch.empty(U, GQA, D, device="cuda")
flush = torch.ones(64 * 1024 * 1024, device="cuda"); _sink = torch.empty(1, device="cuda")
def flush_l2():
    torch.sum(flush, dim=0, out=_sink)
ref = hs.decode_attention(q, kc, vc, out=torch.empty_like(out)).clone()


def run(splits=0, it=30):
    for _ in range(5):
        hs.decode_attention(q, kc, vc, splits=splits, out=out)
    ts = []
    for _ in range(it):
        flush_l2()
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record()
        hs.decode_attention(q, kc, vc, splits=splits, out=out)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    err = (out - ref).abs().max().item()
    return statistics.median(ts), err


variants = [(8, 1, 1), (4, 1, 2), (4, 2, 1), (4, 1, 3)]
for pf in (0, 1, 2, 3, 4, 6, 8):
    os.environ["HS_DECODE_PF"] = str(pf)
    us, err = run()
    print(f"default pf={pf}: {us:8.2f} us  {nbytes / us / 1e3:8.1f} GB/s  err={err:.2e}", flush=True)
os.environ.pop("HS_DECODE_PF")
for w, c, s in variants:
    os.environ["HS_DECODE_WARPS"] = str(w)
    os.environ["HS_DECODE_CTAS_PER_SM"] = str(c)
    os.environ["HS_DECODE_SPW"] = str(s)
    try:
        us, err = run()
        print(f"warps={w} ctas/sm={c} spw={s}: {us:8.2f} us  {nbytes / us / 1e3:8.1f} GB/s  err={err:.2e}", flush=True)
    except Exception as e:  # noqa: BLE001
        print(f"warps={w} ctas/sm={c} spw={s}: failed {e}", flush=True)
for k in ("HS_DECODE_WARPS", "HS_DECODE_CTAS_PER_SM", "HS_DECODE_SPW"):
    os.environ.pop(k, None)
for splits in (9, 18, 19, 36, 37, 74):
    us, err = run(splits)
    print(f"default splits={splits}: {us:8.2f} us  {nbytes / us / 1e3:8.1f} GB/s", flush=True)
