"""Compression timing on configs[1] caches (8 KV heads x 128K x 128 bf16):
prune_cache at S = 1 (static, one pass) and S = 0.5 (loss-driven), plus the
decode-phase recompress 0.5 -> 1.  GB/s = dense read + pools written."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2604_16864_b200 import hierasparse as hs
U, L = 8, 131072
g = torch.Generator(device="cuda").manual_seed(0)
key = torch.randn((U, L, 128), generator=g, device="cuda").to(torch.bfloat16)
val = torch.randn((U, L, 128), generator=g, device="cuda").to(torch.bfloat16)
def best(fn, n=5):
    t = 1e9
    for _ in range(n):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(); r = fn(); e1.record(); torch.cuda.synchronize()
        t = min(t, e0.elapsed_time(e1))
    return t, r
for s in (1.0, 0.5):
    t, (kc, vc) = best(lambda: hs.prune_cache(key, val, hs.SparsityConfig(s, s, 64)))
    byts = 2 * key.numel() * 2 + kc.nbytes() + vc.nbytes()
    print(f"prune_cache S={s}: {t:.3f} ms  {byts / t / 1e6:.0f} GB/s")
kp, vp = hs.prune_cache(key, val, hs.SparsityConfig(0.5, 0.5, 64))
dec = hs.SparsityConfig(1.0, 1.0, 64)
t, (a, b) = best(lambda: (hs.recompress(kp, dec, 1.0), hs.recompress(vp, dec, 1.0)))
print(f"recompress 0.5->1: {t:.3f} ms  {(kp.nbytes() + vp.nbytes() + a.nbytes() + b.nbytes()) / t / 1e6:.0f} GB/s")
