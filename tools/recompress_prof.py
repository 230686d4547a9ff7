"""Decode-phase re-prune timing: fused hs_recompress vs decompress + prune_compress
(configs[1] caches: 8 KV heads x 128K x 128 bf16, prefill S = 0.5 -> decode S = 1)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2604_16864_b200 import hierasparse as hs
U, L = 8, 131072
g = torch.Generator(device="cuda").manual_seed(0)
key = torch.randn((U, L, 128), generator=g, device="cuda").to(torch.bfloat16)
val = torch.randn((U, L, 128), generator=g, device="cuda").to(torch.bfloat16)
kp, vp = hs.prune_cache(key, val, hs.SparsityConfig(0.5, 0.5, 64))
del key, val
dec = hs.SparsityConfig(1.0, 1.0, 64)
def run(fn):
    best = 1e9
    for _ in range(5):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(); a = fn(kp, dec, 1.0); b = fn(vp, dec, 1.0); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best, a, b
tf, a, b = run(hs.recompress)
tu, a2, b2 = run(hs.recompress_unfused)
same = all(torch.equal(getattr(x, n).view(torch.int16) if getattr(x, n).is_floating_point() else getattr(x, n),
                       getattr(y, n).view(torch.int16) if getattr(y, n).is_floating_point() else getattr(y, n))
           for x, y in ((a, a2), (b, b2)) for n in ("index_map", "nnz_pool", "meta_pool", "dense_pool"))
byts = kp.nbytes() + vp.nbytes() + a.nbytes() + b.nbytes()
print(f"fused {tf:.3f} ms ({byts / tf / 1e6:.0f} GB/s)  unfused {tu:.3f} ms  identical={same}")
