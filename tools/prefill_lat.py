"""Per-tile cost of the prefill pipeline with few CTAs (latency) vs a full grid
(bandwidth): one KV head, `ctas` query tiles of 128 at the end of an L-token
causal sequence, so each CTA walks ~L/128 key tiles.  Honours HS_PREFILL_MODE."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2604_16864_b200 import hierasparse as hs
L = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
s = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
ctas = int(sys.argv[3]) if len(sys.argv) > 3 else 1
U, G = 1, 1
torch.manual_seed(0)
k = torch.randn(U, L, 128, device="cuda").half(); v = torch.randn(U, L, 128, device="cuda").half()
kc, vc = hs.prune_cache(k, v, hs.SparsityConfig(s, s, 64))
nq = 128 * ctas
q = torch.randn(U, G, nq, 128, device="cuda").half()
out = torch.empty(U, G, nq, 128, device="cuda")
for _ in range(3):
    hs.prefill_attention(q, kc, vc, causal=True, out=out)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record(); hs.prefill_attention(q, kc, vc, causal=True, out=out); e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
tiles = L // 128  # per CTA (roughly: all blocks visible)
print(f"L={L} s={s} ctas={ctas} mode={os.environ.get('HS_PREFILL_MODE', '0')}: {ms * 1e3:.1f} us, "
      f"{ms * 1e-3 * 1.9e9 / tiles:.0f} cycles/tile @1.9GHz")
