"""Per-tile event clocks of CTA (0,0,0) (the heaviest causal tile, launched first)
while the whole grid runs: 8 kv heads x GQA 4, causal, fp16 (HS_PREFILL_TRACE,
tools-only instrumented build).  Events as in tools/prefill_trace.py:
0 softmax got S(t); 1 after the max check; 2 P buffer free; 3 P(t) stored;
4 GEMM1(t) passed its waits; 5 GEMM2 warp got pfull(t); 6 GEMM2(t) issued;
7 K(t) issue passed kempty; 10 GEMM1 got K(t); 11 GEMM1 warp top of tile."""
import os, sys, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2604_16864_b200 import hierasparse as hs
L = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
s = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
U, G = 8, 4
torch.manual_seed(0)
k = torch.randn(U, L, 128, device="cuda").half(); v = torch.randn(U, L, 128, device="cuda").half()
kc, vc = hs.prune_cache(k, v, hs.SparsityConfig(s, s, 64))
q = torch.randn(U, G, L, 128, device="cuda").half()
out = torch.empty(U, G, L, 128, device="cuda")
hs.prefill_attention(q, kc, vc, causal=True, out=out); torch.cuda.synchronize()
os.environ["HS_PREFILL_TRACE"] = "/tmp/trace.bin"
hs.prefill_attention(q, kc, vc, causal=True, out=out); torch.cuda.synchronize()
tr = np.fromfile("/tmp/trace.bin", dtype=np.int64).reshape(4096, 16)
n = int((tr[:, 4] > 0).sum())
st, nx = slice(n // 4, 3 * n // 4), slice(n // 4 + 1, 3 * n // 4 + 1)
med = lambda a: float(np.median(a))
print(f"L={L} s={s} mode={os.environ.get('HS_PREFILL_MODE', '0')} tiles {n} per tile "
      f"{(tr[3 * n // 4, 4] - tr[n // 4, 4]) / (n // 2):.0f} cycles")
print("  GEMM1 issue period %.0f | S seen by softmax after GEMM1 issue %.0f | GEMM2 got pfull after P stored %.0f"
      " | GEMM2 issue took %.0f | GEMM1 waited for K %.0f | GEMM1 waited for S buffer %.0f"
      % (med(tr[nx, 4] - tr[st, 4]), med(tr[st, 0] - tr[st, 4]), med(tr[st, 5] - tr[st, 3]), med(tr[st, 6] - tr[st, 5]),
         med(tr[st, 10] - tr[st, 11]), med(tr[st, 4] - tr[st, 10])))
if tr[st, 3].min() > 0:
    print("  softmax: got S -> checked %.0f | -> P buffer free %.0f | -> P stored %.0f | -> next S %.0f"
          % (med(tr[st, 1] - tr[st, 0]), med(tr[st, 2] - tr[st, 1]), med(tr[st, 3] - tr[st, 2]),
             med(tr[nx, 0] - tr[st, 3])))
    print("  check: TMEM load %.0f | scale+mask+max %.0f | bar.red.or %.0f | to S release %.0f"
          % (med(tr[st, 12] - tr[st, 0]), med(tr[st, 13] - tr[st, 12]), med(tr[st, 14] - tr[st, 13]),
             med(tr[st, 1] - tr[st, 14])))
    print("  warpgroup 2 got S(t) after warpgroup 0 by %.0f cycles (median; p10 %.0f, p90 %.0f)"
          % (med(tr[st, 15] - tr[st, 0]), np.percentile(tr[st, 15] - tr[st, 0], 10),
             np.percentile(tr[st, 15] - tr[st, 0], 90)))
