"""Per-tile event clocks of CTA (0,0,0) (HS_PREFILL_TRACE), median per-tile gaps.
Events: 0 softmax got S(t); 1 after the max check; 2 P buffer free; 3 P(t) stored;
4 MMA warp passed full/meta/sempty for GEMM1(t); 5 MMA warp got pfull(t);
6 GEMM2(t) issued."""
import os, sys, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2604_16864_b200 import hierasparse as hs
L = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
s = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
torch.manual_seed(0)
k = torch.randn(1, L, 128, device="cuda").half(); v = torch.randn(1, L, 128, device="cuda").half()
kc, vc = hs.prune_cache(k, v, hs.SparsityConfig(s, s, 64))
q = torch.randn(1, 1, 128, 128, device="cuda").half()
hs.prefill_attention(q, kc, vc, causal=True); torch.cuda.synchronize()
os.environ["HS_PREFILL_TRACE"] = "/tmp/trace.bin"
hs.prefill_attention(q, kc, vc, causal=True); torch.cuda.synchronize()
tr = np.fromfile("/tmp/trace.bin", dtype=np.int64).reshape(4096, 16)
n = int((tr[:, 4] > 0).sum())
t0 = tr[0, 4]
d = np.where(tr[:n] > 0, tr[:n] - t0, -1)
print(f"L={L} s={s} mode={os.environ.get('HS_PREFILL_MODE', '0')} tiles {n} cycles {tr[n - 1, 6] - t0} "
      f"per tile {(tr[n - 1, 4] - tr[n // 2, 4]) / (n - 1 - n // 2):.0f}")
for t in list(range(3)) + list(range(n // 2, n // 2 + 4)):
    print(t, " ".join(f"e{e}={d[t, e]}" for e in range(13)))
st = slice(n // 4, 3 * n // 4)
nx = slice(n // 4 + 1, 3 * n // 4 + 1)
med = lambda a: float(np.median(a))
print("median gaps (cycles): e4(t+1)-e4(t) %.0f | e0-e4 (sfull seen after g1 issue) %.0f | e5-e4 %.0f | e6-e5 %.0f | e4(t+1)-e6(t) %.0f"
      % (med(tr[nx, 4] - tr[st, 4]), med(tr[st, 0] - tr[st, 4]), med(tr[st, 5] - tr[st, 4]), med(tr[st, 6] - tr[st, 5]),
         med(tr[nx, 4] - tr[st, 6])))
if tr[st, 3].min() > 0:
    print("softmax: e1-e0 %.0f | e2-e1 %.0f | e3-e2 %.0f | e0(t+1)-e3(t) %.0f | e5(t)-e3(t) %.0f"
          % (med(tr[st, 1] - tr[st, 0]), med(tr[st, 2] - tr[st, 1]), med(tr[st, 3] - tr[st, 2]),
             med(tr[nx, 0] - tr[st, 3]), med(tr[st, 5] - tr[st, 3])))
print("K producer: issue period e7 %.0f | meta start after issue e9-e7 %.0f | kfull wait e12-e9 %.0f | permute e8-e12 %.0f"
      " | MMA kmeta wait e10-e11 %.0f | sempty wait e4-e10 %.0f"
      % (med(tr[nx, 7] - tr[st, 7]), med(tr[st, 9] - tr[st, 7]), med(tr[st, 12] - tr[st, 9]), med(tr[st, 8] - tr[st, 12]),
         med(tr[st, 10] - tr[st, 11]), med(tr[st, 4] - tr[st, 10])))
