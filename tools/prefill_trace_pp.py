"""Per-tile event clocks of CTA (0,0,0) of the ping-pong prefill (HS_PREFILL_TRACE,
DBG instantiation), the heaviest causal query tile.  Softmax events per tile t
(group t % 2): 0 S(t) full; 1 TMEM loaded; 2 logit check done; 3 P^T buffer free;
12 exponentials + P^T stored; 13 previous tile's record seen; 14 P^T(t) released.
MMA warps: 11 loop top, 10 K(t) landed, 4 GEMM1(t) issued, 5 GEMM2(t) inputs ready,
6 GEMM2(t) issued, 7 K(t) TMA issued (producer).
    python tools/prefill_trace_pp.py [L] [S] [units] [gqa]"""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2604_16864_b200 import hierasparse as hs
L = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
s = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
U = int(sys.argv[3]) if len(sys.argv) > 3 else 8
G = int(sys.argv[4]) if len(sys.argv) > 4 else 4
torch.manual_seed(0)
k = torch.randn(U, L, 128, device="cuda").half(); v = torch.randn(U, L, 128, device="cuda").half()
kc, vc = hs.prune_cache(k, v, hs.SparsityConfig(s, s, 64))
q = torch.randn(U, G, L, 128, device="cuda").half()
out = torch.empty(U, G, L, 128, device="cuda")
hs.prefill_attention(q, kc, vc, causal=True, out=out); torch.cuda.synchronize()
os.environ["HS_PREFILL_TRACE"] = "/tmp/trace_pp.bin"
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record(); hs.prefill_attention(q, kc, vc, causal=True, out=out); e1.record(); torch.cuda.synchronize()
del os.environ["HS_PREFILL_TRACE"]
tr = np.fromfile("/tmp/trace_pp.bin", dtype=np.int64).reshape(4096, 16)
n = int((tr[:, 4] > 0).sum())
print(f"L={L} s={s} U={U} G={G}: traced launch {e0.elapsed_time(e1):.3f} ms, CTA(0,0,0) tiles {n}, "
      f"per tile {(tr[n - 2, 4] - tr[n // 4, 4]) / (n - 2 - n // 4):.0f} cycles")
st = np.arange(n // 4, 3 * n // 4)
med = lambda a: float(np.median(a))
def gap(a, b, dt=0):
    return med(tr[st + dt, b] - tr[st, a])
print("softmax (per tile, cycles): LDTM e1-e0 %.0f | check e2-e1 %.0f | pempty wait e3-e2 %.0f | exps+STS e12-e3 %.0f"
      " | record wait e13-e12 %.0f | release e14-e13 %.0f | group idle e0(t+2)-e14(t) %.0f"
      % (gap(0, 1), gap(1, 2), gap(2, 3), gap(3, 12), gap(12, 13), gap(13, 14), med(tr[st + 2, 0] - tr[st, 14])))
print("group chain e0(t+2)-e0(t) %.0f | other group's start e0(t+1)-e0(t) %.0f"
      % (med(tr[st + 2, 0] - tr[st, 0]), med(tr[st + 1, 0] - tr[st, 0])))
print("MMA: GEMM1 issue->S full e0-e4 %.0f | check(t)->GEMM1(t+2) issue e4(t+2)-e2(t) %.0f | "
      "P^T released->GEMM2 issue e6-e14 %.0f | GEMM2(t) issue->P^T(t+2) buffer free seen e3(t+2)-e6(t) %.0f"
      % (gap(4, 0), med(tr[st + 2, 4] - tr[st, 2]), gap(14, 6), med(tr[st + 2, 3] - tr[st, 6])))
print("K: K(t) TMA issue -> landed e10-e7 %.0f | MMA top->K landed wait e10-e11 %.0f"
      % (gap(7, 10), gap(11, 10)))
print("median event offsets from e0(t):", " ".join(f"e{e}={med(tr[st, e] - tr[st, 0]):+.0f}" for e in (11, 7, 10, 4, 0, 1, 2, 13, 12, 3, 14, 5, 6)))
for t in (n // 2, n // 2 + 1, n // 2 + 2, n // 2 + 3):
    b = tr[t, 0]
    print(t, " ".join(f"e{e}={tr[t, e] - b:+d}" for e in (11, 7, 10, 4, 0, 1, 2, 3, 12, 13, 14, 5, 6) if tr[t, e] > 0))
