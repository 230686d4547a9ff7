import os, sys, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2604_16864_b200 import hierasparse as hs
L = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
s = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
torch.manual_seed(0)
k = torch.randn(8, L, 128, device="cuda").half(); v = torch.randn(8, L, 128, device="cuda").half()
kc, vc = hs.prune_cache(k, v, hs.SparsityConfig(s, s, 64))
q = torch.randn(8, 4, L, 128, device="cuda").half()
hs.prefill_attention(q, kc, vc, causal=True); torch.cuda.synchronize()
os.environ["HS_PREFILL_TRACE"] = "/tmp/trace.bin"
hs.prefill_attention(q, kc, vc, causal=True); torch.cuda.synchronize()
tr = np.fromfile("/tmp/trace.bin", dtype=np.int64).reshape(4096, 8)
n = int((tr[:, 0] > 0).sum())
t0 = tr[0, 0]
d = tr[:n] - t0
print("tiles", n, "total cycles", tr[n - 1, 3] - t0, "per tile", (tr[n - 1, 3] - tr[n // 2, 3]) / (n - 1 - n // 2))
names = ["sfull_ok", "pass1_done", "pempty_ok", "pass2_done", "mma_g1_issue", "mma_pfull_ok", "mma_g2_issued"]
for t in list(range(3)) + list(range(n // 2, n // 2 + 6)):
    print(t, " ".join(f"{names[e]}={d[t, e]}" for e in range(7)))
st = tr[n // 4: 3 * n // 4]
print("median durations (cycles):")
print(" pass1 (sfull->bar2):", np.median(st[:, 1] - st[:, 0]))
print(" wait pempty:", np.median(st[:, 2] - st[:, 1]))
print(" pass2:", np.median(st[:, 3] - st[:, 2]))
print(" sfull(t+1) after pass2(t):", np.median(tr[n // 4 + 1: 3 * n // 4 + 1, 0] - st[:, 3]))
print(" pfull->g2 issued:", np.median(st[:, 6] - st[:, 5]))
print(" g2 issued -> pempty_ok(t+1):", np.median(tr[n // 4 + 1: 3 * n // 4 + 1, 2] - st[:, 6]))
print(" pass2_done(t) -> mma pfull_ok(t):", np.median(st[:, 5] - st[:, 3]))
print(" g1 issue(t+1) - pfull? :", np.median(tr[n // 4 + 1: 3 * n // 4 + 1, 4] - st[:, 5]))
