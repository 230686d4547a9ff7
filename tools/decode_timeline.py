"""Per-CTA timeline of one configs[1] decode step (HS_DECODE_TIMES): start,
first data, loop end, exit (ns, relative to the earliest start)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2604_16864_b200 import hierasparse as hs
U, L, GQA, D = 8, 131072, 4, 128
torch.manual_seed(0)
key = torch.randn(U, L, D, device="cuda").bfloat16(); val = torch.randn(U, L, D, device="cuda").bfloat16()
kc, vc = hs.prune_cache(key, val, hs.SparsityConfig(1, 1, 64)); del key, val
q = torch.randn(U, GQA, D, device="cuda").bfloat16()
out = torch.empty(U, GQA, D, device="cuda")
flush = torch.ones(64 * 1024 * 1024, device="cuda"); sink = torch.empty((), device="cuda")
for _ in range(5):
    hs.decode_attention(q, kc, vc, out=out)
torch.cuda.synchronize()
torch.sum(flush, dim=0, out=sink)
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record(); hs.decode_attention(q, kc, vc, out=out); e1.record(); torch.cuda.synchronize()
print(f"event-timed step after flush: {e0.elapsed_time(e1) * 1e3:.1f} us")
e0.record(); hs.decode_attention(q, kc, vc, out=out); e1.record(); torch.cuda.synchronize()
print(f"event-timed step, L2 warm: {e0.elapsed_time(e1) * 1e3:.1f} us")
e0.record()
for _ in range(20):
    hs.decode_attention(q, kc, vc, out=out)
e1.record(); torch.cuda.synchronize()
print(f"20 back-to-back steps: {e0.elapsed_time(e1) * 1e3 / 20:.1f} us each")
plan = hs.DecodePlan(q, kc, vc)
ts = []
for _ in range(20):
    torch.sum(flush, dim=0, out=sink)
    e0.record(); plan(); e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1) * 1e3)
print(f"graph replay after flush (bench protocol): median {np.median(ts):.1f} us")
e0.record()
for _ in range(20):
    plan()
e1.record(); torch.cuda.synchronize()
print(f"graph replay back-to-back: {e0.elapsed_time(e1) * 1e3 / 20:.1f} us each")
if not os.environ.get("TL_NOFLUSH"):  # TL_NOFLUSH=1: the timed launch follows another decode (warm L2)
    torch.sum(flush, dim=0, out=sink)
else:
    hs.decode_attention(q, kc, vc, out=out)
os.environ["HS_DECODE_TIMES"] = "/tmp/dtimes.bin"
hs.decode_attention(q, kc, vc, out=out)
torch.cuda.synchronize()
t = np.fromfile("/tmp/dtimes.bin", dtype=np.int64).reshape(-1, 16).astype(np.float64)
t0 = t[:, 0].min()
t = np.where(t > 0, t - t0, np.nan)
t /= 1000.0  # us
print(f"CTAs {len(t)}  start: min {t[:,0].min():.1f} max {t[:,0].max():.1f} us | first data: min {t[:,1].min():.1f} "
      f"med {np.median(t[:,1]):.1f} max {t[:,1].max():.1f} | loop end: min {t[:,2].min():.1f} med {np.median(t[:,2]):.1f} "
      f"max {t[:,2].max():.1f} | partial written: max {np.nanmax(t[:,3]):.1f} | combine done: max {np.nanmax(t[:,4]):.1f} us")
print("loop-end percentiles (10/25/50/75/90/100):", np.percentile(t[:, 2], [10, 25, 50, 75, 90, 100]).round(1))
nsp = len(t) // U
for u in range(U):
    tu = t[u * nsp:(u + 1) * nsp]
    print(f"unit {u}: first data max {np.nanmax(tu[:, 1]):.1f} | loop end min {np.nanmin(tu[:, 2]):.1f} med {np.nanmedian(tu[:, 2]):.1f} "
          f"max {np.nanmax(tu[:, 2]):.1f} | partial max {np.nanmax(tu[:, 3]):.1f} | done max {np.nanmax(tu[:, 4]):.1f}")
last = ~np.isnan(t[:, 4])
for row in t[last][:12]:
    print(f"combine CTA: loop end {row[2]:.1f} partial {row[3]:.1f} fence1 {row[7]:.1f} ticket {row[5]:.1f} "
          f"O summed {row[10]:.1f} done {row[4]:.1f}")
