"""Per-launch SM placement of the decode grid vs its duration (HS_DECODE_TIMES
dumps; tools): is the step-time bimodality a placement effect?
    python tools/decode_placement.py [launches]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench
from paper_2604_16864_b200 import hierasparse as hs

n = int(sys.argv[1]) if len(sys.argv) > 1 else 40
dev = torch.device("cuda", 0)
scale = 1.0 / 128 ** 0.5
kc, vc, q, _ = bench.build_headline(hs, dev, 0, scale)
flush = bench.Flusher(dev)
out = torch.empty(8, 4, 128, device=dev)
for _ in range(3):
    hs.decode_attention(q, kc, vc, scale=scale, out=out)
os.environ["HS_DECODE_TIMES"] = "/tmp/dp.bin"
rows = []
for i in range(n):
    flush()
    hs.decode_attention(q, kc, vc, scale=scale, out=out)
    torch.cuda.synchronize()
    t = np.fromfile("/tmp/dp.bin", dtype=np.int64).reshape(-1, 16)
    start = t[:, 0].min()
    dur = (t[:, 4].max() - start) / 1e3
    loop_end = (np.median(t[:, 2]) - start) / 1e3
    sms = set(int(x) for x in t[:, 15])
    idle = sorted(set(range(148)) - sms)
    first = (np.median(t[:, 1]) - start) / 1e3
    rows.append((dur, loop_end, first, idle))
    print(f"launch {i}: kernel {dur:.2f} us, first data med {first:.2f}, loop end med {loop_end:.2f}, idle SMs {idle}",
          flush=True)
d = np.array([r[0] for r in rows])
print(f"kernel span: median {np.median(d):.2f} min {d.min():.2f} max {d.max():.2f}")
