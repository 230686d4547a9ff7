"""Where does DecodePlan(host_io)'s extra time go?  configs[1] decode through
decode_attention with q / out on the device or in pinned host memory (the four
combinations), bench protocol (L2 flushed, stream held while the host enqueues).
    python tools/decode_hostio_ab.py [reps]"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
from paper_2604_16864_b200 import hierasparse as hs

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
dev = torch.device("cuda", 0)
scale = 1.0 / 128 ** 0.5
kc, vc, q, _ = bench.build_headline(hs, dev, 0, scale)
flush = bench.Flusher(dev)
qh = q.cpu().pin_memory()
od = torch.empty(8, 4, 128, device=dev)
oh = torch.empty(8, 4, 128).pin_memory()
variants = {"q dev / out dev": (q, od), "q host / out dev": (qh, od), "q dev / out host": (q, oh),
            "q host / out host": (qh, oh)}


def run(qq, oo, steps=40):
    st = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    sp = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    torch.cuda.synchronize()
    torch.cuda._sleep(int(1.965e9 * 0.03))
    for i in range(steps):
        flush()
        st[i].record()
        hs.decode_attention(qq, kc, vc, scale=scale, out=oo)
        sp[i].record()
    torch.cuda.synchronize()
    return statistics.median([a.elapsed_time(b) * 1e3 for a, b in zip(st, sp)])


for name, (qq, oo) in variants.items():
    run(qq, oo, 5)
for r in range(reps):
    print(" | ".join(f"{name}: {run(qq, oo):.2f}" for name, (qq, oo) in variants.items()), flush=True)
