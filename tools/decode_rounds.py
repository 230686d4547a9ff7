"""Per-round distribution of the configs[1] graph-replay step (bench protocol) with
clocks/power sampled after each round: looks for bimodal step times.
    python tools/decode_rounds.py [rounds]"""
import os, sys, statistics, subprocess, torch
sys.path.insert(0, os.getcwd())
import bench
from paper_2604_16864_b200 import hierasparse as hs
dev = torch.device("cuda", 0)
scale = 1.0 / 128 ** 0.5
kc, vc, q, step_bytes = bench.build_headline(hs, dev, 0, scale)
flush = bench.Flusher(dev)
plan = hs.DecodePlan(q, kc, vc, scale=scale)
for _ in range(5): plan()
torch.cuda.synchronize()
def smi():
    return subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,clocks.mem,power.draw,temperature.gpu", "--format=csv,noheader"], capture_output=True, text=True).stdout.strip()
for r in range(int(sys.argv[1]) if len(sys.argv) > 1 else 12):
    st = [torch.cuda.Event(enable_timing=True) for _ in range(50)]
    sp = [torch.cuda.Event(enable_timing=True) for _ in range(50)]
    torch.cuda.synchronize()
    torch.cuda._sleep(int(1.965e9 * 0.02))
    for i in range(50):
        flush(); st[i].record(); plan(); sp[i].record()
    s1 = smi()
    torch.cuda.synchronize()
    t = [a.elapsed_time(b) * 1e3 for a, b in zip(st, sp)]
    slow = sum(x > 56.5 for x in t) / len(t)
    print(f"round {r}: median {statistics.median(t):.2f} mean {statistics.mean(t):.2f} min {min(t):.2f} max {max(t):.2f} slow {slow:.2f} | {s1}", flush=True)
