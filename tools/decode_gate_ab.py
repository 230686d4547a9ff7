import os, sys, statistics, torch
sys.path.insert(0, os.getcwd())
import bench
from paper_2604_16864_b200 import hierasparse as hs
dev = torch.device("cuda", 0)
kc, vc, q, step_bytes = bench.build_headline(hs, dev, 0, 1.0 / 128 ** 0.5)
flush = bench.Flusher(dev)
plan = hs.DecodePlan(q, kc, vc, scale=1.0 / 128 ** 0.5)
for _ in range(5): plan()
torch.cuda.synchronize()
def run(gate, sampler, steps=50):
    st = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    sp = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    ctx = bench.ClockSampler(0) if sampler else None
    if ctx: ctx.__enter__()
    torch.cuda.synchronize()
    if gate: torch.cuda._sleep(int(1.965e9 * 0.02))  # hold the stream ~20 ms while the host enqueues
    for i in range(steps):
        flush(); st[i].record(); plan(); sp[i].record()
    torch.cuda.synchronize()
    if ctx: ctx.__exit__()
    t = [a.elapsed_time(b) * 1e3 for a, b in zip(st, sp)]
    return statistics.mean(t), statistics.median(t), max(t)
for rep in range(3):
    for gate in (False, True):
        for sampler in (False, True):
            m, md, mx = run(gate, sampler)
            print(f"gate={gate} sampler={sampler}: mean {m:.1f} median {md:.1f} max {mx:.1f} us", flush=True)
