"""A/B of a decode run-time switch on the bench headline (default HS_DECODE_MAILBOX:
0 = counter release/acquire then plain partial loads, 1 = tagged mailbox): two
DecodePlans captured under each setting, replayed alternately after an L2 flush with
the stream held while the host enqueues (bench protocol).  Outputs must agree to
fp32 rounding.
    python tools/decode_mailbox_ab.py [reps] [VAR] [value_a value_b]"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
from paper_2604_16864_b200 import hierasparse as hs

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
VAR = sys.argv[2] if len(sys.argv) > 2 else "HS_DECODE_MAILBOX"
VALS = (sys.argv[3], sys.argv[4]) if len(sys.argv) > 4 else ("0", "1")
dev = torch.device("cuda", 0)
scale = 1.0 / 128 ** 0.5
kc, vc, q, step_bytes = bench.build_headline(hs, dev, 0, scale)
flush = bench.Flusher(dev)
plans = {}
for var in VALS:
    os.environ[VAR] = var
    plans[var] = hs.DecodePlan(q, kc, vc, scale=scale)
    for _ in range(5):
        plans[var]()
torch.cuda.synchronize()
d = (plans[VALS[0]].out - plans[VALS[1]].out).abs().max().item()
print(f"max |{VAR}={VALS[1]} - {VAR}={VALS[0]}| = {d:.3e}")
ref = hs.decode_attention(q, kc, vc, scale=scale, splits=18)  # static, deterministic


def run(plan, steps=50):
    st = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    sp = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    torch.cuda.synchronize()
    torch.cuda._sleep(int(1.965e9 * 0.02))
    for i in range(steps):
        flush()
        st[i].record()
        plan()
        sp[i].record()
    torch.cuda.synchronize()
    t = [a.elapsed_time(b) * 1e3 for a, b in zip(st, sp)]
    return statistics.mean(t), statistics.median(t)


for rep in range(reps):
    for var in VALS:
        m, md = run(plans[var])
        err = (plans[var].out - ref).abs().max().item()
        print(f"{VAR}={var}: mean {m:.2f} median {md:.2f} us ({step_bytes / (md * 1e-6) / 1e9:.0f} GB/s) "
              f"max |out - static| {err:.2e}", flush=True)
