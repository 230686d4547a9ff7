"""One prefill timing line: 8 kv heads x GQA 4, causal, given dtype.
    python tools/prefill_prof_dt.py L S {f16|bf16}"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2604_16864_b200 import hierasparse as hs
L = int(sys.argv[1]); s = float(sys.argv[2]); dt = torch.bfloat16 if sys.argv[3] == "bf16" else torch.float16
U, G = 8, 4
torch.manual_seed(0)
k = torch.randn(U, L, 128, device="cuda").to(dt); v = torch.randn(U, L, 128, device="cuda").to(dt)
kc, vc = hs.prune_cache(k, v, hs.SparsityConfig(s, s, 64))
q = torch.randn(U, G, L, 128, device="cuda").to(dt)
out = torch.empty(U, G, L, 128, device="cuda")
for _ in range(2):
    hs.prefill_attention(q, kc, vc, causal=True, out=out)
torch.cuda.synchronize()
ts = []
for _ in range(3):
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(); hs.prefill_attention(q, kc, vc, causal=True, out=out); e1.record(); torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
fl = sum(hs.flop_and_byte_count(L, kc, vc, 0, True, unit=u)[0] for u in range(U)) * G
ms = sorted(ts)[1]
print(f"L={L} s={s} {sys.argv[3]}: {ms:.3f} ms, {fl / ms / 1e9:.1f} counted TFLOPS ({fl / ms / 1e9 / 1662.3:.3f})")
