"""One prefill launch for profiling: 8 kv heads x GQA 4, causal, fp16."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2604_16864_b200 import hierasparse as hs
L = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
s = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
U, G = 8, 4
torch.manual_seed(0)
k = torch.randn(U, L, 128, device="cuda").half(); v = torch.randn(U, L, 128, device="cuda").half()
kc, vc = hs.prune_cache(k, v, hs.SparsityConfig(s, s, 64))
q = torch.randn(U, G, L, 128, device="cuda").half()
out = torch.empty(U, G, L, 128, device="cuda")
for _ in range(3):
    hs.prefill_attention(q, kc, vc, causal=True, out=out)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record(); hs.prefill_attention(q, kc, vc, causal=True, out=out); e1.record(); torch.cuda.synchronize()
fl = sum(hs.flop_and_byte_count(L, kc, vc, 0, True, unit=u)[0] for u in range(U)) * G
print(f"L={L} s={s}: {e0.elapsed_time(e1):.3f} ms, {fl / e0.elapsed_time(e1) / 1e9:.1f} counted TFLOPS")
