import os, sys, math
if os.environ.get("DBG", "1") == "1":
    os.environ["HS_DEBUG_WAIT"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2604_16864_b200 import hierasparse as hs
L = int(sys.argv[1]) if len(sys.argv) > 1 else 512
s = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
dt = torch.bfloat16 if (len(sys.argv) > 3 and sys.argv[3] == "bf16") else torch.float16
U = int(sys.argv[4]) if len(sys.argv) > 4 else 1
G = int(sys.argv[5]) if len(sys.argv) > 5 else 1
torch.manual_seed(0)
k = torch.randn(U, L, 128, device="cuda").to(dt); v = torch.randn(U, L, 128, device="cuda").to(dt)
kc, vc = hs.prune_cache(k, v, hs.SparsityConfig(s, s, 64))
q = torch.randn(U, G, L, 128, device="cuda").to(dt)
try:
    out = hs.prefill_attention(q, kc, vc, causal=True)
    torch.cuda.synchronize()
    # torch reference on decompressed caches
    kd = hs.decompress(kc).float()[-1]; vd = hs.decompress(vc).float()[-1]
    sc = (q[-1, -1].float() @ kd.T) / math.sqrt(128)
    mask = torch.triu(torch.ones(L, L, dtype=torch.bool, device="cuda"), 1)
    sc = sc.masked_fill(mask, float("-inf"))
    ref = torch.softmax(sc, -1) @ vd
    print("L", L, "s", s, dt, U, G, "maxdiff", (out[-1, -1] - ref).abs().max().item(), "ref max", ref.abs().max().item())
except Exception as e:
    print("ERR", e)
