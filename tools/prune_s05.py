import os, sys, torch
sys.path.insert(0, os.getcwd())
from paper_2604_16864_b200 import hierasparse as hs
U, L = 8, 131072
g = torch.Generator(device="cuda").manual_seed(0)
k = torch.randn((U, L, 128), generator=g, device="cuda").bfloat16(); v = torch.randn((U, L, 128), generator=g, device="cuda").bfloat16()
cfg = hs.SparsityConfig(0.5, 0.5, 64)
out = hs.prune_cache(k, v, cfg)
for _ in range(3): hs.prune_cache(k, v, cfg, out=out)
torch.cuda.synchronize()
