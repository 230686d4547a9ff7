"""configs[1] K + V prune_cache at S=1 (static selection, no losses) for an ncu
DRAM-bytes capture of the two pack kernels (tools; profiles/r02j_compress_dram.md).
    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
        -k regex:block_kernel python tools/compress_dram.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2604_16864_b200 import hierasparse as hs

U, L = 8, 131072
g = torch.Generator(device="cuda").manual_seed(0)
k = torch.randn((U, L, 128), generator=g, device="cuda").bfloat16()
v = torch.randn((U, L, 128), generator=g, device="cuda").bfloat16()
cfg = hs.SparsityConfig(1.0, 1.0, 64)
out = hs.prune_cache(k, v, cfg)
hs.prune_cache(k, v, cfg, out=out)
torch.cuda.synchronize()
