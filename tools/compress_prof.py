"""Compression timing on configs[1] caches (8 KV heads x 128K x 128 bf16): the
bench's compress leg (preallocated pools, L2 flushed): prune_cache at S = 1
(static) and S = 0.5 (loss-driven), the decode-phase recompress 0.5 -> 1."""
import json, os, sys, types
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2604_16864_b200 import hierasparse as hs
dev = torch.device("cuda", 0)
args = types.SimpleNamespace(steps=int(sys.argv[1]) if len(sys.argv) > 1 else 10)
print(json.dumps(bench.leg_compress(hs, dev, 0, 1, args, bench.Flusher(dev)), indent=1))
