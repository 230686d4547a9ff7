"""Randomised decode parity sweep (tools): random units, context, block sparsity,
protection, GQA rows (1-16), dense tail, split count, dtype and the plan / host-I/O
entry points against the oracle's decode_attention (attention.hpp:360-409).
    python tools/decode_stress.py [cases] [seed]"""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from oracle.oracle import Oracle
from paper_2604_16864_b200 import hierasparse as hs
from tests.helpers import MAX_ABS_TOL, MEAN_REL_TOL, err_stats, gen_units, to_torch
from tests.test_gpu_decode import build_caches, decode_queries, oracle_decode

port = Oracle("port")
n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
bad = 0
for i in range(n):
    U = int(rng.integers(1, 5))
    L = int(rng.choice([64, 128, 640, 2048, 4096, 8192, 16384]))
    s = float(rng.choice([0.0, 0.25, 0.5, 0.75, 1.0]))
    sink, window = int(rng.choice([0, 64, 100])), int(rng.choice([0, 128, 300]))
    gqa = int(rng.choice([1, 2, 4, 8, 12, 16]))
    tail = int(rng.choice([0, 0, 1, 37, 63]))
    dtype = str(rng.choice(["bf16", "f16"]))
    splits = int(rng.choice([0, 0, 1, 3, 7]))
    mode = str(rng.choice(["call", "plan", "host_io"]))
    kx, vx, kc, vc = build_caches(hs, port, U, L, s, dtype, sink, window, seed=200 + i)
    q = decode_queries(port, U, gqa, dtype, seed=200 + i)
    scale = np.float32(1.0 / math.sqrt(128))
    kt = vt = None
    if tail:
        kt = gen_units(port, U, tail, 128, 300 + i, 0, dtype)
        vt = gen_units(port, U, tail, 128, 300 + i, 1, dtype)
    want = oracle_decode(port, kc, vc, q, scale, 4, kt, vt)
    qt = to_torch(q, dtype)
    if mode == "call" or tail or splits:
        got = hs.decode_attention(qt, kc, vc, None if kt is None else to_torch(kt, dtype),
                                  None if vt is None else to_torch(vt, dtype), float(scale), splits=splits)
        mode = "call"
    else:
        plan = hs.DecodePlan(qt, kc, vc, scale=float(scale), host_io=(mode == "host_io"))
        got = plan()
    torch.cuda.synchronize()
    got = got.cpu().numpy() if hasattr(got, "cpu") else got
    mx, mr = err_stats(np.asarray(got), want)
    ok = mx < MAX_ABS_TOL and mr < MEAN_REL_TOL
    bad += not ok
    print(f"{'ok ' if ok else 'BAD'} U={U} L={L} S={s} sink={sink} win={window} gqa={gqa} tail={tail} {dtype} "
          f"splits={splits} {mode}: max-abs {mx:.2e} mean-rel {mr:.2e}", flush=True)
print(f"{n - bad}/{n} cases within tolerance")
