"""Randomised prefill parity sweep (tools): random L, n_q, sparsity, protection,
causality and GQA against the oracle; prints one line per case and a summary.
    python tools/prefill_stress.py [cases] [seed] [dtype]"""
import math, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle.oracle import Oracle
from tests.helpers import err_stats, to_torch, device_to_oracle, parallel, MAX_ABS_TOL, MEAN_REL_TOL
from tests.test_gpu_prefill import setup
from paper_2604_16864_b200 import hierasparse as hs
port = Oracle("port")
n = int(sys.argv[1]) if len(sys.argv) > 1 else 20
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
dtype = sys.argv[3] if len(sys.argv) > 3 else "f16"
bad = 0
for i in range(n):
    L = int(rng.choice([128, 192, 256, 384, 512, 640, 1024, 1536]))
    n_q = int(rng.integers(1, L + 1))
    s = float(rng.choice([0.0, 0.25, 0.5, 0.75, 1.0]))
    sink, window = int(rng.choice([0, 64, 100])), int(rng.choice([0, 128, 200]))
    causal = bool(rng.integers(0, 2))
    U, gqa = int(rng.integers(1, 3)), int(rng.choice([1, 2, 4]))
    hg = int(rng.choice([g for g in (1, 2, 4) if gqa % g == 0]))  # stacked-head layouts too
    os.environ["HS_PREFILL_HG"] = str(hg)
    kc, vc, q = setup(hs, port, U, L, s, dtype, gqa, n_q, sink, window, seed=100 + i)
    scale = np.float32(1.0 / math.sqrt(128))
    t0 = time.time()
    got = hs.prefill_attention(to_torch(q, dtype), kc, vc, causal=causal, scale=float(scale)).cpu().numpy()

    def one(ug):
        u, g = divmod(ug, gqa)
        return port.prefill(q[u, g], device_to_oracle(kc, u), device_to_oracle(vc, u), None, None, causal, scale, 64)
    want = np.stack(parallel(one, range(U * gqa))).reshape(U, gqa, n_q, 128)
    mx, mr = err_stats(got, want)
    ok = mx < MAX_ABS_TOL and mr < MEAN_REL_TOL
    bad += not ok
    print(f"{'ok ' if ok else 'BAD'} L={L} n_q={n_q} S={s} sink={sink} win={window} causal={causal} U={U} gqa={gqa}"
          f" max-abs {mx:.2e} mean-rel {mr:.2e} ({time.time() - t0:.1f}s)", flush=True)
print(f"{n - bad}/{n} cases within tolerance")
