"""Run one prefill parity case (tests/test_gpu_prefill.py shapes) with the
pipeline watchdog on (HS_DEBUG_WAIT=1): a hang becomes an error naming the wait."""
import math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("HS_DEBUG_WAIT", "1")
import numpy as np
from oracle.oracle import Oracle
from tests.helpers import err_stats, to_torch, device_to_oracle
from tests.test_gpu_prefill import setup
from paper_2604_16864_b200 import hierasparse as hs
L, n_q, s, sink, window, causal, dtype = int(sys.argv[1]), int(sys.argv[2]), float(sys.argv[3]), int(sys.argv[4]), \
    int(sys.argv[5]), sys.argv[6] == "1", sys.argv[7]
port = Oracle("port")
U, gqa = 2, 2
kc, vc, q = setup(hs, port, U, L, s, dtype, gqa, n_q, sink, window)
scale = np.float32(1.0 / math.sqrt(128))
try:
    got = hs.prefill_attention(to_torch(q, dtype), kc, vc, causal=causal, scale=float(scale)).cpu().numpy()
except Exception as e:
    print("ERROR", e)
    sys.exit(1)
want = np.stack([port.prefill(q[u, g], device_to_oracle(kc, u), device_to_oracle(vc, u), None, None, causal, scale, 64)
                 for u in range(U) for g in range(gqa)]).reshape(U, gqa, n_q, 128)
print("err", err_stats(got, want))
