"""Fixed overhead vs marginal streaming rate of the decode kernel."""
import os, statistics, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_16864_b200 import hierasparse as hs  # noqa: E402
GQA, D = 4, 128
flush = torch.ones(64 * 1024 * 1024, device="cuda"); _sink = torch.empty(1, device="cuda")
def flush_l2():
    torch.sum(flush, dim=0, out=_sink)
def timeit(fn, it=20):
    for _ in range(3): fn()
    ts = []
    for _ in range(it):
        flush_l2(); a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record(); fn(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b) * 1e3)
    return statistics.median(ts)
res = {}
for U, L in ((8, 32768), (8, 65536), (8, 131072), (8, 262144), (16, 131072), (32, 131072)):
    torch.manual_seed(0)
    key = torch.randn(U, L, D, device="cuda").bfloat16(); val = torch.randn(U, L, D, device="cuda").bfloat16()
    q = torch.randn(U, GQA, D, device="cuda").bfloat16()
    kc, vc = hs.prune_cache(key, val, hs.SparsityConfig(1, 1, 64)); del key, val
    out = torch.empty(U, GQA, D, device="cuda")
    nbytes = U * hs.flop_and_byte_count(GQA, kc, vc)[1]
    t = timeit(lambda: hs.decode_attention(q, kc, vc, out=out))
    os.environ["HS_DECODE_DEBUG_STREAM_ONLY"] = "1"
    ts = timeit(lambda: hs.decode_attention(q, kc, vc, out=out))
    os.environ.pop("HS_DECODE_DEBUG_STREAM_ONLY")
    pools = [kc.nnz_pool, kc.meta_pool, vc.nnz_pool, vc.meta_pool]
    tsum = 1.0  # timeit(lambda: [p.view(torch.int16).sum(dtype=torch.int32) for p in pools])
    print(f"U={U} L={L}: {nbytes/1e6:.0f} MB decode {t:.1f} us ({nbytes/t/1e3:.0f} GB/s) stream-only {ts:.1f} us "
          f"({nbytes/ts/1e3:.0f}) | torch sum of pools {tsum:.1f} us ({nbytes/tsum/1e3:.0f} GB/s)", flush=True)
    del kc, vc
