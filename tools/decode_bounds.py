"""Split decode time into pipeline-only (no math) and compute-only (L2-resident) bounds."""
import os, statistics, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_16864_b200 import hierasparse as hs  # noqa: E402

U, L, GQA, D = 8, 131072, 4, 128
torch.manual_seed(0)
key = torch.randn(U, L, D, device="cuda").bfloat16()
val = torch.randn(U, L, D, device="cuda").bfloat16()
q = torch.randn(U, GQA, D, device="cuda").bfloat16()
kc, vc = hs.prune_cache(key, val, hs.SparsityConfig(1, 1, 64))
del key, val
out = torch.empty(U, GQA, D, device="cuda")
flush = torch.ones(64 * 1024 * 1024, device="cuda"); _sink = torch.empty(1, device="cuda")
def flush_l2():
    torch.sum(flush, dim=0, out=_sink)
nbytes = U * hs.flop_and_byte_count(GQA, kc, vc)[1]

def run(it=30):
    for _ in range(5):
        hs.decode_attention(q, kc, vc, out=out)
    ts = []
    for _ in range(it):
        flush_l2()
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record(); hs.decode_attention(q, kc, vc, out=out); b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    return statistics.median(ts)

for w in ("8", "4"):
    os.environ["HS_DECODE_WARPS"] = w
    base = run()
    os.environ["HS_DECODE_DEBUG_STREAM_ONLY"] = "1"
    stream = run()
    os.environ.pop("HS_DECODE_DEBUG_STREAM_ONLY")
    im_k, im_v = kc.index_map.clone(), vc.index_map.clone()
    kc.index_map.fill_(-1); vc.index_map.fill_(-1)
    comp = run()
    kc.index_map.copy_(im_k); vc.index_map.copy_(im_v)
    print(f"warps={w}: full {base:.1f} us ({nbytes/base/1e3:.0f} GB/s) | stream-only {stream:.1f} us "
          f"({nbytes/stream/1e3:.0f} GB/s) | compute (L2-resident) {comp:.1f} us", flush=True)
