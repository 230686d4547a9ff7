"""Prefill time and SM clock under load: configs[2] shape (8 KV heads x GQA 4,
causal, fp16) at the given context, each S timed over `reps` back-to-back
launches while nvidia-smi samples the SM clock (bench.ClockSampler).  Reports
cycles per 128x128 tile per SM at the sampled clock.
    python tools/prefill_clock.py [L] [reps] [S,S,...]"""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2604_16864_b200 import hierasparse as hs
from bench import ClockSampler
L = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 8
levels = [float(x) for x in sys.argv[3].split(",")] if len(sys.argv) > 3 else [0.0, 0.5, 1.0]
U, G = 8, 4
nt = L // 128
tiles = sum(min(nt, ((qt + 1) * 128 + 127) // 128) for qt in range(nt)) * U * G  # causal 128x128 tiles
torch.manual_seed(0)
q = torch.randn(U, G, L, 128, device="cuda").half()
out = torch.empty(U, G, L, 128, device="cuda")
for s in levels:
    k = torch.randn(U, L, 128, device="cuda").half(); v = torch.randn(U, L, 128, device="cuda").half()
    kc, vc = hs.prune_cache(k, v, hs.SparsityConfig(s, s, 64))
    fl = sum(hs.flop_and_byte_count(L, kc, vc, 0, True, unit=u)[0] for u in range(U)) * G
    for _ in range(3):
        hs.prefill_attention(q, kc, vc, causal=True, out=out)
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(True), torch.cuda.Event(True)) for _ in range(reps)]
    with ClockSampler(0) as cs:
        for a, b in ev:
            a.record(); hs.prefill_attention(q, kc, vc, causal=True, out=out); b.record()
        torch.cuda.synchronize()
    ms = [a.elapsed_time(b) for a, b in ev]
    c = cs.summary()
    med = statistics.median(ms)
    mhz = c["sm_mhz"] or 1965.0
    cyc = med * 1e-3 * mhz * 1e6 / (tiles / 148)
    print(f"L={L} S={s}: median {med:.3f} ms (min {min(ms):.3f}, first {ms[0]:.3f}), {fl / med / 1e9:.1f} TFLOPS, "
          f"clock {c['sm_mhz']} MHz {c['reasons']} n={c.get('samples')}, {cyc:.0f} cycles/tile/SM", flush=True)
    del kc, vc, k, v
