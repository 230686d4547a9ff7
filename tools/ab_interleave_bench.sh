#!/bin/bash
# Bench-level A/B of the interleaved decode grid (HS_DECODE_INTERLEAVE=0/1), 3 alternating rounds.
O=gpurun_out/ilb
mkdir -p $O
for rep in 1 2 3; do for v in 0 1; do
  echo -n "interleave=$v rep$rep " >> $O/ab.txt
  HS_DECODE_INTERLEAVE=$v timeout 300 python bench.py --headline-only --skip-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['decode_us'], d['roofline']['frac'], d['e2e']['ms_per_step'])" >> $O/ab.txt
done; done
