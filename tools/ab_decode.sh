#!/bin/bash
# A/B of the configs[1] headline decode step (bench protocol: graph replay, L2 flushed) across library variants.
O=gpurun_out/${1:-abd}
mkdir -p $O
for rep in 1 2 3; do for v in ${VARS:-A B}; do
  echo -n "$v rep$rep " >> $O/ab.txt
  HS_LIB=abtest/lib$v.so timeout 300 python bench.py --headline-only --skip-cpu --steps 50 --warmup 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['decode_us'], d['roofline']['frac'])" >> $O/ab.txt
done; done
