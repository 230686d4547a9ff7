#!/bin/bash
# A/B of prefill library builds (abtest/libX.so) at configs[2] shape: alternating
# runs of tools/prefill_ab_env.py (baseline variant only).  Outputs gpurun_out/$1/ab.txt
O=gpurun_out/${1:-abp}; mkdir -p $O
for rep in 1 2; do for v in ${VARS:-A B}; do
  echo "== $v rep$rep" >> $O/ab.txt
  HS_LIB=abtest/lib$v.so timeout 600 python tools/prefill_ab_env.py ${LCTX:-65536} ${SPARS:-0.0,0.5,1.0} "X=" 2 2>&1 | grep "best" >> $O/ab.txt
done; done
