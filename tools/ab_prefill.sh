#!/bin/bash
# A/B timing of two builds of the library in one box session (abtest/libA.so vs libB.so),
# alternating runs to cancel clock drift.
O=gpurun_out/${1:-ab}
mkdir -p $O
for rep in 1 2; do for v in ${VARS:-A B}; do for s in ${SPARS:-0.0 1.0}; do
  echo -n "$v rep$rep " >> $O/ab.txt; HS_LIB=abtest/lib$v.so timeout 300 python tools/prefill_prof.py ${LCTX:-32768} $s >> $O/ab.txt 2>&1
done; done; done
