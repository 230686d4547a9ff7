#!/bin/bash
# A/B timing of compression library variants (abtest/libX.so): tools/compress_prof.py per variant, alternating.
O=gpurun_out/${1:-abc}
mkdir -p $O
for rep in 1 2; do for v in ${VARS:-A B}; do
  echo "== $v rep$rep" >> $O/ab.txt; HS_LIB=abtest/lib$v.so timeout 300 python tools/compress_prof.py 10 >> $O/ab.txt 2>&1
done; done
