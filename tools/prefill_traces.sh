#!/bin/bash
O=gpurun_out/${1:-pt}
mkdir -p $O
python -c 'import __graft_entry__ as g; g.build()' > $O/build.log 2>&1
for s in 0.0 1.0; do for m in ${MODES:-0 3 7}; do HS_PREFILL_MODE=$m timeout 300 python tools/prefill_trace.py 32768 $s >> $O/trace.txt 2>&1; done; done
