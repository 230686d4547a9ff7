#!/bin/bash
# Decompose prefill time: full / no softmax / no MMA / neither (HS_PREFILL_MODE),
# single CTA (latency) vs a 148-CTA grid of one head (bandwidth).  Mode 7 =
# TMA streaming only (stages released on arrival).
O=gpurun_out/${1:-pm}
mkdir -p $O
python -c 'import __graft_entry__ as g; g.build()' > $O/build.log 2>&1
for s in 0.0 1.0; do for m in ${MODES:-0 1 2 3 7}; do for c in 1 148; do HS_PREFILL_MODE=$m timeout 300 python tools/prefill_lat.py 32768 $s $c >> $O/lat.txt 2>&1; done; done; done
