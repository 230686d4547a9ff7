#!/bin/bash
# Prefill parity tests, repeated, each run under its own timeout (hang = rc 124).
O=gpurun_out/${1:-ptest}
mkdir -p $O
python -c 'import __graft_entry__ as g; g.build()' > $O/build.log 2>&1
for i in ${REPS:-1 2 3}; do timeout 240 python -m pytest tests/test_gpu_prefill.py -x -q -p no:cacheprovider > $O/run$i.log 2>&1; echo "run $i rc=$?" >> $O/summary.txt; done
