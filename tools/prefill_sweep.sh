#!/bin/bash
# Prefill timing sweep (configs[2] shape) + one trace; used during kernel work.
O=gpurun_out/${1:-pf}
mkdir -p $O
python -c 'import __graft_entry__ as g; g.build()' > $O/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_prefill.py -x -q > $O/pytest_prefill.log 2>&1; echo "rc=$?" >> $O/pytest_prefill.log
for s in 0.0 0.5 0.75 1.0; do timeout 300 python tools/prefill_prof.py 65536 $s >> $O/sweep.txt 2>&1; done
timeout 300 python tools/prefill_trace.py 16384 1.0 > $O/trace.txt 2>&1
