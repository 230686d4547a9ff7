#!/bin/bash
# One GPU-box pass: parity tests, smoke, bench (both arms), ncu launch list and
# full captures of the decode / prefill / compress kernels.  Outputs -> gpurun_out/.
# Usage: bash tools/gpu_round.sh [tag]
TAG=${1:-r02}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi > $O/smi.txt 2>&1
nproc > $O/nproc.txt; lscpu >> $O/nproc.txt 2>&1
python -c 'import __graft_entry__ as g; g.build()' > $O/build.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c 'import __graft_entry__ as g; g.smoke()' > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "rc=$?" >> $O/bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err
NCU=/usr/local/cuda/bin/ncu
timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv \
   python bench.py --steps 2 --warmup 3 --profile --prefill-steps 1 > $O/ncu_launch_bench.log 2>&1
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:decode_kernel -s 3 -c 1 -o $O/decode_full \
   python bench.py --steps 1 --warmup 3 --profile --no-prefill > $O/ncu_decode.log 2>&1
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:block_kernel -c 1 -o $O/compress_full \
   python bench.py --steps 1 --warmup 3 --profile --no-prefill > $O/ncu_compress.log 2>&1
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:prefill_kernel -s 2 -c 1 -o $O/prefill_full \
   python tools/prefill_prof.py 16384 1.0 > $O/ncu_prefill.log 2>&1
echo done > $O/DONE
