O=gpurun_out/hg1; mkdir -p $O
python -c 'import __graft_entry__ as g; g.build()' > $O/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_prefill.py tests/test_gpu_fullsize.py -x -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 900 python tools/prefill_ab_env.py 65536 "0.0,0.5,0.75,1.0" "HS_PREFILL_HG=1|HS_PREFILL_HG=2|HS_PREFILL_HG=4" 3 > $O/ab.txt 2>&1
AB_BF16=1 timeout 600 python tools/prefill_ab_env.py 65536 "0.0,1.0" "HS_PREFILL_HG=1|HS_PREFILL_HG=4" 2 > $O/ab_bf16.txt 2>&1
