O=gpurun_out/r02k; mkdir -p $O
for rep in 1 2; do for v in A J JN; do for s in 0.0 1.0; do
  lib=$v; env=""; if [ $v = JN ]; then lib=J; env="HS_PREFILL_NO_SAFE=1"; fi
  echo -n "$v rep$rep " >> $O/ab.txt; env $env HS_LIB=abtest/lib$lib.so timeout 300 python tools/prefill_prof.py 65536 $s >> $O/ab.txt 2>&1
done; done; done
