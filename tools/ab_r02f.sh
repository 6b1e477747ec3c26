#!/bin/bash
set -u
O=gpurun_out/r02f; mkdir -p $O
timeout 1800 python -m pytest tests/test_gpu_full_configs.py tests/test_gpu_bench.py tests/test_gpu_batch.py tests/test_gpu_al_general.py -q --timeout 1500 -rf > $O/tests.log 2>&1
timeout 900 compute-sanitizer --tool memcheck python tools/sanitize_cases.py c4s c1 > $O/memcheck_c4s.log 2>&1
timeout 900 compute-sanitizer --tool racecheck python tools/sanitize_cases.py c4s > $O/racecheck_c4s.log 2>&1
for i in 1 2; do
  for v in default nobwds nobwds_u8b1; do
    if [ $v = default ]; then L=paper_2203_16340_b200/liblbfgsb.so; else L=tools/_var/$v/liblbfgsb.so; fi
    LB_LIB=$v timeout 600 python tools/_prof_with_lib.py $L tools/prof_gemv_ab.py c2 3 >> $O/ab_c2.log 2>&1
  done
done
echo done > $O/done
