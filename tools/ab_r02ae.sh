#!/bin/bash
# Round 2 (session 2): C5-chunk GEMV launch times and the C4 AL solve, this build vs the session start (270cbaf)
set -u
O=gpurun_out/r02ae; mkdir -p $O
for v in default head; do
  if [ $v = default ]; then L=paper_2203_16340_b200/liblbfgsb.so; else L=tools/_var/$v/liblbfgsb.so; fi
  LB_LIB=$v timeout 900 python tools/_prof_with_lib.py $L tools/prof_gemv_ab.py c5chunk 2 >> $O/ab_c5chunk.log 2>&1
done
for v in head default; do
  if [ $v = default ]; then L=paper_2203_16340_b200/liblbfgsb.so; else L=tools/_var/$v/liblbfgsb.so; fi
  echo "== $v" >> $O/configs_c4.log
  LB_LIB=$v timeout 900 python tools/_prof_with_lib.py $L tools/run_configs.py C4 >> $O/configs_c4.log 2>&1
done
echo done > $O/done
