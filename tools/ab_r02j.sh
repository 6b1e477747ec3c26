#!/bin/bash
set -u
O=gpurun_out/r02j; mkdir -p $O
for i in 1 2; do
  for v in default wpf fpf wpf_fpf; do
    if [ $v = default ]; then L=paper_2203_16340_b200/liblbfgsb.so; else L=tools/_var/$v/liblbfgsb.so; fi
    LB_LIB=$v timeout 600 python tools/_prof_with_lib.py $L tools/prof_gemv_ab.py c4 3 >> $O/ab_c4.log 2>&1
  done
done
echo done > $O/done
