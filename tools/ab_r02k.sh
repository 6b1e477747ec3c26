#!/bin/bash
set -u
O=gpurun_out/r02k; mkdir -p $O
for i in 1 2; do
  for v in default spf4 spf2; do
    if [ $v = default ]; then L=paper_2203_16340_b200/liblbfgsb.so; else L=tools/_var/$v/liblbfgsb.so; fi
    LB_LIB=$v timeout 600 python tools/_prof_with_lib.py $L tools/prof_gemv_ab.py c2 3 >> $O/ab_c2.log 2>&1
  done
done
echo done > $O/done
