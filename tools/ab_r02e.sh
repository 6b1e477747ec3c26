#!/bin/bash
# round-2 GPU batch E: C2 backward GEMV: k_bwd_s vs the generic k_bwd (four / eight row pairs per trip)
set -u
O=gpurun_out/r02e; mkdir -p $O
for i in 1 2; do
  for v in default nobwds nobwds_u8b1; do
    if [ $v = default ]; then L=paper_2203_16340_b200/liblbfgsb.so; else L=tools/_var/$v/liblbfgsb.so; fi
    LB_LIB=$v timeout 600 python tools/_prof_with_lib.py $L tools/prof_gemv_ab.py c2 3 >> $O/ab_c2.log 2>&1
  done
done
LB_LIB=default timeout 600 python tools/prof_gemv_ab.py c4 3 >> $O/ab_c4_new_default.log 2>&1
echo done > $O/done
