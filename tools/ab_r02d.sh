#!/bin/bash
# round-2 GPU batch D: short-column kernels (C4 shape 1000 x 100000) A/B: k_bwd_w predicated tail /
# register cap / trip length, k_fwd load batch 16
set -u
O=gpurun_out/r02d; mkdir -p $O
for i in 1 2; do
  for v in default w_pred_b3 w_pred_b2 w_pred8_b2 w_b2 f16 f16_wpred_b2; do
    if [ $v = default ]; then L=paper_2203_16340_b200/liblbfgsb.so; else L=tools/_var/$v/liblbfgsb.so; fi
    LB_LIB=$v timeout 600 python tools/_prof_with_lib.py $L tools/prof_gemv_ab.py c4 3 >> $O/ab_c4.log 2>&1
  done
done
echo done > $O/done
