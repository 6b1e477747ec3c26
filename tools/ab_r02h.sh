#!/bin/bash
set -u
O=gpurun_out/r02h; mkdir -p $O
for i in 1 2; do
  for v in default bwds_u4 bwds_u3; do
    if [ $v = default ]; then L=paper_2203_16340_b200/liblbfgsb.so; else L=tools/_var/$v/liblbfgsb.so; fi
    LB_LIB=$v timeout 600 python tools/_prof_with_lib.py $L tools/prof_gemv_ab.py c2 3 >> $O/ab_c2.log 2>&1
  done
done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_bwd_s" -s 12 -c 1 -f -o $O/kbwd_s_c2_full python tools/prof_gemv_ab.py c2 1 > $O/ncu.log 2>&1
echo done > $O/done
