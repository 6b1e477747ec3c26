#!/bin/bash
# Round 2 (session 2): 256-bit loads in the generic k_bwd (C5 chunk 100000 x 25000): U quads per trip, CTAs per SM
set -u
O=gpurun_out/r02au; mkdir -p $O
for i in 1 2; do
  for v in default v40 u1 mb1 u3mb1; do
    if [ $v = default ]; then L=paper_2203_16340_b200/liblbfgsb.so; else L=tools/_var/$v/liblbfgsb.so; fi
    LB_LIB=$v timeout 900 python tools/_prof_with_lib.py $L tools/prof_gemv_ab.py c5chunk 2 >> $O/ab_c5chunk.log 2>&1
  done
done
echo done > $O/done
