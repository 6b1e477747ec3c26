#!/bin/bash
# round-2 GPU batch B: k_bwd unroll A/B (C5 chunk), N2 at the paper's tolerances, transport tests
set -u
O=gpurun_out/r02b; mkdir -p $O
for i in 1 2; do
  for v in default unr4_b2 unr4_b3 unr3_b3; do
    if [ $v = default ]; then L=paper_2203_16340_b200/liblbfgsb.so; else L=tools/_var/$v/liblbfgsb.so; fi
    LB_LIB=$v timeout 600 python tools/_prof_with_lib.py $L tools/prof_gemv_ab.py c5chunk 2 >> $O/ab_c5chunk.log 2>&1
  done
done
timeout 1200 python -m pytest tests/test_gpu_transport.py -q --timeout 900 -rf > $O/transport.log 2>&1
for tol in 1e-4 1e-5; do
  for n in 1000 2000; do timeout 900 python tools/diag_n2.py $n $tol >> $O/n2_paper_tol.log 2>&1; done
done
echo done > $O/done
