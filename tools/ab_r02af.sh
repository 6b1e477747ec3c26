#!/bin/bash
# Round 2 (session 2): the C4 AL solve's inner-iteration count under summation-order variants of this build
# (serial Alg. 3 in the k_bwd tails: rs; k_bwd_wd instead of k_bwd_wo: wd; both: rswd)
set -u
O=gpurun_out/r02af; mkdir -p $O
for v in rs wd rswd; do
  echo "== $v" >> $O/configs_c4.log
  LB_LIB=$v timeout 900 python tools/_prof_with_lib.py tools/_var/$v/liblbfgsb.so tools/run_configs.py C4 >> $O/configs_c4.log 2>&1
done
echo done > $O/done
