#!/bin/bash
# Round 2 (session 2): k_fwd CTAs per SM (LBFGSB_FWD_MINB 1 / 3 / 4; default: 3 for m >= 2048, 1 below)
set -u
O=gpurun_out/r02aw; mkdir -p $O
for i in 1 2; do
  for mb in default 3 4 1; do
    for sh in c2 c4; do
      if [ $mb = default ]; then timeout 600 python tools/ab_solve.py $sh 7 | sed "s/\"lib\": \"default\"/\"lib\": \"fwd_minb_$mb\"/" >> $O/ab_solve.log 2>&1
      else LBFGSB_FWD_MINB=$mb timeout 600 python tools/ab_solve.py $sh 7 | sed "s/\"lib\": \"default\"/\"lib\": \"fwd_minb_$mb\"/" >> $O/ab_solve.log 2>&1; fi
    done
  done
done
echo done > $O/done
