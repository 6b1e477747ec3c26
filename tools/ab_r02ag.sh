#!/bin/bash
# Round 2 (session 2): warp Alg. 3 (default) vs serial Alg. 3 in the k_bwd tails (rs)
set -u
O=gpurun_out/r02ag; mkdir -p $O
for sh in c2 c4; do
  timeout 600 python tools/_prof_with_lib.py tools/_var/trace/liblbfgsb.so tools/trace_phases.py $sh >> $O/trace_trace.jsonl 2>> $O/trace.err
done
for i in 1 2; do
  for v in default rs; do
    if [ $v = default ]; then L=paper_2203_16340_b200/liblbfgsb.so; else L=tools/_var/$v/liblbfgsb.so; fi
    for sh in c2 c4 c1; do
      LB_LIB=$v timeout 600 python tools/_prof_with_lib.py $L tools/ab_solve.py $sh 7 >> $O/ab_solve.log 2>&1
    done
  done
done
echo done > $O/done
