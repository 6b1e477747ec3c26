#!/bin/bash
# Round 2 (session 2): tail traces + PDL / one-level Gram tail / k_bwd_wd A/B (whole solves, no event nodes)
set -u
O=gpurun_out/r02o; mkdir -p $O
for v in trace trace_opt; do
  for sh in c2 c4; do
    timeout 600 python tools/_prof_with_lib.py tools/_var/$v/liblbfgsb.so tools/trace_phases.py $sh >> $O/trace_$v.jsonl 2>> $O/trace.err
  done
done
for i in 1 2; do
  for v in default pdl g1 opt; do
    if [ $v = default ]; then L=paper_2203_16340_b200/liblbfgsb.so; else L=tools/_var/$v/liblbfgsb.so; fi
    for sh in c2 c4 c1; do
      LB_LIB=$v timeout 600 python tools/_prof_with_lib.py $L tools/ab_solve.py $sh 7 >> $O/ab_solve.log 2>&1
    done
  done
done
timeout 1500 python tools/_pytest_with_lib.py tools/_var/opt/liblbfgsb.so tests -m gpu -x -q -k "not c5 and not full" > $O/tests_opt.log 2>&1
echo done > $O/done
