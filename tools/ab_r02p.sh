#!/bin/bash
# Round 2 (session 2): templated Alg. 3 tail, epilogue prefetch, k_bwd_wd default, FWD_BAL A/B; full GPU suite
set -u
O=gpurun_out/r02p; mkdir -p $O
for v in trace trace_bal; do
  for sh in c2 c4; do
    timeout 600 python tools/_prof_with_lib.py tools/_var/$v/liblbfgsb.so tools/trace_phases.py $sh >> $O/trace_$v.jsonl 2>> $O/trace.err
  done
done
for i in 1 2; do
  for v in default nopf bal old; do
    if [ $v = default ]; then L=paper_2203_16340_b200/liblbfgsb.so; else L=tools/_var/$v/liblbfgsb.so; fi
    for sh in c2 c4 c1; do
      LB_LIB=$v timeout 600 python tools/_prof_with_lib.py $L tools/ab_solve.py $sh 7 >> $O/ab_solve.log 2>&1
    done
  done
done
timeout 2400 python -m pytest tests -m gpu -x -q --timeout=1500 > $O/tests.log 2>&1
echo done > $O/done
