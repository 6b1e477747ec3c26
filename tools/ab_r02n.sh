#!/bin/bash
# Round 2 (session 2): phase traces of the iteration kernels (C2, C4 shapes) and the
# deferred-epilogue short-column k_bwd_wd A/B against k_bwd_w (C4 shape), its parity run.
set -u
O=gpurun_out/r02n; mkdir -p $O
for sh in c4 c2; do
  timeout 600 python tools/_prof_with_lib.py tools/_var/trace/liblbfgsb.so tools/trace_phases.py $sh >> $O/trace.jsonl 2>> $O/trace.err
done
for v in wd3 wd2; do
  timeout 600 python tools/_prof_with_lib.py tools/_var/$v/liblbfgsb.so tools/trace_phases.py c4 >> $O/trace_$v.jsonl 2>> $O/trace.err
done
for i in 1 2; do
  for v in default wd3n wd2n; do
    if [ $v = default ]; then L=paper_2203_16340_b200/liblbfgsb.so; else L=tools/_var/$v/liblbfgsb.so; fi
    LB_LIB=$v timeout 600 python tools/_prof_with_lib.py $L tools/prof_gemv_ab.py c4 3 >> $O/ab_c4.log 2>&1
  done
done
timeout 1200 python tools/_pytest_with_lib.py tools/_var/wd3n/liblbfgsb.so tests -m gpu -x -q -k "not c5 and not full and not group" > $O/tests_wd3n.log 2>&1
echo done > $O/done
