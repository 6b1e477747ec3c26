#!/bin/bash
# Round 2 (session 2): Gram accumulate with batched shared-memory loads + predicated k_fwd remainder batch (default), FWD_SHORT_B 16 (fb16), vs cdd3044 (prev) and 270cbaf (head)
set -u
O=gpurun_out/r02w; mkdir -p $O
for sh in c2 c4; do
  timeout 600 python tools/_prof_with_lib.py tools/_var/trace/liblbfgsb.so tools/trace_phases.py $sh >> $O/trace_trace.jsonl 2>> $O/trace.err
done
for i in 1 2; do
  for v in default prev head fb16; do
    if [ $v = default ]; then L=paper_2203_16340_b200/liblbfgsb.so; else L=tools/_var/$v/liblbfgsb.so; fi
    for sh in c2 c4 c1; do
      LB_LIB=$v timeout 600 python tools/_prof_with_lib.py $L tools/ab_solve.py $sh 7 >> $O/ab_solve.log 2>&1
    done
  done
done
timeout 2400 python -m pytest tests -m gpu -x -q --timeout=1200 > $O/tests.log 2>&1
echo done > $O/done
