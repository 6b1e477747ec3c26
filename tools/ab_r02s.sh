#!/bin/bash
# Round 2 (session 2): acq_rel last-CTA tickets, batched split-K tail loads, Ctrl scalars cached for the
# Alg. 3 tail, k_bwd_wd per-warp ranges; against the session's starting HEAD (270cbaf) build
set -u
O=gpurun_out/r02s; mkdir -p $O
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,clocks.mem,power.draw,clocks_throttle_reasons.active --format=csv > $O/smi.txt
for v in trace trace_tail0; do
  for sh in c2 c4; do
    timeout 600 python tools/_prof_with_lib.py tools/_var/$v/liblbfgsb.so tools/trace_phases.py $sh >> $O/trace_$v.jsonl 2>> $O/trace.err
  done
done
for i in 1 2; do
  for v in default head tail0 tail8; do
    if [ $v = default ]; then L=paper_2203_16340_b200/liblbfgsb.so; else L=tools/_var/$v/liblbfgsb.so; fi
    for sh in c2 c4 c1; do
      LB_LIB=$v timeout 600 python tools/_prof_with_lib.py $L tools/ab_solve.py $sh 7 >> $O/ab_solve.log 2>&1
    done
  done
done
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,clocks.mem,power.draw,clocks_throttle_reasons.active --format=csv >> $O/smi.txt
timeout 2400 python -m pytest tests -m gpu -x -q --timeout=1200 > $O/tests.log 2>&1
echo done > $O/done
