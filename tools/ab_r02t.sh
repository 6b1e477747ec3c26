#!/bin/bash
# Round 2 (session 2): finer traces (k_bwd_wd barrier / epilogue split, k_fwd row-block / global tails) at C2, C4, C1
set -u
O=gpurun_out/r02t; mkdir -p $O
for sh in c2 c4 c1; do
  timeout 600 python tools/_prof_with_lib.py tools/_var/trace/liblbfgsb.so tools/trace_phases.py $sh >> $O/trace.jsonl 2>> $O/trace.err
done
echo done > $O/done
