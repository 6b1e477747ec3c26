#!/bin/bash
set -u
O=gpurun_out/r02m2; mkdir -p $O
LB_LIB=wt timeout 900 python tools/_prof_with_lib.py tools/_var/wt/liblbfgsb.so tools/check_wt.py > $O/check_wt.log 2>&1
for i in 1 2; do
  for v in default wt; do
    if [ $v = default ]; then L=paper_2203_16340_b200/liblbfgsb.so; else L=tools/_var/$v/liblbfgsb.so; fi
    LB_LIB=$v timeout 600 python tools/_prof_with_lib.py $L tools/prof_gemv_ab.py c4 3 >> $O/ab_c4.log 2>&1
  done
done
LB_LIB=wt timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:k_bwd -c 12 --csv --log-file $O/wt_names.csv python tools/_prof_with_lib.py tools/_var/wt/liblbfgsb.so tools/prof_gemv_ab.py c4 1 > /dev/null 2>&1
LB_LIB=wt timeout 600 compute-sanitizer --tool memcheck python tools/_prof_with_lib.py tools/_var/wt/liblbfgsb.so tools/sanitize_cases.py c4s > $O/memcheck_wt.log 2>&1
LB_LIB=wt timeout 900 compute-sanitizer --tool racecheck python tools/_prof_with_lib.py tools/_var/wt/liblbfgsb.so tools/sanitize_cases.py c4s > $O/racecheck_wt.log 2>&1
LB_LIB=wt timeout 900 compute-sanitizer --tool synccheck python tools/_prof_with_lib.py tools/_var/wt/liblbfgsb.so tools/sanitize_cases.py c4s > $O/synccheck_wt.log 2>&1
echo done > $O/done
