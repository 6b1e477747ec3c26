#!/bin/bash
# Round 2 (session 2): k_tsum with 4 columns per trip (default; 2 CTAs/SM), at 3 / 4 CTAs per SM (tb3, tb4), vs prev
set -u
O=gpurun_out/r02ar; mkdir -p $O
for i in 1 2; do
  for v in default prev tb3 tb4; do
    if [ $v = default ]; then L=paper_2203_16340_b200/liblbfgsb.so; else L=tools/_var/$v/liblbfgsb.so; fi
    echo "== $v" >> $O/n2.log
    LB_LIB=$v timeout 900 python tools/_prof_with_lib.py $L tools/run_n2.py --cases ds2:entropy:1000,ds2:entropy:2000,ds1:gaussian:1000 --tol 1e-4 >> $O/n2.log 2>&1
  done
done
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:"k_tsum" -s 200 -c 4 --csv --log-file $O/ktsum_n2.csv python tools/run_n2.py --cases ds2:entropy:1000 --tol 1e-4 > /dev/null 2>&1
timeout 1200 python -m pytest tests/test_gpu_transport.py -x -q --timeout=1000 > $O/tests.log 2>&1
echo done > $O/done
