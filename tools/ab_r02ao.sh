#!/bin/bash
# Round 2 (session 2): N2 entropy search with 1 / 2 / 3 in-graph continuation passes (TS_NCONT)
set -u
O=gpurun_out/r02ao; mkdir -p $O
for i in 1 2; do
  for v in default nc1 nc3; do
    if [ $v = default ]; then L=paper_2203_16340_b200/liblbfgsb.so; else L=tools/_var/$v/liblbfgsb.so; fi
    echo "== $v" >> $O/n2.log
    LB_LIB=$v timeout 900 python tools/_prof_with_lib.py $L tools/run_n2.py --cases ds2:entropy:1000,ds2:entropy:2000 --tol 1e-4 >> $O/n2.log 2>&1
    LB_LIB=$v timeout 900 python tools/_prof_with_lib.py $L tools/run_n2.py --cases ds2:entropy:1000 --tol 1e-5 >> $O/n2.log 2>&1
  done
done
timeout 1200 python -m pytest tests/test_gpu_transport.py -x -q --timeout=1000 > $O/tests.log 2>&1
echo done > $O/done
