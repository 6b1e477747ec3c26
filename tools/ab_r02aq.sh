#!/bin/bash
# Round 2 (session 2): k_dir ring loads not predicated on the mask (default) vs the committed k_dir (prev)
set -u
O=gpurun_out/r02aq; mkdir -p $O
for i in 1 2; do
  for v in default prev; do
    if [ $v = default ]; then L=paper_2203_16340_b200/liblbfgsb.so; else L=tools/_var/$v/liblbfgsb.so; fi
    echo "== $v" >> $O/n2.log
    LB_LIB=$v timeout 900 python tools/_prof_with_lib.py $L tools/run_n2.py --cases ds2:entropy:1000,ds2:entropy:2000 --tol 1e-4 >> $O/n2.log 2>&1
    for sh in c2 c4 c1; do
      LB_LIB=$v timeout 600 python tools/_prof_with_lib.py $L tools/ab_solve.py $sh 7 >> $O/ab_solve.log 2>&1
    done
  done
done
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_dir" -s 200 -c 3 --csv --log-file $O/kdir_n2.csv python tools/run_n2.py --cases ds2:entropy:1000 --tol 1e-4 > /dev/null 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q --timeout=1200 -k "not full and not c5" > $O/tests.log 2>&1
echo done > $O/done
