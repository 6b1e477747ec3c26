#!/bin/bash
# Round measurement batch (run on the GPU box via gpurun): tests, configs,
# side-lines, bench, bench launch list and the k_bwd_s full ncu capture.
set -u
O=gpurun_out/meas; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q --timeout=400 > $O/tests.log 2>&1
timeout 600 python tools/run_configs.py > $O/configs.log 2>&1
timeout 400 python tools/run_c5.py > $O/c5.log 2>&1
timeout 300 python tools/run_n1.py 10000 > $O/n1.log 2>&1
LBFGSB_NO_QEPI_T=1 timeout 300 python tools/run_n1.py 10000 > $O/n1_noqt.log 2>&1
timeout 900 python tools/run_n2.py --eps 1e-20 --tol 1e-6 --cases ds1:entropy:1000,ds1:gaussian:1000,ds2:entropy:1000,ds2:gaussian:1000,ds1:gaussian:2000,ds1:gaussian:3000,ds2:gaussian:2000,ds2:gaussian:3000,ds1:entropy:2000,ds2:entropy:2000 > $O/n2.log 2>&1
timeout 600 python bench.py > $O/bench.log 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/bench_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > $O/bench_ncu.log 2>&1
timeout 600 ncu --set full --import-source on -k regex:k_bwd_s -s 5 -c 1 -f -o $O/kbwd_s_full python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --set full --import-source on -k regex:k_fwd -s 5 -c 1 -f -o $O/kfwd_full python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
echo done > $O/done
