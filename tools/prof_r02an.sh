#!/bin/bash
# N2 (DS2 entropy, n = 1000: 2M variables) launch list at the paper's tolerance, and an ncu full capture of k_qepi_d / k_tsum
set -u
O=gpurun_out/r02an; mkdir -p $O
timeout 600 python tools/run_n2.py --cases ds2:entropy:1000 --tol 1e-4 > $O/n2.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $O/launches_n2.csv python tools/run_n2.py --cases ds2:entropy:1000 --tol 1e-4 > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_qepi_d" -s 200 -c 1 -f -o $O/kqepi_d python tools/run_n2.py --cases ds2:entropy:1000 --tol 1e-4 > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_tsum" -s 200 -c 1 -f -o $O/ktsum python tools/run_n2.py --cases ds2:entropy:1000 --tol 1e-4 > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_dir" -s 200 -c 1 -f -o $O/kdir python tools/run_n2.py --cases ds2:entropy:1000 --tol 1e-4 > /dev/null 2>&1
echo done > $O/done
