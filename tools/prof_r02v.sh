#!/bin/bash
# ncu --set full (source-level stall sampling) of k_bwd_wd (C4 shape) and k_bwd_s (C2) at HEAD
set -u
O=gpurun_out/r02v; mkdir -p $O
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_bwd_wd" -s 8 -c 1 -f -o $O/kbwd_wd_c4 python tools/ab_solve.py c4 1 > $O/ncu_wd.log 2>&1

echo done > $O/done
