#!/bin/bash
# ncu evidence for the C5 bench line: launch list of the bench command, DRAM
# traffic of k_bwd / k_fwd launches, one full capture of k_bwd.  gpurun_out/ncu5/.
set -u
O=gpurun_out/ncu5; mkdir -p $O
B="python bench.py --steps 1 --warmup 3 --no-c2 --no-cpu-baseline"
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file $O/launches_c5.csv $B > $O/launches_c5.log 2>&1
echo "launches rc=$?" >> $O/summary.txt
timeout 1200 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
  -k regex:"k_bwd|k_fwd" -s 40 -c 6 --csv --log-file $O/traffic_c5.csv $B > $O/traffic_c5.log 2>&1
echo "traffic rc=$?" >> $O/summary.txt
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:"k_bwd" -s 40 -c 1 -f -o $O/kbwd_c5_full $B > $O/kbwd_full.log 2>&1
echo "full rc=$?" >> $O/summary.txt
echo done >> $O/summary.txt
