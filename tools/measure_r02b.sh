#!/bin/bash
# Round-2 (second session) measurement batch (GPU box, one B200): tests, smoke, bench (default C5 at N=1 with the
# embedded C2 line), reference arm, ncu launch list + traffic + full captures, BASELINE configs, side-lines,
# sanitizer of the general AL path.  Output in gpurun_out/final/.
set -u
O=gpurun_out/final2; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $O/smi.txt 2>&1
T0=$(date +%s); timeout 2400 python -m pytest tests -m gpu -q --timeout=1500 -rf > $O/tests.log 2>&1; echo "rc=$? seconds=$(( $(date +%s) - T0 ))" >> $O/tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 1500 python bench.py > $O/bench.log 2>&1
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref.log 2>&1
timeout 900 python bench.py --impl reference --config C2 --steps 2 --warmup 1 > $O/bench_ref_c2.log 2>&1
B="python bench.py --steps 1 --warmup 3 --no-c2 --no-cpu-baseline"
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file $O/launches_c5.csv $B > /dev/null 2>&1
timeout 1200 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
  -k regex:"k_bwd" -s 40 -c 6 --csv --log-file $O/traffic_c5.csv $B > /dev/null 2>&1
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:"k_bwd" -s 40 -c 1 -f -o $O/kbwd_c5_full $B > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_fwd" -s 40 -c 1 -f -o $O/kfwd_c5_full $B > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file $O/launches_c2.csv python bench.py --config C2 --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_bwd_s" -s 12 -c 1 -f -o $O/kbwd_s_c2_full python tools/ab_solve.py c2 1 > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_bwd_wo" -s 8 -c 1 -f -o $O/kbwd_wo_c4_full python tools/ab_solve.py c4 1 > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_fwd" -s 8 -c 1 -f -o $O/kfwd_c4_full python tools/ab_solve.py c4 1 > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c4.csv python tools/ab_solve.py c4 1 > /dev/null 2>&1
for sh in c2 c4; do timeout 600 python tools/ab_solve.py $sh 7 >> $O/ab_solve.log 2>&1; done
timeout 1800 python tools/run_configs.py C1 C3 C3en C4 > $O/configs.log 2>&1
timeout 600 python tools/run_n1.py 10000 > $O/n1.log 2>&1
echo done > $O/done
