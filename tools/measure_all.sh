#!/bin/bash
# Round measurement batch (run on the GPU box via gpurun): tests, configs,
# side-lines, bench, bench launch list and the full ncu captures of the
# dominant kernels (k_bwd_s, k_fwd on C2; k_bwd_w on C4).
set -u
O=gpurun_out/meas; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $O/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q --timeout=600 > $O/tests.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 600 python bench.py > $O/bench.log 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref.log 2>&1
timeout 600 python bench.py --force-sharded --steps 10 > $O/bench_sharded_p2p.log 2>&1
timeout 600 python bench.py --force-sharded --xchg nccl --steps 10 > $O/bench_sharded_nccl.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/bench_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > $O/bench_ncu.log 2>&1
timeout 600 ncu --set full --import-source on -k regex:k_bwd_s -s 5 -c 1 -f -o $O/kbwd_s_full python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --set full --import-source on -k regex:k_fwd -s 5 -c 1 -f -o $O/kfwd_full python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --set full --import-source on -k regex:k_bwd_w -s 40 -c 1 -f -o $O/kbwd_w_full python tools/prof_bwdw.py C4 60 > /dev/null 2>&1
timeout 900 python tools/run_configs.py > $O/configs.log 2>&1
timeout 600 python tools/run_c5.py > $O/c5.log 2>&1
timeout 300 python tools/run_n1.py 10000 > $O/n1.log 2>&1
timeout 900 python tools/run_n2.py --tol 1e-6 --cases ds1:entropy:1000,ds1:gaussian:1000,ds2:entropy:1000,ds2:gaussian:1000,ds1:gaussian:2000,ds1:gaussian:3000,ds2:gaussian:2000,ds2:gaussian:3000,ds1:entropy:2000,ds2:entropy:2000 > $O/n2.log 2>&1
echo done > $O/done
