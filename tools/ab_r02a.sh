#!/bin/bash
# round-2 GPU batch A: general-AL tests, N2 diagnostics, k_bwd unroll A/B, IPC sanitizer (2 processes)
set -u
O=gpurun_out/r02a; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_al_general.py -q --timeout 600 -rf > $O/al_general.log 2>&1
for i in 1 2; do
  for v in default unr2_b3 unr2_b4; do
    if [ $v = default ]; then L=paper_2203_16340_b200/liblbfgsb.so; else L=tools/_var/$v/liblbfgsb.so; fi
    LB_LIB=$v timeout 600 python tools/_prof_with_lib.py $L tools/prof_gemv_ab.py c5chunk 2 >> $O/ab_c5chunk.log 2>&1
    LB_LIB=$v timeout 600 python tools/_prof_with_lib.py $L tools/prof_gemv_ab.py c2 3 >> $O/ab_c2.log 2>&1
  done
done
timeout 900 python tools/diag_n2.py 1000 2e-6 > $O/n2_1000.log 2>&1
timeout 900 python tools/diag_n2.py 400 1e-8 > $O/n2_400.log 2>&1
# two-process P2P exchange under memcheck, each rank its own sanitizer process
for r in 0 1; do
  RANK=$r WORLD_SIZE=2 LOCAL_RANK=$r MASTER_ADDR=127.0.0.1 MASTER_PORT=29741 timeout 900 \
    compute-sanitizer --tool memcheck --print-limit 20 python tests/_p2p_worker.py /tmp/p2p_san_$r.npz 1200 900 83 1 \
    > $O/memcheck_ipc_rank$r.log 2>&1 &
done
wait
echo done > $O/done
