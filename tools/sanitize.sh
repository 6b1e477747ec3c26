#!/bin/bash
# compute-sanitizer runs (memcheck on every kernel family; racecheck and
# synccheck on the ones with shared-memory / barrier protocols; memcheck of the
# two-process CUDA-IPC P2P exchange).  Run on the GPU box via gpurun; logs in
# gpurun_out/san/.
set -u
O=gpurun_out/san; mkdir -p $O
CS="compute-sanitizer --print-limit 20 --error-exitcode 99"
for c in c1 c2s c4s lasso al loop3 group batch qp transport; do
  timeout 900 $CS --tool memcheck python tools/sanitize_cases.py $c > $O/memcheck_$c.log 2>&1; echo "memcheck $c rc=$?" >> $O/summary.txt
done
for c in c1 c2s c4s loop3 group batch qp; do
  timeout 1200 $CS --tool racecheck --racecheck-report hazard python tools/sanitize_cases.py $c > $O/racecheck_$c.log 2>&1; echo "racecheck $c rc=$?" >> $O/summary.txt
  timeout 900 $CS --tool synccheck python tools/sanitize_cases.py $c > $O/synccheck_$c.log 2>&1; echo "synccheck $c rc=$?" >> $O/summary.txt
done
timeout 1200 $CS --tool memcheck --target-processes all python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 \
  --master-addr=127.0.0.1 --master-port=29731 tests/_p2p_worker.py /tmp/p2p_san.npz 1200 900 83 1 > $O/memcheck_ipc2.log 2>&1
echo "memcheck ipc2 rc=$?" >> $O/summary.txt
echo done >> $O/summary.txt
