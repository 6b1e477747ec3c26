mkdir -p gpurun_out/s12
timeout 900 python -m pytest tests/test_gpu_p2p.py tests/test_gpu_sharded.py tests/test_gpu_parity.py -q -x --timeout=600 > gpurun_out/s12/tests.log 2>&1
for mb in 1 3 4; do
  for i in 1 2; do LBFGSB_FWD_MINB=$mb timeout 300 python bench.py --no-cpu-baseline --steps 20 > gpurun_out/s12/b_mb${mb}_$i.log 2>&1; done
  LBFGSB_FWD_MINB=$mb python tools/prof_bwdw.py C4 200 > gpurun_out/s12/c4_mb$mb.log 2>&1
done
timeout 300 python bench.py --force-sharded --steps 10 > gpurun_out/s12/bench_sh_p2p.log 2>&1
timeout 300 python bench.py --force-sharded --xchg nccl --steps 10 > gpurun_out/s12/bench_sh_nccl.log 2>&1
