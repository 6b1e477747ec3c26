# A/B against tools/_oldlib/liblbfgsb.so (a build of the baseline commit), one GPU job
mkdir -p gpurun_out/s28
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout=600 > gpurun_out/s28/tests.log 2>&1
for i in 1 2; do
  python tools/_prof_with_lib.py tools/_oldlib/liblbfgsb.so bench.py --no-cpu-baseline --steps 20 > gpurun_out/s28/b_old$i.log 2>&1
  python bench.py --no-cpu-baseline --steps 20 > gpurun_out/s28/b_new$i.log 2>&1
done
python tools/_prof_with_lib.py tools/_oldlib/liblbfgsb.so tools/bwd_sweep.py --child > gpurun_out/s28/gemvt_old.log 2>&1
python tools/bwd_sweep.py --child > gpurun_out/s28/gemvt_new.log 2>&1
