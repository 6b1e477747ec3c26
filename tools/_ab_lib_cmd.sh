# A/B against tools/_oldlib/liblbfgsb.so (a build of the baseline commit), one GPU job
mkdir -p gpurun_out/s30
timeout 900 python -m pytest tests -m gpu -q -x --timeout=600 > gpurun_out/s30/tests.log 2>&1
for i in 1 2; do
  python tools/_prof_with_lib.py tools/_oldlib/liblbfgsb.so bench.py --no-cpu-baseline --steps 20 > gpurun_out/s30/b_old$i.log 2>&1
  python bench.py --no-cpu-baseline --steps 20 > gpurun_out/s30/b_new$i.log 2>&1
done
python tools/_prof_with_lib.py tools/_oldlib/liblbfgsb.so tools/bwd_sweep.py --child > gpurun_out/s30/gemvt_old.log 2>&1
python tools/bwd_sweep.py --child > gpurun_out/s30/gemvt_new.log 2>&1
