# A/B against tools/_oldlib/liblbfgsb.so (a build of the baseline commit), one GPU job
mkdir -p gpurun_out/s27
timeout 600 python -m pytest tests/test_gpu_variants_env.py -q -x --timeout=600 > gpurun_out/s27/tests.log 2>&1
python tools/bwd_sweep.py --bench > gpurun_out/s27/sweep.log 2>&1
