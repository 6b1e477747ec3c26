# A/B against tools/_oldlib/liblbfgsb.so (a build of the baseline commit), one GPU job
mkdir -p gpurun_out/s31
timeout 900 python -m pytest tests -m gpu -q -x --timeout=600 > gpurun_out/s31/tests.log 2>&1
for i in 1 2; do
  python tools/_prof_with_lib.py tools/_oldlib/liblbfgsb.so tools/prof_bwdw.py C1 100 >> gpurun_out/s31/c1.log 2>&1
  python tools/prof_bwdw.py C1 100 >> gpurun_out/s31/c1.log 2>&1
  python tools/_prof_with_lib.py tools/_oldlib/liblbfgsb.so tools/prof_bwdw.py C4 200 >> gpurun_out/s31/c4.log 2>&1
  python tools/prof_bwdw.py C4 200 >> gpurun_out/s31/c4.log 2>&1
done
