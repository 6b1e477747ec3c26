# A/B of the working tree against _ab (a worktree at the previous commit), one GPU job
mkdir -p gpurun_out/s13
timeout 900 python -m pytest tests -m gpu -q -x --timeout=600 > gpurun_out/s13/tests.log 2>&1
for i in 1 2; do
  (cd _ab && python ../tools/prof_bwdw.py C4 200) >> gpurun_out/s13/c4.log 2>&1
  python tools/prof_bwdw.py C4 200 >> gpurun_out/s13/c4.log 2>&1
done
(cd _ab && timeout 300 python bench.py --no-cpu-baseline --steps 20) > gpurun_out/s13/b_old.log 2>&1
timeout 300 python bench.py --no-cpu-baseline --steps 20 > gpurun_out/s13/b_new.log 2>&1
timeout 300 python tools/run_n2.py --eps 1e-20 --tol 1e-6 --cases ds1:gaussian:1000 > gpurun_out/s13/n2_g_eps20.log 2>&1
timeout 300 python tools/run_n2.py --tol 1e-6 --cases ds1:gaussian:1000,ds2:gaussian:1000,ds2:entropy:1000 > gpurun_out/s13/n2.log 2>&1
