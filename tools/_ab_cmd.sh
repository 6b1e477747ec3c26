# A/B of the working tree against _ab (a worktree at the previous commit), one GPU job
mkdir -p gpurun_out/s20
timeout 900 python -m pytest tests -m gpu -q -x --timeout=600 > gpurun_out/s20/tests.log 2>&1
for i in 1 2; do
  (cd _ab && python ../tools/prof_bwdw.py C4 200) >> gpurun_out/s20/c4.log 2>&1
  python tools/prof_bwdw.py C4 200 >> gpurun_out/s20/c4.log 2>&1
  (cd _ab && timeout 300 python bench.py --no-cpu-baseline --steps 20) > gpurun_out/s20/b_old$i.log 2>&1
  timeout 300 python bench.py --no-cpu-baseline --steps 20 > gpurun_out/s20/b_new$i.log 2>&1
done
(cd _ab && python ../tools/bwd_sweep.py --child) > gpurun_out/s20/gemvt_old.log 2>&1
python tools/bwd_sweep.py --child > gpurun_out/s20/gemvt_new.log 2>&1
