# A/B of the working tree against _ab, one GPU job (gpurun -- 'bash tools/_ab_cmd.sh').
# _ab is a worktree of the baseline commit with its own built library:
#   git worktree add -f _ab <commit> && echo _ab/ >> .git/info/exclude
#   (cd _ab && python -c "from paper_2203_16340_b200 import _build; _build.build()")
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
