#!/bin/bash
# Round 2 (session 2): the new short-column tests (compute-sanitizer is closed on this pool)
set -u
O=gpurun_out/r02ac; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_short.py -q --timeout=1200 > $O/tests_short.log 2>&1
echo done > $O/done
