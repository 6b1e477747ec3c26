#!/bin/bash
# Round 2 (session 2): k_bwd_wo / k_bwd_wd under the LB_CHECK debug build (device-side bounds checks that trap;
# compute-sanitizer is closed on this pool): the short-column tests, the parity suite, the C4 shape solve
set -u
O=gpurun_out/r02ak; mkdir -p $O
L=tools/_var/check/liblbfgsb.so
timeout 1500 python tools/_pytest_with_lib.py $L tests/test_gpu_short.py tests/test_gpu_parity.py -q --timeout=1200 -k "not full" > $O/tests_check.log 2>&1
LB_LIB=check timeout 600 python tools/_prof_with_lib.py $L tools/ab_solve.py c4 3 > $O/c4_check.log 2>&1
LB_LIB=check timeout 900 python tools/_prof_with_lib.py $L tools/run_configs.py C1 C3en > $O/configs_check.log 2>&1
echo done > $O/done
