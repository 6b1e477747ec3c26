#!/bin/bash
# HEAD verification (second session): the whole GPU suite, smoke, the default bench line
set -u
O=gpurun_out/verify2; mkdir -p $O
T0=$(date +%s); timeout 2400 python -m pytest tests -m gpu -q --timeout=1500 -rf > $O/tests.log 2>&1; echo "rc=$? seconds=$(( $(date +%s) - T0 ))" >> $O/tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 1500 python bench.py > $O/bench.log 2>&1
echo done > $O/done
