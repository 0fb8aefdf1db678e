#!/bin/bash
# Last verification of the round's HEAD: the whole GPU suite and smoke().
TAG=${1:-final3}
OUT=gpurun_out/$TAG; mkdir -p $OUT
export PYTHONPATH=.
ls -la cache/oracle_ref tests/golden > $OUT/cache_listing.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -s -rs > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
grep -E "passed|failed|SKIP|L2 c" $OUT/pytest_gpu.log | cut -c1-200; tail -2 $OUT/smoke.log
