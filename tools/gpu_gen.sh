#!/bin/bash
# General-path check: the whole GPU suite, then per-config solve timings.
TAG=${1:-gen}
OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 600 python tools/config_sweep.py c1 c2 c4 > $OUT/sweep.jsonl 2>&1
grep -E "passed|failed|FAILED|Error|error" $OUT/pytest_gpu.log | tail -30; cat $OUT/sweep.jsonl
