#!/bin/bash
# Whole GPU test suite (no -x: every failure reported) + a short bench.
# usage: gpurun -- bash tools/gpu_all.sh TAG [pytest -k expr]
TAG=${1:-all}; KX=${2:-}
OUT=gpurun_out/$TAG; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/gpu.txt 2>&1
if [ -n "$KX" ]; then timeout 1500 python -m pytest tests -m gpu -q -k "$KX" > $OUT/pytest_gpu.log 2>&1; else
timeout 1500 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; fi; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $OUT/bench.log 2>&1; echo "bench rc=$?" >> $OUT/bench.log
grep -E "passed|failed|FAILED|Error" $OUT/pytest_gpu.log | tail -30; tail -2 $OUT/bench.log
