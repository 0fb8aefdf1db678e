#!/bin/bash
# Quick GPU check: parity tests + short bench.  usage: gpurun -- bash tools/gpu_quick.sh TAG [pytest -k expr]
TAG=${1:-q}; KX=${2:-}
OUT=gpurun_out/$TAG; mkdir -p $OUT
if [ -n "$KX" ]; then timeout 900 python -m pytest tests -m gpu -x -q -k "$KX" > $OUT/pytest_gpu.log 2>&1; else
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; fi; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $OUT/bench.log 2>&1; echo "bench rc=$?" >> $OUT/bench.log
tail -4 $OUT/pytest_gpu.log; tail -2 $OUT/bench.log
