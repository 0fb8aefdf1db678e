#!/bin/bash
# Guarded quick check for risky kernel changes: small parity first (short timeout), then bench.
TAG=${1:-q}; OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 120 python -m pytest tests/test_gpu_parity.py -x -q -k "c5s or c3s" > $OUT/pytest_small.log 2>&1; rc=$?; echo "small rc=$rc" >> $OUT/pytest_small.log
if [ $rc -ne 0 ]; then tail -20 $OUT/pytest_small.log; exit 1; fi
timeout 300 python -m pytest tests -m gpu -x -q -k parity > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $OUT/bench.log 2>&1; echo "bench rc=$?" >> $OUT/bench.log
tail -3 $OUT/pytest_gpu.log; tail -1 $OUT/bench.log
