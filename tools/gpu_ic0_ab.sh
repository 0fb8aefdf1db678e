#!/bin/bash
# IC(0) triangular-solve pipelining: MINRES parity tests, then Jacobi-PCG vs MINRES vs MINRES+IC(0) on c1, c2.
TAG=${1:-ic0}
OUT=gpurun_out/$TAG; mkdir -p $OUT
export PYTHONPATH=.
timeout 900 python -m pytest tests/test_gpu_minres.py -q > $OUT/pytest_minres.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_minres.log
timeout 900 python tools/solver_compare.py c1 c2 > $OUT/solver_compare.jsonl 2> $OUT/solver_compare.err
tail -3 $OUT/pytest_minres.log; cat $OUT/solver_compare.jsonl | cut -c1-600
