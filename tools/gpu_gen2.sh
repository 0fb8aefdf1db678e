#!/bin/bash
# General-path iteration: parity tests of the general path, timings, one ncu capture.
TAG=${1:-gen}
OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_amr.py tests/test_gpu_minres.py -m gpu -q -x > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 600 python tools/config_sweep.py c2 c4 > $OUT/sweep.jsonl 2>&1
python tools/prof_gen.py c4 200 > $OUT/plain.txt 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_gen_ --launch-skip 20 --launch-count 1 \
    -o $OUT/gen_c4 python tools/prof_gen.py c4 30 > $OUT/ncu.log 2>&1
grep -E "passed|failed|FAILED|Error|error" $OUT/pytest_gpu.log | tail -30; cat $OUT/sweep.jsonl $OUT/plain.txt
