#!/bin/bash
# Published in-kernel step (step_in = 2): parity, determinism, timings.
TAG=${1:-pub}
OUT=gpurun_out/$TAG; mkdir -p $OUT
export PYTHONPATH=.
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_amr.py -q -x > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest.log
timeout 600 python tools/repeat_check.py > $OUT/repeat.log 2>&1; echo "repeat rc=$?" >> $OUT/repeat.log
timeout 600 python tools/mid_ab.py > $OUT/mid_ab.log 2>&1
timeout 900 python tools/config_sweep.py c2 c4 c4L > $OUT/config_sweep.jsonl 2> $OUT/config_sweep.err
tail -3 $OUT/pytest.log; tail -4 $OUT/repeat.log; cat $OUT/mid_ab.log | tail -3; cut -c1-330 $OUT/config_sweep.jsonl
