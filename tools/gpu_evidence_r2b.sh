#!/bin/bash
# Round-2 final evidence: default bench line, the ncu launch list of a short bench, ncu
# --set full of one even and one odd K1 launch (c5), the config sweep and the full-size
# L2 parity with the measured errors printed.
TAG=${1:-ev2}
OUT=gpurun_out/$TAG; mkdir -p $OUT
export PYTHONPATH=.
timeout 900 python bench.py > $OUT/bench.jsonl 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1200 --csv \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-general > $OUT/launches.csv 2> $OUT/launches.err
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_apply_s3 -s 10 -c 2 \
    -o $OUT/k1_full_c5 python tools/prof_gen.py c5 20 > $OUT/ncu_k1.log 2>&1
timeout 900 python tools/config_sweep.py > $OUT/config_sweep.jsonl 2> $OUT/config_sweep.err
timeout 1200 python -m pytest tests/test_gpu_fullsize.py -m gpu -q -s -k L2 > $OUT/fullsize_L2.log 2>&1
tail -c 1500 $OUT/bench.jsonl; tail -3 $OUT/bench.err; grep "L2 c" $OUT/fullsize_L2.log; tail -1 $OUT/fullsize_L2.log
