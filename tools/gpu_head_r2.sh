#!/bin/bash
# HEAD evidence on one B200: default bench line, config sweep, ncu launch list of a short bench.
TAG=${1:-head}
OUT=gpurun_out/$TAG; mkdir -p $OUT
export PYTHONPATH=.
timeout 900 python bench.py > $OUT/bench.jsonl 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/bench.err
timeout 900 python tools/config_sweep.py > $OUT/config_sweep.jsonl 2> $OUT/config_sweep.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1200 --csv \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-general > $OUT/launches.csv 2> $OUT/launches.err
tail -c 1500 $OUT/bench.jsonl; tail -3 $OUT/bench.err
