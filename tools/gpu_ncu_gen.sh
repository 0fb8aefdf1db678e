#!/bin/bash
# ncu --set full of one general-path iteration kernel (k_gen_fused) on a config.
TAG=${1:-ncugen}; CFG=${2:-c4}
OUT=gpurun_out/$TAG; mkdir -p $OUT
python tools/prof_gen.py $CFG 50 > $OUT/plain.txt 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_gen_ --launch-skip 20 --launch-count 1 \
    -o $OUT/gen_$CFG python tools/prof_gen.py $CFG 30 > $OUT/ncu.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:k_ python tools/prof_gen.py $CFG 30 > $OUT/launches.csv 2>&1
cat $OUT/plain.txt; tail -3 $OUT/ncu.log
