#!/bin/bash
# Round-2 (late) evidence for the general path: default bench line, ncu --set
# full of the general block kernel on c4 and c4L, the config sweep.
TAG=${1:-ev3}
OUT=gpurun_out/$TAG; mkdir -p $OUT
export PYTHONPATH=.
timeout 900 python bench.py > $OUT/bench.jsonl 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/bench.err
for c in c4 c4L; do
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_gen_fused --launch-skip 20 --launch-count 1 \
      -o $OUT/gen_${c}_full python tools/prof_gen.py $c 30 > $OUT/ncu_$c.log 2>&1
done
timeout 900 python tools/config_sweep.py > $OUT/config_sweep.jsonl 2> $OUT/config_sweep.err
tail -c 2500 $OUT/bench.jsonl; tail -3 $OUT/bench.err; tail -2 $OUT/ncu_c4L.log
