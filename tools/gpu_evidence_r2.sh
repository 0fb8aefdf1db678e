#!/bin/bash
# Round-2 evidence: bench line (default run), the ncu launch list of a short bench,
# ncu --set full of K1 (c5) and of the general-path kernel on c4L.
TAG=${1:-ev}
OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 900 python bench.py --steps 5 --warmup 3 > $OUT/bench.jsonl 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/bench.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 1200 --csv \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-general > $OUT/launches.csv 2> $OUT/launches.err
ncu --set full --import-source on --clock-control none -k regex:k_gen_fused --launch-skip 20 --launch-count 1 \
    -o $OUT/c4L_gen_full python tools/prof_gen.py c4L 30 > $OUT/ncu_c4L.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_gen_fused --launch-skip 20 --launch-count 1 \
    -o $OUT/c4_gen_full python tools/prof_gen.py c4 30 > $OUT/ncu_c4.log 2>&1
tail -c 3000 $OUT/bench.jsonl; tail -3 $OUT/bench.err
