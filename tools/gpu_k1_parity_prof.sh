#!/bin/bash
# K1 per-parity evidence on c5: the launch list of a 20-iteration fixed solve
# (even kernels update x, odd ones defer it), then ncu --set full of one even
# and one odd launch (launches 10 and 11).
# usage: gpurun -- bash tools/gpu_k1_parity_prof.sh TAG
TAG=${1:-k1par}; OUT=gpurun_out/$TAG; mkdir -p $OUT
export PYTHONPATH=.
timeout 300 python tools/prof_gen.py c5 20 > $OUT/plain.log 2>&1 || { echo "plain run failed"; tail $OUT/plain.log; exit 1; }
cat $OUT/plain.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_apply_s3 --csv \
  --log-file $OUT/launches.csv python tools/prof_gen.py c5 20 > $OUT/ncu_list.log 2>&1; echo "list rc=$?"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_apply_s3 -s 10 -c 2 \
  -o $OUT/full_c5 python tools/prof_gen.py c5 20 > $OUT/ncu_full.log 2>&1; echo "full rc=$?"
tail -3 $OUT/ncu_full.log
