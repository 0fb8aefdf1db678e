#!/bin/bash
# Full default bench (with the oracle CPU baseline) + the ncu launch list of the same command.
TAG=${1:-ev}; OUT=gpurun_out/$TAG; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/nvsmi.txt 2>&1
timeout 900 python bench.py > $OUT/bench.log 2>&1; echo "bench rc=$?" >> $OUT/bench.log
timeout 900 python bench.py --impl reference --steps 1 --warmup 0 > $OUT/bench_ref.log 2>&1; echo "ref rc=$?" >> $OUT/bench_ref.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1200 --csv --log-file $OUT/launches.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $OUT/ncu_launch.log 2>&1; echo "ncu rc=$?" >> $OUT/ncu_launch.log
tail -2 $OUT/bench.log; tail -2 $OUT/bench_ref.log
