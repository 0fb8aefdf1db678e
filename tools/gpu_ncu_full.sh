#!/bin/bash
# ncu --set full of the hot kernels on a shortened bench step.
# usage: gpurun -- bash tools/gpu_ncu_full.sh TAG CONFIG ITERS KERNEL_REGEX COUNT
TAG=${1:-r1}; CFG=${2:-c5}; IT=${3:-4}; KR=${4:-"k_apply_s3|k_u1|k_u2|k_sens|k_filter"}; CNT=${5:-5}
OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 300 python tools/prof_run.py $CFG $IT > $OUT/prof_plain.log 2>&1 || { echo "plain run failed"; tail $OUT/prof_plain.log; exit 1; }
timeout 1500 ncu --set full --clock-control none --import-source on -k "regex:$KR" -c $CNT \
   -o $OUT/full_$CFG python tools/prof_run.py $CFG $IT > $OUT/ncu_full.log 2>&1; echo "ncu rc=$?"
tail -5 $OUT/ncu_full.log
