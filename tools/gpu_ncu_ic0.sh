#!/bin/bash
# ncu --set full of the IC(0) triangular solve on c2 (after a plain run).
TAG=${1:-ic0ncu}
OUT=gpurun_out/$TAG; mkdir -p $OUT
export PYTHONPATH=.
timeout 300 python tools/prof_ic0.py c2 6 > $OUT/plain.log 2>&1 || { tail $OUT/plain.log; exit 1; }
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_ic0_tri --launch-skip 4 --launch-count 2 \
   -o $OUT/ic0_tri_c2 python tools/prof_ic0.py c2 6 > $OUT/ncu.log 2>&1; echo "ncu rc=$?"
tail -3 $OUT/ncu.log
