#!/bin/bash
# General path: deterministic gather (default) vs the TOMESH_GENERAL_ATOMIC experiment, same box.
OUT=gpurun_out/${1:-atomab}; mkdir -p $OUT
TOMESH_GENERAL_ATOMIC=1 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "L2 and (c4s or amr3d or c5s_general)" 2>&1 | tail -2 | tee -a $OUT/ab.txt
for r in 1 2; do for v in det atom; do
  if [ $v = atom ]; then export TOMESH_GENERAL_ATOMIC=1; else unset TOMESH_GENERAL_ATOMIC; fi
  echo "$v c4 $(python tools/config_sweep.py c4 | python -c 'import json,sys; print(json.loads(sys.stdin.read())["us_per_iter_fixed200"])')  mid $(python tools/prof_c4mid.py 8 4 4 3 30 | awk '{print $NF}')  small $(python tools/prof_c4mid.py 8 4 4 2 30 | awk '{print $NF}')" | tee -a $OUT/ab.txt
done; done
