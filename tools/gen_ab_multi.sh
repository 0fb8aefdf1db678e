#!/bin/bash
# General-path A/B of several library builds ab/lib_<v>.so on one box: c4 and two mid-size 3D AMR meshes.
OUT=gpurun_out/${1:-genab}; shift; mkdir -p $OUT
for r in 1 2; do for v in "$@"; do
  cp ab/lib_$v.so paper_1009_4975_b200/libtomesh.so
  echo "$v c4 $(python tools/config_sweep.py c4 | python -c 'import json,sys; print(json.loads(sys.stdin.read())["us_per_iter_fixed200"])')  mid $(python tools/prof_c4mid.py 8 4 4 3 30 | awk '{print $NF}')  small $(python tools/prof_c4mid.py 8 4 4 2 30 | awk '{print $NF}')" | tee -a $OUT/ab.txt
done; done
