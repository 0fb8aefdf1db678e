#!/bin/bash
# General-path A/B of two library builds (ab/lib_old.so, ab/lib_new.so) on one box.
for r in 1 2; do for v in old new; do
  cp ab/lib_$v.so paper_1009_4975_b200/libtomesh.so
  echo "$v c4 $(python tools/config_sweep.py c4 | python -c 'import json,sys; print(json.loads(sys.stdin.read())["us_per_iter_fixed200"])')  mid $(python tools/prof_c4mid.py 8 4 4 3 30 | awk '{print $NF}')  small $(python tools/prof_c4mid.py 8 4 4 2 30 | awk '{print $NF}')"
done; done
cp ab/lib_new.so paper_1009_4975_b200/libtomesh.so
