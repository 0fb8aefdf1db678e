#!/bin/bash
# A/B of library variants on c4 and c4L (us per iteration, fixed iterations).
TAG=${1:-genab}; shift
OUT=gpurun_out/$TAG; mkdir -p $OUT
cp paper_1009_4975_b200/libtomesh.so /tmp/lib_keep.so
for r in 1 2; do for v in "$@"; do
  cp ab/lib_$v.so paper_1009_4975_b200/libtomesh.so
  echo "$v c4 $(python tools/prof_gen.py c4 300 | awk '{print $5}') c4L $(python tools/prof_gen.py c4L 100 | awk '{print $5}')" | tee -a $OUT/ab.txt
done; done
cp /tmp/lib_keep.so paper_1009_4975_b200/libtomesh.so
