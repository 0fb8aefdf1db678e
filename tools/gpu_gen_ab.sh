#!/bin/bash
# A/B of general-path library variants (ab/lib_*.so) on c4: us per iteration.
TAG=${1:-genab}; shift
OUT=gpurun_out/$TAG; mkdir -p $OUT
cp paper_1009_4975_b200/libtomesh.so /tmp/lib_keep.so
for r in 1 2; do for v in "$@"; do
  cp ab/lib_$v.so paper_1009_4975_b200/libtomesh.so
  echo "$v $(python tools/prof_gen.py ${CFG:-c4} 300 | awk '{print $5}')" | tee -a $OUT/ab.txt
done; done
cp /tmp/lib_keep.so paper_1009_4975_b200/libtomesh.so
