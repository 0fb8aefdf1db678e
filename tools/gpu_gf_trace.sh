#!/bin/bash
TAG=${1:-gftrace}; shift
OUT=gpurun_out/$TAG; mkdir -p $OUT
cp paper_1009_4975_b200/libtomesh.so /tmp/lib_keep.so
cp ab/lib_trace.so paper_1009_4975_b200/libtomesh.so
for c in "$@"; do python tools/${TR:-gf}_trace.py $c 30 2>&1 | tee -a $OUT/trace.txt; done
cp /tmp/lib_keep.so paper_1009_4975_b200/libtomesh.so
