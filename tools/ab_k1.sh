#!/bin/bash
# Parity of the new build's structured path, then an A/B of ab/lib_old.so vs ab/lib_new.so (c5 bench).
OUT=gpurun_out/${1:-ab}; mkdir -p $OUT
cp ab/lib_new.so paper_1009_4975_b200/libtomesh.so
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q 2>&1 | tail -2 | tee -a $OUT/ab.txt
bash tools/ab_bench.sh ${1:-ab}
cp ab/lib_new.so paper_1009_4975_b200/libtomesh.so
