#!/bin/bash
# General-path change check: parity (normal + checking build), A/B vs a kept library, phase trace.
TAG=${1:-gchk}; shift
OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_amr.py tests/test_gpu_minres.py -m gpu -q -x > $OUT/pytest.log 2>&1; tail -2 $OUT/pytest.log
cp paper_1009_4975_b200/libtomesh.so /tmp/keep.so; cp ab/lib_debug.so paper_1009_4975_b200/libtomesh.so
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_amr.py -m gpu -q -x > $OUT/pytest_debug.log 2>&1; tail -2 $OUT/pytest_debug.log
cp /tmp/keep.so paper_1009_4975_b200/libtomesh.so
bash tools/gpu_gen_ab2.sh $TAG "$@"
bash tools/gpu_gf_trace.sh $TAG c4L
