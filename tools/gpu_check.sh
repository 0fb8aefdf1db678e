#!/bin/bash
# One gpurun session: GPU parity tests, smoke, short bench, ncu launch list.
# usage: gpurun -- bash tools/gpu_check.sh [tag]
TAG=${1:-r1}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $OUT/nvsmi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || echo "BUILD FAILED"
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" | tee -a $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" | tee -a $OUT/smoke.log
timeout 900 python bench.py --steps 3 --warmup 3 > $OUT/bench.log 2>&1; echo "bench rc=$?" | tee -a $OUT/bench.log
if [ "${NCU:-1}" = "1" ]; then
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $OUT/launches.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline > $OUT/ncu_launch.log 2>&1; echo "ncu rc=$?" | tee -a $OUT/ncu_launch.log
fi
tail -3 $OUT/pytest_gpu.log; tail -2 $OUT/bench.log
