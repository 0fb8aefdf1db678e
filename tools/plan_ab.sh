#!/bin/bash
# K1 grid plan on/off on the same box (TOMESH_S3_NO_PLAN), c5 bench.
OUT=gpurun_out/${1:-plan}; mkdir -p $OUT
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "c3s or c5s" 2>&1 | tail -1 | tee -a $OUT/ab.txt
for r in 1 2 3; do
  for v in on off; do
    if [ $v = on ]; then unset TOMESH_S3_NO_PLAN; else export TOMESH_S3_NO_PLAN=1; fi
    timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | grep "^{" | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('c5 plan=$v', round(d['value'],1), round(r['avg_launch_ms']*1000,2), round(r['frac'],4))" | tee -a $OUT/ab.txt
  done
done
