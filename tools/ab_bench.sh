#!/bin/bash
# A/B of two builds of libtomesh.so on the same box: ab/lib_old.so vs ab/lib_new.so, alternating.
OUT=gpurun_out/${1:-ab}; mkdir -p $OUT
for r in 1 2 3; do
  for v in old new; do
    cp ab/lib_$v.so paper_1009_4975_b200/libtomesh.so
    timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-general 2>/dev/null | grep "^{" | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$v', round(d['value'],1), round(r['avg_launch_ms']*1000,2), round(r['frac'],4))" | tee -a $OUT/ab.txt
  done
done
