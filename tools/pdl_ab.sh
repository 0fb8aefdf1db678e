#!/bin/bash
# PDL on/off on the same box: c5 bench K1 average launch duration and general-path iteration times.
OUT=gpurun_out/${1:-pdl}; mkdir -p $OUT
for r in 1 2; do
  for v in on off; do
    if [ $v = off ]; then export TOMESH_NO_PDL=1; else unset TOMESH_NO_PDL; fi
    timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | grep "^{" | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('c5 pdl=$v', round(d['value'],1), round(r['avg_launch_ms']*1000,2), round(r['frac'],4))" | tee -a $OUT/ab.txt
    echo -n "c4mid pdl=$v " | tee -a $OUT/ab.txt; python tools/prof_c4mid.py 8 4 4 3 30 | tee -a $OUT/ab.txt
    python tools/config_sweep.py c4 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c4 pdl=$v', d['us_per_iter_fixed200'])" | tee -a $OUT/ab.txt
  done
done
