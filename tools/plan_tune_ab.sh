#!/bin/bash
# Upload-time K1 plan check (new) vs the simulation-only choice (old): c3 and c5 per-iteration times.
OUT=gpurun_out/${1:-plantune}; mkdir -p $OUT
cp ab/lib_new.so paper_1009_4975_b200/libtomesh.so
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "c3s or c5s" 2>&1 | tail -1 | tee -a $OUT/ab.txt
for r in 1 2; do for v in old new; do
  cp ab/lib_$v.so paper_1009_4975_b200/libtomesh.so
  echo "$v $(for c in c3 c5; do python tools/config_sweep.py $c | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["config"], d["us_per_iter_fixed200"], d["upload_s"])'; done | tr '\n' ' ')" | tee -a $OUT/ab.txt
done; done
cp ab/lib_new.so paper_1009_4975_b200/libtomesh.so
