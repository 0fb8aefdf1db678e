#!/bin/bash
# IC(0) triangular solves: warps per CTA (= rows per step) 8 / 16 / 32.
OUT=gpurun_out/${1:-ic0w}; mkdir -p $OUT
export PYTHONPATH=.
cp paper_1009_4975_b200/libtomesh.so /tmp/lib_keep.so
for w in 8 16 32; do
  cp ab/lib_ic$w.so paper_1009_4975_b200/libtomesh.so
  python tools/solver_compare.py c1 c2 2>/dev/null | grep minres_ic0 | python -c '
import json,sys
for l in sys.stdin:
    d=json.loads(l); print("warps", sys.argv[1], d["config"], "iters", d["iters"], "ms %.1f" % d["ms"], "us/it %.0f" % d["us_per_iter"])' $w | tee -a $OUT/ab.txt
done
cp /tmp/lib_keep.so paper_1009_4975_b200/libtomesh.so
