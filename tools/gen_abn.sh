#!/bin/bash
# General-path A/B of library builds ab/lib_<v>.so on one box: us per iteration
# (fixed 200) and iterations to tolerance on c1, c2, c4 and c4L, two rounds;
# then the GPU test suite on the last library.
# usage: gpurun -- bash tools/gen_abn.sh TAG v1 v2 ...
OUT=gpurun_out/${1:-genab}; shift; mkdir -p $OUT
CFGS=${CFGS:-"c1 c2 c4 c4L"}
for r in 1 2; do for v in "$@"; do
  cp ab/lib_$v.so paper_1009_4975_b200/libtomesh.so
  python tools/config_sweep.py $CFGS 2>>$OUT/err.txt | python -c '
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(sys.argv[1], d["config"], d["us_per_iter_fixed200"], d["iters"], d["solve_ms"], "blocks", d["gen_blocks"], "smem", d["gen_smem_bytes"], "loc/el max", d["gen_max_loc"], d["gen_max_el"], "recompute %.2f" % (d["gen_local_el"] / d["n_el"]), "local/node %.2f" % (d["gen_local_nodes"] / (d["n_dof"] / (3 if d["config"] != "c2" else 2))))' $v | tee -a $OUT/ab.txt
done; done
if [ -z "$NOTEST" ]; then
timeout 1200 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
tail -3 $OUT/pytest_gpu.log
fi
