#!/bin/bash
# Round-2 final verification on one B200: the whole GPU suite (incl. the
# full-size L2 parity against the cached oracle solutions), smoke(), the
# default bench line, the config sweep, ncu --set full of the general kernel
# on c4L, the ncu launch list of a short bench.
TAG=${1:-final}
OUT=gpurun_out/$TAG; mkdir -p $OUT
export PYTHONPATH=.
ls -la cache/oracle_ref > $OUT/cache_listing.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -s -rs > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 900 python bench.py > $OUT/bench.jsonl 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/bench.err
timeout 900 python tools/config_sweep.py > $OUT/config_sweep.jsonl 2> $OUT/config_sweep.err
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_gen_fused --launch-skip 20 --launch-count 1 \
    -o $OUT/gen_c4L_full python tools/prof_gen.py c4L 30 > $OUT/ncu_c4L.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1200 --csv \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-general > $OUT/launches.csv 2> $OUT/launches.err
grep -E "passed|failed" $OUT/pytest_gpu.log | tail -3; tail -2 $OUT/smoke.log; tail -c 400 $OUT/bench.jsonl
