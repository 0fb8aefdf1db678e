#!/bin/bash
# Sharded path on one GPU: parity tests, the slab-count sweep (tools/shard_bench.py), bench --shard at N=1.
OUT=gpurun_out/${1:-shard}; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_shard.py ${PYTEST_EXTRA:-} -x -q > $OUT/pytest_gpu.log 2>&1; tail -2 $OUT/pytest_gpu.log
timeout 300 python tools/shard_bench.py 1 2 4 8 > $OUT/shard_bench.jsonl 2>&1; cut -c1-300 $OUT/shard_bench.jsonl
timeout 300 python bench.py --shard --steps 3 --warmup 3 > $OUT/bench_shard.log 2>&1; tail -1 $OUT/bench_shard.log | cut -c1-300
